"""Per-parameter-group gradient errors of the view-parallel test scene (GPU), for
choosing the accumulation precision of the streaming backward."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from conftest import rel_err
from oracle import oracle as O
from paper_2505_19175_b200 import scenes
from paper_2505_19175_b200.rasterizer import DeviceSoup, Rasterizer
soup = scenes.make_soup(2000, seed=21, size=0.2, sigma=(0.5, 3.0))
intr, _ = scenes.frontal_camera(96, 80, 100.0)
poses = scenes.orbit_cameras(4, seed=4)
r = Rasterizer()
ds = DeviceSoup.from_soup(soup, dtype=torch.float32)
worst = {}
for v in range(4):
    d = np.random.default_rng(100 + v).normal(size=(80, 96, 3))
    r.forward(ds, intr, poses[v], precision="fast")
    g = r.backward(torch.as_tensor(d, dtype=torch.float32, device="cuda"))
    gr = O.render_backward(soup, intr, poses[v], d_image=d)
    for k in ("d_vertices", "d_opacity", "d_sigma", "d_sh"):
        e = rel_err(getattr(g, k).double().cpu().numpy(), getattr(gr, k))
        worst[k] = max(worst.get(k, 0), e)
print({k: "%.2e" % v for k, v in worst.items()})
