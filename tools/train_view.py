"""One C3 training view (forward with fragment records + streaming backward +
chain), repeated a few times: a small target for ncu captures of the training
kernels (`ncu -k regex:k_blend_dense -s 2 -c 1 python tools/train_view.py`)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_19175_b200 import scenes  # noqa: E402
from paper_2505_19175_b200.rasterizer import DeviceSoup, Rasterizer  # noqa: E402

cfg = scenes.CONFIGS["c3"]
soup, intr, _ = scenes.make_scene(cfg)
poses = scenes.orbit_cameras(4, seed=4)
rast = Rasterizer(0)
ds = DeviceSoup.from_soup(soup, dtype=torch.float32)
d = torch.randn((cfg.height, cfg.width, 3), device="cuda", generator=torch.Generator("cuda").manual_seed(103))
g = None
for p in poses:
    rast.forward(ds, intr, p, keep_backward=True)
    g = rast.backward(d, g, accumulate=g is not None)
torch.cuda.synchronize()
print("ok")
