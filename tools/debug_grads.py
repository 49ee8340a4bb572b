"""Debug: compare per-triangle screen-space gradients GPU vs oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle as O
from paper_2505_19175_b200 import scenes
from paper_2505_19175_b200.rasterizer import Rasterizer, DeviceSoup
mode = sys.argv[1] if len(sys.argv) > 1 else "normalized"
soup = scenes.make_soup(200_000, seed=7, size=0.03, sigma=(0.3, 3.0))
intr, pose = scenes.frontal_camera(640, 360, 560.0)
r = Rasterizer()
ds = DeviceSoup.from_soup(soup)
bg = (0.2, 0.1, 0.3)
fwd = r.forward(ds, intr, pose, mode=mode, background=bg, precision="exact", debug=True)
d_image = scenes.make_d_image(7, intr.height, intr.width)
g = r.backward(torch.as_tensor(d_image, dtype=torch.float32, device="cuda"))
sg = r.dump_sgrad(len(soup))
osg = O.render_backward(soup, intr, pose, mode=mode, background=bg, d_image=d_image, return_screen=True)
names = ["gq0x","gq0y","gq1x","gq1y","gq2x","gq2y","go","gsig","gr","gg","gb","gphis","gz"]
for j, nm in enumerate(names):
    a, b = sg[:, j], osg[:, j]
    d = np.abs(a - b)
    i = int(np.argmax(d))
    print(f"{nm:6s} maxabs={np.abs(b).max():.3e} maxdiff={d.max():.3e} at {i}: gpu={a[i]:.6e} ora={b[i]:.6e}")
go = O.render_backward(soup, intr, pose, mode=mode, background=bg, d_image=d_image)
dv = g.d_vertices.double().cpu().numpy(); ov = go.d_vertices
d = np.abs(dv - ov).reshape(len(soup), -1).max(1)
i = int(np.argmax(d)); print("worst dv tri", i, dv[i].ravel(), ov[i].ravel())
print("sgrad gpu", sg[i]); print("sgrad ora", osg[i])
print("verts", soup.vertices[i], "sigma", soup.sigma[i], "opa", soup.opacity[i])
