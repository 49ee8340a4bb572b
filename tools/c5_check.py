"""c5 stress config (5M triangles, 1920x1080, sigma 0.1): tile-list structure and
depth order properties, determinism, fast vs exact precision agreement."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_19175_b200 import scenes
from paper_2505_19175_b200.rasterizer import DeviceSoup, Rasterizer
soup, intr, pose = scenes.make_scene("c5")
ds = DeviceSoup.from_soup(soup, dtype=torch.float32)
r = Rasterizer()
a = r.forward(ds, intr, pose, debug=True, keep_backward=False)
m, e = a.n_visible, a.n_entries
ntiles = ((intr.width + 15) // 16) * ((intr.height + 15) // 16)
ts = r.dump_tile_start(ntiles)
print("visible", m, "entries", e, "max tile", int(np.diff(ts).max()), "tiles>2048", int((np.diff(ts) > 2048).sum()))
er = r.dump_entry_rank(e)
seg = np.repeat(np.arange(ntiles), np.diff(ts))
same = seg[1:] == seg[:-1]
assert np.all(er[1:][same] > er[:-1][same]), "rank order"
img = a.image.clone()
b = r.forward(ds, intr, pose, debug=True, keep_backward=False)
assert torch.equal(img, b.image)
x = r.forward(ds, intr, pose, precision="exact", debug=True, keep_backward=False)
d = (x.image - img).abs().max().item()
print("fast vs exact max |drgb|", d, "last_src equal", torch.equal(x.last_src, b.last_src))
assert d <= 1e-5
