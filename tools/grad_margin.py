"""Gradient parity margin at C3 (2M triangles, 1297x840): per group, the worst
|got - want| / (1e-4 |want| + 1e-7) over all elements (the reference's own
criterion, test_backward.py:171), for the streaming, tile and exact backwards."""
import json
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(HERE, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import scale_golden as SG  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2505_19175_b200 import _lib, scenes  # noqa: E402
from paper_2505_19175_b200.rasterizer import DeviceSoup, Rasterizer  # noqa: E402

soup, intr, pose = scenes.make_scene("c3")
d_image = scenes.make_d_image(3, intr.height, intr.width, fp32=True)
gref = O.render_backward(soup, intr, pose, d_image=d_image)
rast = Rasterizer()
ds = DeviceSoup.from_soup(soup, dtype=torch.float32)
out = {}
for path in ("stream", "tile", "exact"):
    rast.set_option(_lib.TS_OPT_TILE_BACKWARD, 1 if path == "tile" else 0)
    rast.forward(ds, intr, pose, precision="exact" if path == "exact" else "fast")
    g = rast.backward(torch.as_tensor(d_image, dtype=torch.float32, device="cuda"))
    torch.cuda.synchronize()
    res = {}
    for k in SG.GROUPS:
        got = getattr(g, k).double().cpu().numpy()
        nb, worst = SG.grad_violations(got, getattr(gref, k))
        rel = np.abs(got - getattr(gref, k)) / np.maximum(np.abs(getattr(gref, k)), 1e-30)
        res[k] = {"worst_ratio_to_tolerance": round(worst, 4), "violations": nb,
                  "median_rel_err": float(np.median(rel[np.abs(getattr(gref, k)) > 1e-7]))}
    out[path] = res
rast.set_option(_lib.TS_OPT_TILE_BACKWARD, 0)
print(json.dumps(out, indent=1))
