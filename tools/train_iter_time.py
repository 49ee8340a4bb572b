"""One default training iteration of the reference (training.py:121-160 with
beta_distortion, beta_normal > 0: fragments every iteration) on the device at
C3 (2M triangles, 1297x840): forward with fragment collection, photometric +
distortion + normal losses, backward with fragment gradients.  CUDA events per
part, for DESIGN.md."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_19175_b200 import losses, scenes  # noqa: E402
from paper_2505_19175_b200.rasterizer import DeviceSoup, Rasterizer  # noqa: E402

c3 = scenes.CONFIGS["c3"]
soup = scenes.make_soup(c3.n, c3.seed, c3.size, c3.sigma)
ds = DeviceSoup.from_soup(soup, dtype=torch.float32)
intr, _ = scenes.frontal_camera(c3.width, c3.height, c3.f)
pose = scenes.orbit_cameras(4, seed=4)[1]
target = torch.rand((c3.height, c3.width, 3), device="cuda")
r = Rasterizer()


def it(ev=None):
    mark = (lambda k: ev[k].record()) if ev else (lambda k: None)
    mark(0)
    f = r.forward(ds, intr, pose)
    mark(1)
    frags = r.fragments()
    mark(2)
    _, d_img = losses.photometric_loss(f.image, target, 0.2, rasterizer=r)
    _, d_w, d_z = losses.distortion_loss(frags, rasterizer=r)
    depth = losses.depth_from_fragments(frags, c3.height, c3.width, rasterizer=r)
    _, dv, d_w2 = losses.normal_loss(ds, frags, depth, intr, pose, rasterizer=r)
    mark(3)
    g = r.backward_fragments(d_img, frags.offsets, d_w * 100.0 + d_w2 * 1e-4, d_z * 100.0, weight=frags.weight)
    mark(4)
    return g


for _ in range(2):
    it()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
it(ev)
torch.cuda.synchronize()
names = ["forward", "collect_fragments", "losses", "backward_fragments"]
res = {n: round(ev[i].elapsed_time(ev[i + 1]), 3) for i, n in enumerate(names)}
res["total_ms"] = round(ev[0].elapsed_time(ev[4]), 3)
res["fragments"] = int(r.fragments().weight.numel())
r.profile(True)
it()
torch.cuda.synchronize()
res["stages_last"] = {k: round(v, 3) for k, v in r.stage_times().items() if k in ("blend_bwd", "chain_bwd")}
r.profile(False)
print(res)
