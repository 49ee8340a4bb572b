"""Split of the default iteration's backward at C3: the caller's loss-weight
combination (torch element-wise) vs backward_fragments itself."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_19175_b200 import losses, scenes  # noqa: E402
from paper_2505_19175_b200.rasterizer import DeviceSoup, Rasterizer  # noqa: E402

c3 = scenes.CONFIGS["c3"]
ds = DeviceSoup.from_soup(scenes.make_soup(c3.n, c3.seed, c3.size, c3.sigma), dtype=torch.float32)
intr, _ = scenes.frontal_camera(c3.width, c3.height, c3.f)
pose = scenes.orbit_cameras(4, seed=4)[1]
target = torch.rand((c3.height, c3.width, 3), device="cuda")
r = Rasterizer()
f = r.forward(ds, intr, pose)
fr = r.fragments()
_, d_img = losses.photometric_loss(f.image, target, 0.2, rasterizer=r)
_, d_w, d_z = losses.distortion_loss(fr, rasterizer=r)
dep = losses.depth_from_fragments(fr, c3.height, c3.width, rasterizer=r)
_, _, d_w2 = losses.normal_loss(ds, fr, dep, intr, pose, rasterizer=r)
print("fragments", int(fr.weight.numel()))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for rep in range(4):
    ev[0].record()
    a, b = d_w * 100.0 + d_w2 * 1e-4, d_z * 100.0
    ev[1].record()
    g = r.backward_fragments(d_img, fr.offsets, a, b, weight=fr.weight)
    ev[2].record()
    torch.cuda.synchronize()
    print(f"combine {ev[0].elapsed_time(ev[1]):.3f} ms  backward_fragments {ev[1].elapsed_time(ev[2]):.3f} ms")
