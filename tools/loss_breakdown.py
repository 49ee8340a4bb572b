"""Device time of each loss of the reference's default training iteration at C3."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_19175_b200 import losses, scenes  # noqa: E402
from paper_2505_19175_b200.rasterizer import DeviceSoup, Rasterizer  # noqa: E402

c3 = scenes.CONFIGS["c3"]
ds = DeviceSoup.from_soup(scenes.make_soup(c3.n, c3.seed, c3.size, c3.sigma), dtype=torch.float32)
intr, _ = scenes.frontal_camera(c3.width, c3.height, c3.f)
pose = scenes.orbit_cameras(4, seed=4)[1]
target = torch.rand((c3.height, c3.width, 3), device="cuda")
r = Rasterizer()
f = r.forward(ds, intr, pose)
frags = r.fragments()
parts = {
    "photometric(L1+SSIM)": lambda: losses.photometric_loss(f.image, target, 0.2, rasterizer=r),
    "distortion": lambda: losses.distortion_loss(frags, rasterizer=r),
    "depth_from_fragments": lambda: losses.depth_from_fragments(frags, c3.height, c3.width, rasterizer=r),
}
depth = losses.depth_from_fragments(frags, c3.height, c3.width, rasterizer=r)
parts["normal"] = lambda: losses.normal_loss(ds, frags, depth, intr, pose, rasterizer=r)
for name, fn in parts.items():
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 5:.3f} ms")
