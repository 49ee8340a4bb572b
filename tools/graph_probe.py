"""Capture an asynchronous north-star forward in a CUDA graph and replay it."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_19175_b200 import scenes  # noqa: E402
from paper_2505_19175_b200.rasterizer import DeviceSoup, Rasterizer  # noqa: E402

soup, intr, pose = scenes.make_scene("ns")
ds = DeviceSoup.from_soup(soup, dtype=torch.float32)
r = Rasterizer()
ref = r.forward(ds, intr, pose, keep_backward=False)
img_ref = ref.image.clone()
r.set_async(True)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        out = r.forward(ds, intr, pose, keep_backward=False)
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    out = r.forward(ds, intr, pose, keep_backward=False)
torch.cuda.synchronize()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
print("graph image equal:", torch.equal(out.image, img_ref))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(f"graph replay: {200 / e0.elapsed_time(e1) * 1e3:.1f} frames/s")
print(r.status())
