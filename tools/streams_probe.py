"""Frames of the north-star scene on 1, 2 or 3 rasterizer contexts, each on its
own CUDA stream (independent frames in flight): whole-job frames/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_19175_b200 import scenes  # noqa: E402
from paper_2505_19175_b200.rasterizer import DeviceSoup, Rasterizer  # noqa: E402

soup, intr, pose = scenes.make_scene("ns")
ds = DeviceSoup.from_soup(soup, dtype=torch.float32)
K = 300
for ns in (1, 2, 3, 1, 2):
    rs = [Rasterizer() for _ in range(ns)]
    sts = [torch.cuda.Stream() for _ in range(ns)]
    for r, s in zip(rs, sts):
        with torch.cuda.stream(s):
            r.forward(ds, intr, pose, keep_backward=False)
            r.set_async(True)
            for _ in range(20):
                r.forward(ds, intr, pose, keep_backward=False)
    torch.cuda.synchronize()
    cur = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for s in sts:
        s.wait_stream(cur)
    for i in range(K):
        with torch.cuda.stream(sts[i % ns]):
            rs[i % ns].forward(ds, intr, pose, keep_backward=False)
    for s in sts:
        cur.wait_stream(s)
    e1.record(cur)
    torch.cuda.synchronize()
    for r, s in zip(rs, sts):
        r.status(stream=s)
    ms = e0.elapsed_time(e1)
    print(f"{ns} stream(s): {K / ms * 1e3:.1f} frames/s ({ms / K:.4f} ms/frame)")
    del rs
