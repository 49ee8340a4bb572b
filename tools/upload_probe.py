"""Lossless fp32 upload of the north-star fp64 soup (ts_upload_f32): chunk size,
ring depth and store kind sweep."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_19175_b200 import rasterizer as R, scenes  # noqa: E402

soup, intr, pose = scenes.make_scene("ns")
cfgs = [(c, s, f) for f in (0, 1) for c, s in ((1, 4), (2, 4), (4, 4), (8, 4), (16, 4), (32, 6), (4, 8))]
for chunk_mb, nslot, flags in cfgs:
    R._UPLOAD_F32 = (chunk_mb << 20, nslot, flags)
    R.DeviceSoup.from_soup_f32_exact(soup)
    torch.cuda.synchronize()
    ts = []
    for _ in range(8):
        t0 = time.perf_counter()
        R.DeviceSoup.from_soup_f32_exact(soup)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    ts.sort()
    print(f"chunk {chunk_mb:2d} MB x {nslot} {'stream' if flags & 1 else 'store '}: "
          f"median {ts[len(ts) // 2]:.2f} ms, best {ts[0]:.2f} ms")
