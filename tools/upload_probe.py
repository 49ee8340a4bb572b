"""Packed fp32 upload of the north-star fp64 soup: chunk size / ring depth sweep."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_19175_b200 import rasterizer as R, scenes  # noqa: E402

soup, intr, pose = scenes.make_scene("ns")
for chunk_mb, nbuf in ((16, 6), (32, 4), (32, 6), (64, 3), (64, 4)):
    R._STAGE32_CHUNK, R._STAGE32_NBUF = chunk_mb << 20, nbuf
    R._STAGE32.clear()
    R.DeviceSoup.from_soup_f32_exact(soup)
    torch.cuda.synchronize()
    ts = []
    for _ in range(8):
        t0 = time.perf_counter()
        R.DeviceSoup.from_soup_f32_exact(soup)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    ts.sort()
    print(f"chunk {chunk_mb} MB x {nbuf}: median {ts[len(ts) // 2]:.2f} ms, best {ts[0]:.2f} ms")
