"""Work statistics of the forward blend (debug build with -DTS_BLEND_STATS).

    python tools/blend_stats.py [workload]     # on the GPU box
Builds a separate library into _stats/ (not the product .so) and renders one frame.
"""
import ctypes
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)
from paper_2505_19175_b200 import build as B  # noqa: E402

out = os.path.join(HERE, "_stats")
os.makedirs(out, exist_ok=True)
lib = os.path.join(out, "libstats.so")
if not os.path.exists(lib):
    objs = []
    for src in B.sources():
        o = os.path.join(out, src.replace(".cu", ".o"))
        subprocess.run([B.nvcc()] + B.ARCH + B.COMMON + B.EXTRA.get(src, []) + ["-DTS_BLEND_STATS", "-c",
                        os.path.join(B.CSRC, src), "-o", o], check=True)
        objs.append(o)
    subprocess.run([B.nvcc()] + B.ARCH + ["-shared", "-o", lib] + objs + ["-lcudart"], check=True)
if len(sys.argv) > 1 and sys.argv[1] == "--build-only":
    sys.exit(0)
import torch  # noqa: E402

from paper_2505_19175_b200 import _lib, scenes  # noqa: E402
L = _lib.load(lib)
from paper_2505_19175_b200.rasterizer import DeviceSoup, Rasterizer  # noqa: E402

cfg = scenes.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "ns"]
soup, intr, pose = scenes.make_scene(cfg)
ds = DeviceSoup.from_soup(soup, dtype=torch.float32)
r = Rasterizer(0)
r.forward(ds, intr, pose, precision="fast", keep_backward=False)
st = (ctypes.c_ulonglong * 16)()
L.ts_debug_blend_stats(st, 1)
r.forward(ds, intr, pose, precision="fast", keep_backward=False)
L.ts_debug_blend_stats(st, 0)
names = ["tiles", "batches", "pairs", "pairs_done_pixel", "passing", "composite_iters", "live_px_at_batch",
         "entries_total", "entries_consumed"]
v = {n: st[i] for i, n in enumerate(names)}
print(v)
t = v["tiles"]
print("per tile: batches %.2f pairs %.0f (done-pixel %.1f%%) passing %.0f composite %.0f live/batch %.1f "
      "entries %.0f consumed %.0f pairs/entry %.1f" % (
          v["batches"] / t, v["pairs"] / t, 100 * v["pairs_done_pixel"] / max(v["pairs"], 1), v["passing"] / t,
          v["composite_iters"] / t, v["live_px_at_batch"] / max(v["batches"], 1), v["entries_total"] / t,
          v["entries_consumed"] / t, v["pairs"] / max(v["entries_consumed"], 1)))
