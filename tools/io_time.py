"""Wall-clock of the model I/O and density drop-ins at the north-star size
(2M triangles), for DESIGN.md: PLY export / import through the device
pack / unpack, and the PLY body kernels alone (CUDA events)."""
import os
import sys
import tempfile
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_19175_b200 import scene_io as IO  # noqa: E402
from paper_2505_19175_b200 import scenes  # noqa: E402
from paper_2505_19175_b200.rasterizer import DeviceSoup  # noqa: E402

soup = scenes.make_soup(2_000_000, seed=3, size=0.02, sigma=1.0)
ds = DeviceSoup.from_soup(soup, dtype=torch.float32)
IO.ply_body(ds)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    IO.ply_body(ds)
e1.record()
torch.cuda.synchronize()
pack_ms = e0.elapsed_time(e1) / 10
with tempfile.TemporaryDirectory() as td:
    p = os.path.join(td, "m.ply")
    IO.export_mesh(ds, p)
    t = time.perf_counter()
    IO.export_mesh(ds, p)
    exp_ms = (time.perf_counter() - t) * 1e3
    IO.import_ply(p, sigma=1.0)
    torch.cuda.synchronize()
    t = time.perf_counter()
    IO.import_ply(p, sigma=1.0)
    torch.cuda.synchronize()
    imp_ms = (time.perf_counter() - t) * 1e3
    size = os.path.getsize(p)
print({"ply_pack_kernel_ms": round(pack_ms, 4), "pack_GBps": round((36 + 12 + 61) * 2e6 / (pack_ms / 1e3) / 1e9, 1),
       "export_ms": round(exp_ms, 1), "import_ms": round(imp_ms, 1), "file_MB": round(size / 1e6, 1)})
