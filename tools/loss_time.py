import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_19175_b200 import losses as DL
x = torch.rand((840, 1297, 3), device="cuda"); y = torch.rand((840, 1297, 3), device="cuda")
for _ in range(5): DL.photometric_loss(x, y, 0.2)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
from paper_2505_19175_b200.rasterizer import default_rasterizer
import ctypes
r = default_rasterizer(); out = torch.empty(2, dtype=torch.float64, device="cuda"); g = torch.empty_like(x)
st = torch.cuda.current_stream().cuda_stream
e0.record()
for _ in range(100):
    r.lib.ts_photometric_loss(r._ctx, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), 840, 1297, 0.2, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(st))
e1.record(); torch.cuda.synchronize()
print("photometric loss 1297x840: %.1f us" % (e0.elapsed_time(e1) * 10))
