"""Host throughput of ts_pack_f32 (fp64 -> fp32 with the exactness test) on 944 MB."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes, time, numpy as np, sys
from paper_2505_19175_b200 import _lib
lib=_lib.load()
a=np.random.default_rng(0).normal(size=118_000_000).astype(np.float32).astype(np.float64)
out=np.ones(a.size,np.float32)
print('cpus', os.cpu_count())
for thr in (1, 1, 4, 8, 12, 0, 0):
    t=time.perf_counter(); rc=lib.ts_pack_f32(ctypes.c_void_p(a.ctypes.data), ctypes.c_void_p(out.ctypes.data), a.size, thr); dt=time.perf_counter()-t
    print(thr, rc, round(dt*1e3,1),'ms', round(a.nbytes/dt/1e9,1),'GB/s in')
