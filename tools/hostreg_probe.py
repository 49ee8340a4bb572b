import time
import numpy as np
import torch

cr = torch.cuda.cudart()
a = np.random.default_rng(1).standard_normal((2_000_000, 16, 3))
d = torch.empty(a.shape, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for it in range(3):
    t0 = time.perf_counter()
    r = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t1 = time.perf_counter()
    d.copy_(torch.from_numpy(a), non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    cr.cudaHostUnregister(a.ctypes.data)
    t3 = time.perf_counter()
    print(f"register {1e3*(t1-t0):.2f} ms (rc {r}), copy {1e3*(t2-t1):.2f} ms ({a.nbytes/(t2-t1)/1e9:.1f} GB/s), unregister {1e3*(t3-t2):.2f} ms")
