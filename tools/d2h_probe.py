import time
import torch

def t(f, k=10):
    f(); f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        r = f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e3

n = 61 << 20
d = torch.empty(n // 8, dtype=torch.float64, device="cuda")
print("pinned alloc 61 MB:", round(t(lambda: torch.empty(n // 8, dtype=torch.float64, pin_memory=True)), 3), "ms")
h = torch.empty(n // 8, dtype=torch.float64, pin_memory=True)
def cp():
    h.copy_(d, non_blocking=True); torch.cuda.current_stream().synchronize()
print("D2H 61 MB into preallocated pinned:", round(t(cp), 3), "ms")
def both():
    x = torch.empty(n // 8, dtype=torch.float64, pin_memory=True)
    x.copy_(d, non_blocking=True); torch.cuda.current_stream().synchronize()
    return x
print("alloc + D2H:", round(t(both), 3), "ms")
def both_np():
    x = torch.empty(n // 8, dtype=torch.float64, pin_memory=True)
    x.copy_(d, non_blocking=True); torch.cuda.current_stream().synchronize()
    return x.numpy()
print("alloc + D2H + numpy():", round(t(both_np), 3), "ms")
