"""Host<->device copy rates for the drop-in render() e2e (944 MB fp64 soup)."""
import time

import numpy as np
import torch

n = 2_000_000
arrs = [np.random.default_rng(0).standard_normal((n, 3, 3)), np.ones(n), np.ones(n),
        np.random.default_rng(1).standard_normal((n, 16, 3))]
tot = sum(a.nbytes for a in arrs)
torch.cuda.synchronize()


def timeit(f, k=5):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k


def pageable():
    return [torch.from_numpy(a).to("cuda") for a in arrs]


print("torch threads", torch.get_num_threads())
dt = timeit(pageable)
print(f"pageable H2D: {dt*1e3:.1f} ms  {tot/dt/1e9:.1f} GB/s")
CH = 64 << 20
ring = [torch.empty(CH, dtype=torch.uint8).pin_memory() for _ in range(3)]
evs = [torch.cuda.Event() for _ in range(3)]
dev = torch.empty(tot, dtype=torch.uint8, device="cuda")


def staged():
    off = 0
    i = 0
    for a in arrs:
        src = torch.from_numpy(a.reshape(-1).view(np.uint8))
        for s in range(0, src.numel(), CH):
            c = min(CH, src.numel() - s)
            slot = i % 3
            evs[slot].synchronize()
            ring[slot][:c].copy_(src[s:s + c])
            dev[off:off + c].copy_(ring[slot][:c], non_blocking=True)
            evs[slot].record()
            off += c
            i += 1


dt = timeit(staged)
print(f"staged pinned H2D: {dt*1e3:.1f} ms  {tot/dt/1e9:.1f} GB/s")
pin = torch.empty(tot, dtype=torch.uint8).pin_memory()
dt = timeit(lambda: dev.copy_(pin, non_blocking=True))
print(f"pinned H2D DMA only: {dt*1e3:.1f} ms  {tot/dt/1e9:.1f} GB/s")
src = torch.from_numpy(np.concatenate([a.reshape(-1) for a in arrs]).view(np.uint8))
dt = timeit(lambda: pin.copy_(src))
print(f"host memcpy into pinned (torch copy_): {dt*1e3:.1f} ms  {tot/dt/1e9:.1f} GB/s")
out = np.empty(80 << 20, dtype=np.uint8)
d = torch.empty(80 << 20, dtype=torch.uint8, device="cuda")
dt = timeit(lambda: torch.from_numpy(out).copy_(d))
print(f"pageable D2H 80 MB: {dt*1e3:.2f} ms  {out.nbytes/dt/1e9:.1f} GB/s")
dt = timeit(lambda: d.cpu())
print(f".cpu() 80 MB: {dt*1e3:.2f} ms")
