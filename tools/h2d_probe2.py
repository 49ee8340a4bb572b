"""Upload variants for the drop-in render()'s 944 MB fp64 soup."""
import time

import numpy as np
import torch

n = 2_000_000
arrs = [np.random.default_rng(0).standard_normal((n, 3, 3)), np.ones(n), np.ones(n),
        np.random.default_rng(1).standard_normal((n, 16, 3))]
tot = sum(a.nbytes for a in arrs)
dev = [torch.empty(a.shape, dtype=torch.float64, device="cuda") for a in arrs]


def timeit(f, k=6):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k


def make(chunk, nbuf, nstream):
    ring = [torch.empty(chunk, dtype=torch.uint8).pin_memory() for _ in range(nbuf)]
    evs = [torch.cuda.Event() for _ in range(nbuf)]
    streams = [torch.cuda.Stream() for _ in range(nstream)]
    cur = torch.cuda.current_stream()

    def run():
        i = 0
        for a, d in zip(arrs, dev):
            src = torch.from_numpy(a.reshape(-1).view(np.uint8))
            dst = d.reshape(-1).view(torch.uint8)
            for s in range(0, src.numel(), chunk):
                c = min(chunk, src.numel() - s)
                slot = i % nbuf
                st = streams[i % nstream]
                evs[slot].synchronize()
                ring[slot][:c].copy_(src[s:s + c])
                st.wait_stream(cur) if i < nstream else None
                with torch.cuda.stream(st):
                    dst[s:s + c].copy_(ring[slot][:c], non_blocking=True)
                    evs[slot].record(st)
                i += 1
        for st in streams:
            cur.wait_stream(st)
    return run


for chunk, nbuf, nst in [(32 << 20, 3, 1), (32 << 20, 4, 2), (16 << 20, 6, 2), (64 << 20, 4, 2), (8 << 20, 8, 2),
                         (16 << 20, 8, 4)]:
    dt = timeit(make(chunk, nbuf, nst))
    print(f"chunk {chunk >> 20} MB x{nbuf} buffers, {nst} streams: {dt * 1e3:.1f} ms {tot / dt / 1e9:.1f} GB/s")
print("torch threads", torch.get_num_threads())
