"""Host logic of render()'s page-locked output pool (CPU: pin_memory stubbed):
a buffer is reused only after every numpy array handed out from it is gone,
and free buffers too small for a new request are released."""
import gc

import torch

from paper_2505_19175_b200 import rasterizer as R


def test_pool_reuse_and_release(monkeypatch):
    orig = torch.empty

    def fake_empty(*a, **k):
        k.pop("pin_memory", None)
        return orig(*a, **k)

    monkeypatch.setattr(R.torch, "empty", fake_empty)
    pool = R._PinnedPool()
    h1, a1 = pool.get(1000, torch.float64)
    view = a1[10:20]                       # an output array derived from the buffer
    del h1, a1
    gc.collect()
    h2, a2 = pool.get(1000, torch.float64)
    assert len(pool.entries) == 2          # the first buffer is still referenced by `view`
    view[:] = 7.0
    del view
    gc.collect()
    h3, a3 = pool.get(800, torch.float64)
    assert len(pool.entries) == 2          # reused the first buffer
    del h2, a2, h3, a3
    gc.collect()
    h4, a4 = pool.get(10 ** 6, torch.float64)
    assert len(pool.entries) == 1 and a4.size == 10 ** 6
