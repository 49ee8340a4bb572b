"""Fused Adam on the device: drop-in for the reference's
``adam_step`` / ``AdamState`` (trisplat/training.py:49-110) over a
``DeviceSoup`` (fp32 parameters, updated in place) and ``DeviceGrads``.

Same semantics as the reference: the first triangle with a non-finite
gradient (first group in vertices, opacity, sigma, sh order) raises
``ValueError("non-finite <group> gradient for triangle <i>")`` before any
state changes; otherwise t += 1, bias-corrected Adam per group with the
per-group learning rates, then opacity clamped to (1e-4, 1-1e-4) and sigma
to (1e-3, 1e3).  Moments are fp32 device buffers in the flat gradient layout.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

GROUPS = ("vertices", "opacity", "sigma", "sh")


@dataclass
class DeviceAdamState:
    m: "object"       # torch fp32 (59 N,)
    v: "object"
    n: int
    t_dev: "object"   # torch int64 (1,): steps taken (AdamState.t), kept on the device

    @classmethod
    def zeros(cls, n: int, device="cuda") -> "DeviceAdamState":
        import torch
        return cls(torch.zeros(59 * n, dtype=torch.float32, device=device),
                   torch.zeros(59 * n, dtype=torch.float32, device=device), n,
                   torch.zeros(1, dtype=torch.int64, device=device))

    @property
    def t(self) -> int:
        """Steps taken (reads the device counter: the kernel advances it only
        when an update ran, so a step skipped for a non-finite gradient does not
        count, as in the reference, which raises without touching the state)."""
        return int(self.t_dev.item())

    @t.setter
    def t(self, value: int):
        self.t_dev.fill_(int(value))

    def remap(self, origin, rasterizer=None, stream=None) -> "DeviceAdamState":
        """AdamState.remap (training.py:64-78) after densification: output
        triangle i takes the moments of origin[i] (zeros where origin[i] < 0);
        one row gather per parameter group on the device."""
        import numpy as np
        import torch
        from . import _lib
        from .rasterizer import default_rasterizer
        r = rasterizer or default_rasterizer()
        org = torch.as_tensor(np.asarray(origin, dtype=np.int64)).to("cuda")
        n_new = int(org.numel())
        new = DeviceAdamState.zeros(n_new)
        new.t_dev.copy_(self.t_dev)
        st = ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)
        o_old = o_new = 0
        for w in (9, 1, 1, 48):
            for a, b in ((self.m, new.m), (self.v, new.v)):
                _lib.check(r.lib.ts_gather_rows(r._ctx, n_new, ctypes.c_void_p(org.data_ptr()),
                                                ctypes.c_void_p(a.data_ptr() + 4 * o_old),
                                                ctypes.c_void_p(b.data_ptr() + 4 * o_new), w, 4, st), "gather_rows")
            o_old += w * self.n
            o_new += w * n_new
        return new


def adam_step(soup, grads, state: DeviceAdamState, lrs: dict, rasterizer=None, stream=None, check=True):
    """One in-place Adam update of ``soup`` (DeviceSoup, fp32) with ``grads``
    (DeviceGrads).  ``check=False`` skips the host read of the finiteness flags:
    the device still skips the whole update (step count included) if any
    gradient is non-finite; the flags stay in ``state.last_bad`` (device
    int64[4], -1 = finite) for the caller to inspect."""
    import torch
    from . import _lib
    from .rasterizer import default_rasterizer
    if soup.vertices.dtype != torch.float32:
        raise TypeError("adam_step needs fp32 device parameters")
    n = len(soup)
    if state.n != n or grads.n != n:
        raise ValueError("state / gradient size differs from the soup")
    r = rasterizer or default_rasterizer()
    bad = torch.empty(4, dtype=torch.int64, device="cuda")
    lr = (ctypes.c_double * 4)(*[float(lrs[k]) for k in GROUPS])
    st = (stream or torch.cuda.current_stream()).cuda_stream
    g = grads._ts()
    rc = r.lib.ts_adam_step(r._ctx, ctypes.c_void_p(soup.vertices.data_ptr()),
                            ctypes.c_void_p(soup.opacity.data_ptr()), ctypes.c_void_p(soup.sigma.data_ptr()),
                            ctypes.c_void_p(soup.sh.data_ptr()), n, ctypes.byref(g),
                            ctypes.c_void_p(state.m.data_ptr()), ctypes.c_void_p(state.v.data_ptr()),
                            ctypes.c_void_p(state.t_dev.data_ptr()), lr, ctypes.c_void_p(bad.data_ptr()),
                            ctypes.c_void_p(st))
    _lib.check(rc, "adam_step")
    state.last_bad = bad
    if check:
        b = bad.cpu().tolist()
        for k, i in zip(GROUPS, b):
            if i >= 0:
                raise ValueError(f"non-finite {k} gradient for triangle {i}")
    return state
