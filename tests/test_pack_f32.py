"""ts_pack_f32, the host half of render()'s upload of the reference's fp64 soups
(CPU only: no device memory involved): fp64 -> fp32 conversion on the library's
host thread pool, reporting whether every value converted exactly."""
import numpy as np
import pytest


def _pack(a, threads=0):
    import ctypes

    from paper_2505_19175_b200 import _lib
    lib = _lib.load()
    a = np.ascontiguousarray(a, dtype=np.float64)
    out = np.empty(a.size, dtype=np.float32)
    rc = lib.ts_pack_f32(ctypes.c_void_p(a.ctypes.data), ctypes.c_void_p(out.ctypes.data), a.size, threads)
    return rc, out


@pytest.mark.parametrize("n", [0, 1, 1000, (1 << 16) + 7, 3_000_001])
@pytest.mark.parametrize("threads", [0, 1, 3])
def test_pack_exact_and_inexact(n, threads):
    rng = np.random.default_rng(n)
    a = rng.normal(size=n).astype(np.float32).astype(np.float64)
    rc, out = _pack(a, threads)
    assert rc == 1
    assert np.array_equal(out, a.astype(np.float32))
    if n:
        b = a.copy()
        b[n // 2] += 1e-12 * max(1.0, abs(b[n // 2]))   # one value that is not an fp32 value
        rc, out = _pack(b, threads)
        assert rc == 0
        assert np.array_equal(out, b.astype(np.float32))


def test_pack_non_finite():
    rc, _ = _pack(np.array([1.0, np.nan, 2.0]))
    assert rc == 0                       # NaN: the upload falls back to fp64 (which reports it)
    rc, out = _pack(np.array([1.0, np.inf, -np.inf]))
    assert rc == 1 and np.isinf(out[1:]).all()
    rc, _ = _pack(np.array([1e300]))     # out of fp32 range
    assert rc == 0


def test_pack_invalid():
    import ctypes

    from paper_2505_19175_b200 import _lib
    assert _lib.load().ts_pack_f32(None, None, 5, 0) == _lib.TS_ERR_INVALID_ARG
    assert _lib.load().ts_pack_f32(ctypes.c_void_p(8), ctypes.c_void_p(8), -1, 0) == _lib.TS_ERR_INVALID_ARG
