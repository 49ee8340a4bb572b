"""GPU parity of the fused Adam step (ts_optim.cu) against the oracle and the
live reference's fixtures, plus the reference's own adam tests
(test_training.py:52-107) on the device."""
import os

import numpy as np
import pytest

from oracle import optim as OP

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "adam.npz")


def _dev(v, o, s, h):
    from paper_2505_19175_b200.rasterizer import DeviceSoup
    t = lambda a: torch.as_tensor(np.asarray(a, dtype=np.float32), device="cuda").contiguous()  # noqa: E731
    return DeviceSoup(t(v), t(o), t(s), t(h))


def _grads(n, gv, go, gs, gh):
    from paper_2505_19175_b200.rasterizer import DeviceGrads
    g = DeviceGrads.zeros(n)
    g.d_vertices.copy_(torch.as_tensor(np.asarray(gv, np.float32)))
    g.d_opacity.copy_(torch.as_tensor(np.asarray(go, np.float32)))
    g.d_sigma.copy_(torch.as_tensor(np.asarray(gs, np.float32)))
    g.d_sh.copy_(torch.as_tensor(np.asarray(gh, np.float32)))
    return g


def _np(t):
    return t.detach().double().cpu().numpy()


def test_matches_reference_steps():
    from paper_2505_19175_b200.optim import DeviceAdamState, adam_step
    z = np.load(GOLD)
    n = len(z["o0"])
    soup = _dev(z["v0"], z["o0"], z["s0"], z["h0"])
    st = DeviceAdamState.zeros(n)
    lrs = dict(zip(OP.GROUPS, z["lrs"]))
    for k in range(5):
        adam_step(soup, _grads(n, z[f"gv{k}"], z[f"go{k}"], z[f"gs{k}"], z[f"gh{k}"]), st, lrs)
        # fp32 parameters / moments vs the reference's fp64: relative 1e-6 of the step scale
        for got, name in ((soup.vertices, "v"), (soup.opacity, "o"), (soup.sigma, "s"), (soup.sh, "h")):
            want = z[f"{name}{k + 1}"]
            err = np.abs(_np(got) - want).max()
            assert err <= 2e-6 * max(1.0, np.abs(want).max()), (k, name, err)
    assert st.t == 5


def test_reference_adam_cases():
    from paper_2505_19175_b200.optim import DeviceAdamState, adam_step
    rng = np.random.default_rng(0)
    n = 2
    base = (rng.normal(0, 1, (n, 3, 3)), np.array([0.5, 0.6]), np.array([1.0, 2.0]), rng.normal(0, 0.3, (n, 16, 3)))
    unit = lambda lr=1.0: {k: lr for k in OP.GROUPS}  # noqa: E731
    zeros = lambda: _grads(n, np.zeros((n, 3, 3)), np.zeros(n), np.zeros(n), np.zeros((n, 16, 3)))  # noqa: E731
    # zero gradient keeps the parameters
    soup = _dev(*base)
    v0 = soup.vertices.clone()
    st = DeviceAdamState.zeros(n)
    adam_step(soup, zeros(), st, unit())
    assert st.t == 1 and torch.equal(v0, soup.vertices)
    # first step with g = 1 moves by about -lr
    soup = _dev(*base)
    g = zeros()
    g.d_sigma[0] = 1.0
    adam_step(soup, g, DeviceAdamState.zeros(n), unit(0.001))
    assert 1.0 - soup.sigma[0].item() == pytest.approx(0.001, abs=1e-7)  # (fp32 parameter: ulp 6e-8)
    # clamps
    soup, st = _dev(*base), DeviceAdamState.zeros(n)
    g = zeros()
    g.d_opacity[:] = -1.0
    g.d_sigma[:] = 1.0
    for _ in range(200):
        adam_step(soup, g, st, unit(0.5))
    assert np.allclose(_np(soup.opacity), 1.0 - 1e-4) and np.allclose(_np(soup.sigma), 1e-3)
    # per-group rates
    soup = _dev(*base)
    v0, h0 = soup.vertices.clone(), soup.sh.clone()
    g = zeros()
    g.d_vertices[:] = 1.0
    g.d_sh[:] = 1.0
    lrs = unit(0.0)
    lrs["vertices"] = 0.002
    adam_step(soup, g, DeviceAdamState.zeros(n), lrs)
    assert np.allclose(_np(v0 - soup.vertices), 0.002, rtol=0, atol=3e-7)  # (fp32 parameters)
    assert torch.equal(h0, soup.sh)
    # non-finite gradient: raises naming the triangle, nothing changes
    soup, st = _dev(*base), DeviceAdamState.zeros(n)
    v0 = soup.vertices.clone()
    g = _grads(n, np.ones((n, 3, 3)), np.zeros(n), np.zeros(n), np.zeros((n, 16, 3)))
    g.d_sh[1, 0, 0] = float("nan")
    with pytest.raises(ValueError, match="triangle 1"):
        adam_step(soup, g, st, unit())
    assert st.t == 0 and torch.equal(v0, soup.vertices) and float(st.m.abs().max()) == 0.0


def test_unchecked_step_skips_and_keeps_the_step_count():
    """check=False (no host read of the flags): a non-finite gradient skips the
    whole update on the device, the step count included (t must not
    drift from the reference, which raises without touching the state)."""
    from paper_2505_19175_b200.optim import DeviceAdamState, adam_step
    n = 4
    rng = np.random.default_rng(1)
    base = (rng.normal(0, 1, (n, 3, 3)), np.full(n, 0.5), np.full(n, 1.0), rng.normal(0, 0.3, (n, 16, 3)))
    unit = lambda: {k: 1e-3 for k in OP.GROUPS}  # noqa: E731
    soup, st = _dev(*base), DeviceAdamState.zeros(n)
    v0 = soup.vertices.clone()
    g = _grads(n, np.ones((n, 3, 3)), np.zeros(n), np.zeros(n), np.zeros((n, 16, 3)))
    g.d_opacity[2] = float("inf")  # (first non-finite group: opacity)
    adam_step(soup, g, st, unit(), check=False)
    assert st.t == 0 and torch.equal(v0, soup.vertices)
    assert st.last_bad.cpu().tolist() == [-1, 2, -1, -1]
    g.d_opacity[2] = 0.0
    adam_step(soup, g, st, unit(), check=False)
    adam_step(soup, g, st, unit(), check=False)
    assert st.t == 2 and not torch.equal(v0, soup.vertices)


def test_quad_path_equals_element_path():
    """n % 4 == 0 takes the 16-byte (four elements per thread) kernels: every
    element's update is bit-identical to the element-per-thread kernels' (n + 1
    triangles), and the first non-finite triangle of each group is the same."""
    from paper_2505_19175_b200.optim import DeviceAdamState, adam_step
    rng = np.random.default_rng(7)
    n = 1000
    base = (rng.normal(0, 1, (n + 1, 3, 3)), rng.uniform(0.1, 0.9, n + 1), rng.uniform(0.5, 3, n + 1),
            rng.normal(0, 0.3, (n + 1, 16, 3)))
    gr = (rng.normal(0, 1, (n + 1, 3, 3)), rng.normal(0, 1, n + 1), rng.normal(0, 1, n + 1),
          rng.normal(0, 1, (n + 1, 16, 3)))
    lrs = {k: 1e-3 * (i + 1) for i, k in enumerate(OP.GROUPS)}
    a, sa = _dev(*(x[:n] for x in base)), DeviceAdamState.zeros(n)
    b, sb = _dev(*base), DeviceAdamState.zeros(n + 1)
    for _ in range(3):
        adam_step(a, _grads(n, *(x[:n] for x in gr)), sa, lrs)
        adam_step(b, _grads(n + 1, *gr), sb, lrs)
    for ta, tb in ((a.vertices, b.vertices), (a.opacity, b.opacity), (a.sigma, b.sigma), (a.sh, b.sh)):
        assert torch.equal(ta, tb[:n])
    g = _grads(n, *(x[:n] for x in gr))
    g.d_sh[517, 3, 1] = float("nan")
    g.d_sh[516, 15, 2] = float("inf")   # (same quad region, smaller triangle)
    g.d_vertices[999, 2, 2] = float("-inf")
    adam_step(a, g, sa, lrs, check=False)
    assert sa.last_bad.cpu().tolist() == [999, -1, -1, 516]
