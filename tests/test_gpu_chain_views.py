"""Deferred multi-view chain (ts_backward_screen / ts_chain_views): the
summed parameter gradients of several views chained in one pass equal the
per-view backward accumulated view by view (the batch gradient of SURVEY 8e,
test_backward.py:44-55 linearity), chunked and unchunked alike, and the
entry points reject what they cannot defer."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import rel_err  # noqa: E402


def _scene(n=3000, views=5, w=96, h=80):
    from paper_2505_19175_b200 import DeviceSoup, scenes
    soup = DeviceSoup.from_soup(scenes.make_soup(n, seed=31, size=0.15, sigma=(0.5, 3.0)), dtype=torch.float32)
    intr, _ = scenes.frontal_camera(w, h, 110.0)
    poses = scenes.orbit_cameras(views, seed=4)
    gen = torch.Generator("cuda").manual_seed(5)
    d_imgs = [torch.randn((h, w, 3), device="cuda", generator=gen) for _ in poses]
    return soup, intr, poses, d_imgs


def _sequential(r, soup, intr, poses, d_imgs, base=None):
    from paper_2505_19175_b200 import DeviceGrads
    g = DeviceGrads(base.flat.clone(), base.n) if base is not None else DeviceGrads.zeros(len(soup))
    for k, (p, d) in enumerate(zip(poses, d_imgs)):
        r.forward(soup, intr, p, keep_backward=True)
        r.backward(d, g, accumulate=base is not None or k > 0)
    return g


def _deferred(r, soup, intr, poses, d_imgs, base=None, chunks=None):
    from paper_2505_19175_b200 import DeviceGrads
    g = DeviceGrads(base.flat.clone(), base.n) if base is not None else DeviceGrads.zeros(len(soup))
    for k, (p, d) in enumerate(zip(poses, d_imgs)):
        r.forward(soup, intr, p, keep_backward=True)
        assert r.backward_screen(d) == k + 1
    r.chain_views(g, accumulate=base is not None, chunks=chunks)
    assert r.pending_views() == 0
    return g


def _close(got, want, tol=2e-5):
    # view by view, each view's contribution is rounded to fp32 before it is
    # added; deferred, the vertex / opacity / sigma terms of the views are summed
    # in fp64 and rounded once: a few fp32 ulps of the partial sums apart
    n = got.n
    a = got.flat.double().cpu().numpy()
    b = want.flat.double().cpu().numpy()
    for lo, hi in [(0, 9 * n), (9 * n, 10 * n), (10 * n, 11 * n), (11 * n, 59 * n)]:
        assert rel_err(a[lo:hi], b[lo:hi]) < tol, (lo, hi, rel_err(a[lo:hi], b[lo:hi]))


@pytest.mark.parametrize("views", [1, 5, 8])
def test_chain_views_equals_sequential_backward(views):
    from paper_2505_19175_b200 import Rasterizer
    r = Rasterizer()
    soup, intr, poses, d_imgs = _scene(views=views)
    want = _sequential(r, soup, intr, poses, d_imgs)
    got = _deferred(r, soup, intr, poses, d_imgs)
    _close(got, want)
    # accumulating into a non-zero buffer
    base = want
    _close(_deferred(r, soup, intr, poses, d_imgs, base=base), _sequential(r, soup, intr, poses, d_imgs, base=base))


def test_chain_views_chunked_is_identical():
    from paper_2505_19175_b200 import Rasterizer
    from paper_2505_19175_b200.parallel import chunk_bounds
    r = Rasterizer()
    soup, intr, poses, d_imgs = _scene(views=3)
    whole = _deferred(r, soup, intr, poses, d_imgs)
    bounds = chunk_bounds(len(soup), 5)
    events = [torch.cuda.Event() for _ in range(5)]
    parts = _deferred(r, soup, intr, poses, d_imgs, chunks=(bounds, events))
    torch.cuda.synchronize()
    assert all(e.query() for e in events)
    assert torch.equal(whole.flat, parts.flat)


def test_chain_views_at_c3_scale():
    """Two C3 views (2M triangles, 1297x840): deferred == sequential."""
    from paper_2505_19175_b200 import DeviceSoup, Rasterizer, scenes
    c3 = scenes.CONFIGS["c3"]
    soup = DeviceSoup.from_soup(scenes.make_soup(c3.n, c3.seed, c3.size, c3.sigma), dtype=torch.float32)
    intr, _ = scenes.frontal_camera(c3.width, c3.height, c3.f)
    poses = scenes.orbit_cameras(2, seed=4)
    gen = torch.Generator("cuda").manual_seed(103)
    d_imgs = [torch.randn((c3.height, c3.width, 3), device="cuda", generator=gen) for _ in poses]
    r = Rasterizer()
    want = _sequential(r, soup, intr, poses, d_imgs)
    got = _deferred(r, soup, intr, poses, d_imgs)
    _close(got, want)


def test_chain_views_errors():
    from paper_2505_19175_b200 import DeviceGrads, DeviceSoup, Rasterizer, scenes
    r = Rasterizer()
    soup, intr, poses, d_imgs = _scene(views=1)
    g = DeviceGrads.zeros(len(soup))
    with pytest.raises(RuntimeError):
        r.chain_views(g)                      # nothing pending
    r.forward(soup, intr, poses[0], keep_backward=True)
    for k in range(Rasterizer.MAX_PENDING_VIEWS):
        r.backward_screen(d_imgs[0])
    with pytest.raises(RuntimeError):
        r.backward_screen(d_imgs[0])          # slots full
    r.chain_views(g)
    assert r.pending_views() == 0
    # a different soup cannot join pending views
    other = DeviceSoup.from_soup(scenes.make_soup(len(soup), seed=32, size=0.15, sigma=(0.5, 3.0)),
                                 dtype=torch.float32)
    r.forward(soup, intr, poses[0], keep_backward=True)
    r.backward_screen(d_imgs[0])
    r.forward(other, intr, poses[0], keep_backward=True)
    with pytest.raises(RuntimeError):
        r.backward_screen(d_imgs[0])
    r.chain_views(g)
    # exact precision is not deferred
    r.forward(soup, intr, poses[0], keep_backward=True, precision="exact")
    with pytest.raises(RuntimeError):
        r.backward_screen(d_imgs[0])
    with pytest.raises(ValueError):
        r.backward_screen(d_imgs[0][:10])
    # four pending copies of one view: the deferred sum is 4x that view's gradient
    r.forward(soup, intr, poses[0], keep_backward=True)
    one = r.backward(d_imgs[0])
    r.forward(soup, intr, poses[0], keep_backward=True)
    for _ in range(4):
        r.backward_screen(d_imgs[0])
    four = DeviceGrads.zeros(len(soup))
    r.chain_views(four)
    np.testing.assert_allclose(four.flat.double().cpu().numpy(), 4 * one.flat.double().cpu().numpy(),
                               rtol=2e-6, atol=1e-6 * float(one.flat.abs().max()))
