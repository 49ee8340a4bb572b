"""The reference's closed-form gradient tests (tests/test_backward.py:21-67 of
the reference package) through the drop-in ``render_backward`` on the GPU:
zero upstream -> zero gradients, dC/do = I(p) * colour for one triangle over
black, linearity in the upstream gradient, and exactly zero gradients for a
triangle that never passes the contribution threshold."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

PRECISIONS = ["fast", "exact"]


def _T():
    from paper_2505_19175_b200 import types as T
    return T


def _ident():
    return _T().CameraPose(rotation=np.eye(3), translation=np.zeros(3))


def _cam():
    return _T().CameraIntrinsics(fx=12.0, fy=12.0, cx=6.0, cy=6.0, width=12, height=12)


def _tri(v, opacity=0.5, sigma=1.0):
    return _T().Triangle3D(vertices=np.asarray(v, float), opacity=opacity, sigma=sigma, sh=np.zeros((16, 3)))


def _random_soup(seed, n):
    from paper_2505_19175_b200 import scenes
    T = _T()
    rng = np.random.default_rng(seed)
    v = rng.uniform(-0.8, 0.8, (n, 3, 3)) * np.array([1.0, 1.0, 0.4])
    soup = T.TriangleSoup(vertices=v, opacity=rng.uniform(0.1, 0.9, n), sigma=rng.uniform(0.5, 5.0, n),
                          sh=rng.normal(0, 0.3, (n, 16, 3)))
    intr = T.CameraIntrinsics(fx=41.6, fy=33.6, cx=16.0, cy=12.0, width=32, height=24)
    return soup, intr, scenes.look_at(np.array([0.1, -0.2, -2.8]), np.zeros(3))


def _window(v, intr, p, sigma):
    # normalized window I(p) = (phi(p) / phi(s))^sigma inside (geometry.py window_value)
    q = np.array([[intr.fx * a[0] / a[2] + intr.cx, intr.fy * a[1] / a[2] + intr.cy] for a in v])
    cen = q.mean(axis=0)
    phi, lens = [], []
    for e in range(3):
        a, b = q[e], q[(e + 1) % 3]
        d = b - a
        ln = np.hypot(d[0], d[1])
        n = np.array([d[1], -d[0]]) / ln
        off = -(n @ a)
        if n @ cen + off > 0:
            n, off = -n, -off
        phi.append((n, off))
        lens.append(ln)
    f = lambda x: max(n @ x + o for n, o in phi)  # noqa: E731
    a_, b_, c_ = (np.linalg.norm(q[1] - q[2]), np.linalg.norm(q[2] - q[0]), np.linalg.norm(q[0] - q[1]))
    s = (a_ * q[0] + b_ * q[1] + c_ * q[2]) / (a_ + b_ + c_)
    return min(f(np.asarray(p)) / f(s), 1.0) ** sigma


@pytest.mark.parametrize("precision", PRECISIONS)
def test_zero_upstream_gives_zero_gradients(precision):
    from paper_2505_19175_b200 import render_backward
    soup, intr, pose = _random_soup(1, 3)
    g = render_backward(soup, intr, pose, d_image=np.zeros((intr.height, intr.width, 3)), precision=precision)
    for k in ("d_vertices", "d_opacity", "d_sigma", "d_sh"):
        assert np.allclose(getattr(g, k), 0), k


@pytest.mark.parametrize("precision", PRECISIONS)
def test_opacity_gradient_closed_form(precision):
    from paper_2505_19175_b200 import render_backward
    intr = _cam()
    v = [[-0.5, -0.5, 1], [0.5, -0.5, 1], [0, 0.5, 1]]
    d_image = np.zeros((12, 12, 3))
    d_image[6, 6, 0] = 1.0
    g = render_backward([_tri(v, 0.5, 2.0)], intr, _ident(), d_image=d_image, precision=precision)
    assert g.d_opacity[0] == pytest.approx(_window(np.array(v, float), intr, (6.5, 6.5), 2.0) * 0.5, rel=1e-6)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_linearity_in_upstream_gradient(precision):
    from paper_2505_19175_b200 import render_backward
    soup, intr, pose = _random_soup(2, 4)
    rng = np.random.default_rng(5)
    da = rng.normal(size=(intr.height, intr.width, 3))
    db = rng.normal(size=(intr.height, intr.width, 3))
    ga = render_backward(soup, intr, pose, d_image=da, precision=precision)
    gb = render_backward(soup, intr, pose, d_image=db, precision=precision)
    gs = render_backward(soup, intr, pose, d_image=da + db, precision=precision)
    for k in ("d_vertices", "d_opacity", "d_sigma", "d_sh"):
        a, b, s = getattr(ga, k), getattr(gb, k), getattr(gs, k)
        assert np.allclose(s, a + b, rtol=1e-5, atol=1e-6 * max(1.0, np.abs(s).max())), k


@pytest.mark.parametrize("precision", PRECISIONS)
def test_zero_support_triangle_gets_zero_gradient(precision):
    from paper_2505_19175_b200 import render_backward
    intr = _cam()
    visible = _tri([[-0.5, -0.5, 1], [0.5, -0.5, 1], [0, 0.5, 1]], 0.6, 1.0)
    faint = _tri([[-0.3, -0.3, 1.5], [0.3, -0.3, 1.5], [0, 0.3, 1.5]], 1.0 / 300.0, 1.0)
    g = render_backward([visible, faint], intr, _ident(), d_image=np.ones((12, 12, 3)), precision=precision)
    assert np.allclose(g.d_vertices[1], 0) and g.d_opacity[1] == 0.0
    assert not np.allclose(g.d_vertices[0], 0)
