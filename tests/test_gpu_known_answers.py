"""The reference's closed-form render tests (tests/test_render.py:83-118,
204-222 of the reference package) through the drop-in ``render`` on the GPU:
empty scene, a single near-opaque triangle, two-layer compositing, the area of
a culled triangle, a solid soup, and conservation (sum of fragment weights +
final transmittance = 1), each in both precisions; images also equal the
reference's own outputs (tests/golden/kat.npz) to 1e-5."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
C0 = 0.28209479177387814
PRECISIONS = ["fast", "exact"]


def _t():
    from paper_2505_19175_b200 import types as T
    return T


def _ident():
    T = _t()
    return T.CameraPose(rotation=np.eye(3), translation=np.zeros(3))


def _red_sh():
    sh = np.zeros((16, 3))
    sh[0, 0] = 1.0
    return sh


def _incenter_pixel(v, intr):
    q = np.array([[intr.fx * p[0] / p[2] + intr.cx, intr.fy * p[1] / p[2] + intr.cy] for p in v])
    a, b, c = (np.linalg.norm(q[1] - q[2]), np.linalg.norm(q[2] - q[0]), np.linalg.norm(q[0] - q[1]))
    s = (a * q[0] + b * q[1] + c * q[2]) / (a + b + c)
    return int(s[0]), int(s[1])


@pytest.mark.parametrize("precision", PRECISIONS)
def test_empty_scene_is_background(precision):
    from paper_2505_19175_b200 import render
    T = _t()
    intr = T.CameraIntrinsics(fx=10, fy=10, cx=8, cy=8, width=16, height=16)
    out = render(T.TriangleSoup.empty(), intr, _ident(), background=(0.2, 0.3, 0.4), precision=precision)
    assert np.allclose(out.image.rgb, [0.2, 0.3, 0.4]) and np.allclose(out.alpha_map, 0.0)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_single_opaque_triangle(precision):
    from paper_2505_19175_b200 import render
    T = _t()
    intr = T.CameraIntrinsics(fx=20, fy=20, cx=8, cy=8, width=16, height=16)
    v = [[-0.4, -0.4, 1], [0.4, -0.4, 1], [0, 0.4, 1]]
    tri = T.Triangle3D(vertices=v, opacity=0.99, sigma=1e-3, sh=_red_sh())
    out = render([tri], intr, _ident(), precision=precision)
    x, y = _incenter_pixel(np.array(v, float), intr)
    px = out.image.rgb[y, x]
    assert px[0] == pytest.approx(0.99 * 0.78209479, abs=1e-3)
    assert px[1] == pytest.approx(0.99 * 0.5, abs=1e-3)
    ref = np.load(os.path.join(GOLDEN, "kat.npz"))["opaque_image"]
    assert np.abs(out.image.rgb - ref).max() <= 1e-5


@pytest.mark.parametrize("precision", PRECISIONS)
def test_two_layer_compositing(precision):
    from paper_2505_19175_b200 import render
    T = _t()
    intr = T.CameraIntrinsics(fx=4, fy=4, cx=8, cy=8, width=16, height=16)
    sh1, sh2 = np.zeros((16, 3)), np.zeros((16, 3))
    sh1[0] = (np.array([0.9, 0.1, 0.1]) - 0.5) / C0
    sh2[0] = (np.array([0.1, 0.9, 0.1]) - 0.5) / C0
    big = np.array([[-8, -8, 0], [8, -8, 0], [0, 12, 0]], float)
    front = T.Triangle3D(vertices=big + [0, 0, 1], opacity=0.5, sigma=1e-5, sh=sh1)
    back = T.Triangle3D(vertices=big * 2 + [0, 0, 2], opacity=0.5, sigma=1e-5, sh=sh2)
    bg = np.array([0.0, 0.0, 1.0])
    out = render([front, back], intr, _ident(), background=bg, precision=precision)
    expect = 0.5 * np.array([0.9, 0.1, 0.1]) + 0.25 * np.array([0.1, 0.9, 0.1]) + 0.25 * bg
    assert np.allclose(out.image.rgb[8, 8], expect, atol=1e-3)
    ref = np.load(os.path.join(GOLDEN, "kat.npz"))["two_layer_image"]
    assert np.abs(out.image.rgb - ref).max() <= 1e-5


@pytest.mark.parametrize("precision", PRECISIONS)
def test_area_zero_for_culled(precision):
    from paper_2505_19175_b200 import render
    T = _t()
    intr = T.CameraIntrinsics(fx=10, fy=10, cx=8, cy=8, width=16, height=16)
    sh = np.zeros((16, 3))
    visible = T.Triangle3D(vertices=[[-0.3, -0.3, 1], [0.3, -0.3, 1], [0, 0.3, 1]], opacity=0.5, sigma=1.0, sh=sh)
    behind = T.Triangle3D(vertices=[[0, 0, -2], [1, 0, -2], [0, 1, -2]], opacity=0.5, sigma=1.0, sh=sh)
    out = render([visible, behind], intr, _ident(), precision=precision)
    assert out.per_triangle_area[0] > 0 and out.per_triangle_area[1] == 0.0


@pytest.mark.parametrize("precision", PRECISIONS)
def test_solid_soup_ignores_opacity(precision):
    from paper_2505_19175_b200 import render
    T = _t()
    intr = T.CameraIntrinsics(fx=20, fy=20, cx=8, cy=8, width=16, height=16)
    v = [[-0.4, -0.4, 1], [0.4, -0.4, 1], [0, 0.4, 1]]
    soup = T.TriangleSoup.from_triangles([T.Triangle3D(vertices=v, opacity=0.5, sigma=0.05, sh=_red_sh())])
    soup.solid = True
    out = render(soup, intr, _ident(), precision=precision)
    x, y = _incenter_pixel(np.array(v, float), intr)
    assert out.alpha_map[y, x] == pytest.approx(0.99, abs=1e-2)


def test_weights_and_transmittance_conserve():
    # fragment collection runs on the fast path (fp64 weights per fragment)
    from paper_2505_19175_b200 import render, scenes
    soup, intr, pose = scenes.make_scene("c1")
    out = render(soup, intr, pose, collect_fragments=True)
    f = out.fragments
    cs = np.concatenate([[0.0], np.cumsum(f.weight)])
    wsum = cs[f.offsets[1:]] - cs[f.offsets[:-1]]
    assert len(f.weight) > 10000
    assert np.allclose(wsum, out.alpha_map.reshape(-1), atol=1e-6)
