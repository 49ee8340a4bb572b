"""The CPU oracle (oracle/trisplat_oracle.c) pinned against the reference.

Golden fixtures were produced by the live reference package
(tests/golden/make_golden.py).  The restatement must reproduce every
discrete output bit-for-bit (sort order, tile lists, fragment lists, last
contributors, pixel counts) and the floating-point ones to ~1 ulp.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN, digest, rel_err
from oracle import oracle as O
from paper_2505_19175_b200 import scenes
from paper_2505_19175_b200.types import (CameraIntrinsics, CameraPose, TriangleSoup,
                                         Triangle3D, WindowMode)

IDENTITY = CameraPose(rotation=np.eye(3), translation=np.zeros(3))


def test_golden_small_scene(golden_scene):
    g = golden_scene
    out = O.render(g.soup, g.intr, g.pose, mode=g.mode, background=g.background,
                   collect_fragments=True)
    assert np.array_equal(out.proj.sorted_idx, g["sorted_idx"])
    assert np.array_equal(out.proj.z, g["z"])
    assert np.array_equal(out.proj.bbox, g["bbox"])
    assert np.array_equal(out.tile_start, g["tile_start"])
    assert np.array_equal(out.entry_tri, g["entry_tri"])
    assert np.abs(out.image - g["image"]).max() <= 1e-14
    assert np.array_equal(out.alpha_map, g["alpha_map"])
    assert np.array_equal(out.per_triangle_max_weight, g["maxw"])
    assert np.array_equal(out.per_triangle_pixel_count, g["pixcount"])
    assert np.array_equal(out.per_triangle_area, g["area"])
    assert np.array_equal(out.fragments.offsets, g["frag_offsets"])
    assert np.array_equal(out.fragments.triangle, g["frag_triangle"])
    assert np.array_equal(out.fragments.weight, g["frag_weight"])
    assert np.array_equal(out.fragments.depth, g["frag_depth"])
    assert np.array_equal(out.last_src, g["last_src"])
    assert np.array_equal(out.nfrag, g["nfrag"])
    gr = O.render_backward(g.soup, g.intr, g.pose, mode=g.mode, background=g.background,
                           d_image=g.d_image)
    for k in ("d_vertices", "d_opacity", "d_sigma", "d_sh"):
        assert rel_err(getattr(gr, k), g[k], floor=1e-9) < 1e-9, k


def test_golden_c1():
    z = np.load(os.path.join(GOLDEN, "c1.npz"))
    cfg = scenes.CONFIGS["c1"]
    soup, intr, pose = scenes.make_scene(cfg)
    assert digest(soup.vertices, soup.opacity, soup.sigma, soup.sh) == str(z["input_digest"])
    out = O.render(soup, intr, pose, collect_fragments=True)
    assert np.array_equal(out.proj.sorted_idx, z["sorted_idx"])
    assert np.array_equal(out.tile_start, z["tile_start"])
    assert np.array_equal(out.entry_tri, z["entry_tri"])
    assert np.abs(out.image - z["image"]).max() <= 1e-14
    assert np.array_equal(out.alpha_map, z["alpha_map"])
    assert np.array_equal(out.last_src, z["last_src"])
    assert np.array_equal(out.nfrag, z["nfrag"])
    assert np.array_equal(out.per_triangle_pixel_count, z["pixcount"])
    assert np.array_equal(out.per_triangle_max_weight, z["maxw"])
    assert digest(out.fragments.offsets, out.fragments.triangle) == str(z["frag_digest"])
    d_image = scenes.make_d_image(cfg.seed, cfg.height, cfg.width)
    gr = O.render_backward(soup, intr, pose, d_image=d_image)
    keep = len(z["d_opacity"])
    for k in ("d_vertices", "d_opacity", "d_sigma", "d_sh"):
        assert rel_err(getattr(gr, k)[:keep], z[k], floor=1e-9) < 1e-9, k
    sums = [getattr(gr, k).sum() for k in ("d_vertices", "d_opacity", "d_sigma", "d_sh")]
    assert np.allclose(sums, z["grad_sum"], rtol=1e-9, atol=1e-12)


def test_known_answers():
    """test_render.py:235-262 closed forms, and the reference's own values."""
    z = np.load(os.path.join(GOLDEN, "kat.npz"))
    intr = CameraIntrinsics(fx=20, fy=20, cx=8, cy=8, width=16, height=16)
    sh = np.zeros((16, 3)); sh[0, 0] = 1.0
    tri = Triangle3D(vertices=[[-0.4, -0.4, 1], [0.4, -0.4, 1], [0, 0.4, 1]], opacity=0.99,
                     sigma=1e-3, sh=sh)
    out = O.render(TriangleSoup.from_triangles([tri]), intr, IDENTITY)
    assert np.array_equal(out.image, z["opaque_image"])
    intr2 = CameraIntrinsics(fx=4, fy=4, cx=8, cy=8, width=16, height=16)
    sh1 = np.zeros((16, 3)); sh2 = np.zeros((16, 3))
    sh1[0] = (np.array([0.9, 0.1, 0.1]) - 0.5) / 0.28209479177387814
    sh2[0] = (np.array([0.1, 0.9, 0.1]) - 0.5) / 0.28209479177387814
    big = np.array([[-8, -8, 0], [8, -8, 0], [0, 12, 0]], float)
    soup = TriangleSoup.from_triangles([
        Triangle3D(vertices=big + [0, 0, 1], opacity=0.5, sigma=1e-5, sh=sh1),
        Triangle3D(vertices=big * 2 + [0, 0, 2], opacity=0.5, sigma=1e-5, sh=sh2)])
    out2 = O.render(soup, intr2, IDENTITY, background=(0.0, 0.0, 1.0))
    assert np.array_equal(out2.image, z["two_layer_image"])
    expect = 0.5 * np.array([0.9, 0.1, 0.1]) + 0.25 * np.array([0.1, 0.9, 0.1]) \
        + 0.25 * np.array([0.0, 0.0, 1.0])
    assert np.allclose(out2.image[8, 8], expect, atol=1e-3)


def test_empty_scene_is_background():
    intr = CameraIntrinsics(fx=10, fy=10, cx=8, cy=8, width=16, height=16)
    out = O.render(TriangleSoup.empty(), intr, IDENTITY, background=(0.2, 0.3, 0.4))
    assert np.allclose(out.image, [0.2, 0.3, 0.4])
    assert np.allclose(out.alpha_map, 0.0)


def test_non_finite_message_order():
    intr = CameraIntrinsics(fx=10, fy=10, cx=8, cy=8, width=16, height=16)
    soup = TriangleSoup(vertices=np.zeros((3, 3, 3)), opacity=[0.5] * 3, sigma=[1.0] * 3,
                        sh=np.zeros((3, 16, 3)))
    soup.sh[0, 0, 0] = np.nan
    soup.sigma[2] = np.inf
    with pytest.raises(ValueError, match="non-finite sigma in triangle 2"):
        O.render(soup, intr, IDENTITY)


def test_thread_count_invariance():
    soup, intr, pose = scenes.make_scene("c1")
    O.set_threads(1)
    a = O.render(soup, intr, pose)
    O.set_threads(4)
    b = O.render(soup, intr, pose)
    assert np.array_equal(a.image, b.image)
    assert np.array_equal(a.per_triangle_max_weight, b.per_triangle_max_weight)
