"""The rest of the drop-in surface: project_scene / build_tile_lists
shadows and tile sizes other than 16.

* project_scene (render.py:253-312): every SceneProjection field against the
  oracle's restatement (pinned to the live reference by tests/golden), on the
  golden scenes and configs[0] -- integer fields and the depth order exact,
  the fp64 fields bit-exact (the dump follows the reference's operation order
  without contractions);
* build_tile_lists (render.py:315-361) for tile sizes 1..64 against the oracle;
* render / render_backward with tile_size != 16 give the tile-16 outputs (every
  output is independent of the tiling); tile_size 0 raises like the reference.
"""
import os

import numpy as np
import pytest

from conftest import GoldenScene, golden_paths

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FIELDS = ("sorted_idx", "z", "xc", "q", "nrm", "doff", "esign", "phis", "area", "sig", "opa", "rgb",
          "raw_rgb", "basis", "viewdir", "u_norm", "bbox", "area_full")


def _scenes():
    out = [(os.path.basename(p), p) for p in golden_paths()[:6]]
    out.append(("c1", "c1"))
    return out


def _load(p):
    from paper_2505_19175_b200 import scenes
    from paper_2505_19175_b200.types import WindowMode
    if p == "c1":
        soup, intr, pose = scenes.make_scene("c1")
        return soup, intr, pose, WindowMode.NORMALIZED
    g = GoldenScene(p)
    return g.soup, g.intr, g.pose, g.mode


@pytest.mark.parametrize("name,path", _scenes(), ids=[s[0] for s in _scenes()])
def test_project_scene_matches_oracle(name, path):
    from paper_2505_19175_b200 import rasterizer as tsb
    from oracle import oracle as O
    soup, intr, pose, mode = _load(path)
    got = tsb.project_scene(soup, intr, pose, mode)
    want = O.project_scene(soup, intr, pose, mode)
    assert got.n_total == want.n_total
    for k in FIELDS:
        a, b = np.asarray(getattr(got, k)), np.asarray(getattr(want, k))
        assert a.shape == b.shape, f"{name} {k} shape {a.shape} vs {b.shape}"
        assert np.array_equal(a, b), f"{name} {k}: max |diff| {np.abs(a.astype(float) - b).max()}"


@pytest.mark.parametrize("tile_size", [1, 5, 16, 23, 64])
def test_build_tile_lists_any_tile_size(tile_size):
    from paper_2505_19175_b200 import rasterizer as tsb
    from oracle import oracle as O
    soup, intr, pose, mode = _load("c1")
    proj = O.project_scene(soup, intr, pose, mode)
    got = tsb.build_tile_lists(proj, intr, tile_size)
    want = O.build_tile_lists(proj, intr, tile_size)
    assert got[0] == want[0] and got[1] == want[1]
    assert np.array_equal(got[2], want[2]) and np.array_equal(got[3], want[3])


def test_build_tile_lists_empty():
    from paper_2505_19175_b200 import rasterizer as tsb
    from paper_2505_19175_b200.types import CameraIntrinsics

    class P:
        bbox = np.zeros((0, 4), np.int64)

    intr = CameraIntrinsics(fx=10.0, fy=10.0, cx=8.0, cy=8.0, width=40, height=24)
    ntx, nty, start, entry = tsb.build_tile_lists(P(), intr, 16)
    assert (ntx, nty) == (3, 2) and np.array_equal(start, np.zeros(7, np.int64)) and len(entry) == 0


@pytest.mark.parametrize("tile_size", [8, 32])
def test_render_independent_of_tile_size(tile_size):
    from paper_2505_19175_b200 import rasterizer as tsb
    from paper_2505_19175_b200 import scenes
    soup, intr, pose, mode = _load(golden_paths()[0])
    a = tsb.render(soup, intr, pose, mode)
    b = tsb.render(soup, intr, pose, mode, tile_size=tile_size)
    assert np.array_equal(a.image.rgb, b.image.rgb) and np.array_equal(a.alpha_map, b.alpha_map)
    assert np.array_equal(a.per_triangle_pixel_count, b.per_triangle_pixel_count)
    assert np.array_equal(a.per_triangle_max_weight, b.per_triangle_max_weight)
    d = scenes.make_d_image(5, intr.height, intr.width)
    ga = tsb.render_backward(soup, intr, pose, mode, d_image=d)
    gb = tsb.render_backward(soup, intr, pose, mode, d_image=d, tile_size=tile_size)
    for k in ("d_vertices", "d_opacity", "d_sigma", "d_sh"):
        assert np.array_equal(getattr(ga, k), getattr(gb, k)), k


def test_tile_size_zero_raises_like_reference():
    from paper_2505_19175_b200 import rasterizer as tsb
    soup, intr, pose, mode = _load(golden_paths()[0])
    with pytest.raises(ZeroDivisionError):
        tsb.render(soup, intr, pose, mode, tile_size=0)
    with pytest.raises(ValueError):
        tsb.render(soup, intr, pose, mode, tile_size=-16)


def test_render_outputs_are_independent_across_calls():
    """render() returns arrays in pooled page-locked buffers: a buffer is reused
    only after every array of an earlier call is gone, so holding the outputs of
    one call while rendering another never changes them."""
    import gc
    from paper_2505_19175_b200 import rasterizer as tsb
    soup, intr, pose, mode = _load(golden_paths()[0])
    a = tsb.render(soup, intr, pose, mode, background=(0.1, 0.2, 0.3))
    img_a, maxw_a, pix_a = a.image.rgb.copy(), a.per_triangle_max_weight.copy(), a.per_triangle_pixel_count.copy()
    assert np.isfinite(img_a).all() and img_a.min() >= 0.0 and img_a.max() <= 1.0  # (ImageBuffer.trusted)
    b = tsb.render(soup, intr, pose, mode, background=(0.9, 0.8, 0.7))
    assert np.array_equal(a.image.rgb, img_a) and np.array_equal(a.per_triangle_max_weight, maxw_a)
    assert np.array_equal(a.per_triangle_pixel_count, pix_a)
    assert not np.array_equal(a.image.rgb, b.image.rgb)
    del a, b
    gc.collect()
    c = tsb.render(soup, intr, pose, mode, background=(0.1, 0.2, 0.3))
    assert np.array_equal(c.image.rgb, img_a)


@pytest.mark.parametrize("perturb", [False, True])
def test_render_upload_f32_exact_or_f64(perturb):
    """render() with the reference's fp64 soup: a soup of fp32 values crosses PCIe
    as fp32 (ts_pack_f32), one value that is not an fp32 value sends the whole soup
    as fp64; both render the oracle's frame (discrete outputs exact, RGB 1e-5)."""
    from oracle import oracle as O
    from paper_2505_19175_b200 import rasterizer as R
    from paper_2505_19175_b200 import scenes
    from paper_2505_19175_b200.types import TriangleSoup
    soup, intr, pose = scenes.make_scene("c1")
    if perturb:
        sh = np.array(soup.sh, dtype=np.float64)
        sh[len(sh) // 2, 0, 0] += 1e-13
        soup = TriangleSoup(np.asarray(soup.vertices), np.asarray(soup.opacity), np.asarray(soup.sigma), sh)
    out = R.render(soup, intr, pose)
    assert R.LAST_RENDER_TIMES["upload"] == ("f64" if perturb else "f32")
    n = len(soup.vertices)
    assert R.LAST_RENDER_TIMES["upload_bytes"] == (8 if perturb else 4) * 59 * n
    ref = O.render(soup, intr, pose)
    np.testing.assert_array_equal(out.per_triangle_pixel_count, ref.per_triangle_pixel_count)
    np.testing.assert_allclose(out.image.rgb, getattr(ref.image, "rgb", ref.image), atol=1e-5, rtol=0)
    np.testing.assert_allclose(out.alpha_map, ref.alpha_map, atol=1e-5, rtol=0)
    np.testing.assert_allclose(out.per_triangle_max_weight, ref.per_triangle_max_weight, atol=1e-6, rtol=0)
    np.testing.assert_allclose(out.per_triangle_area, ref.per_triangle_area, rtol=1e-6, atol=0)


@pytest.mark.parametrize("n", [1, 1000, 5_000_003])
def test_upload_f32(n):
    """ts_upload_f32 (the lossless upload of render()): fp32 values arrive bit for
    bit; one value that is not an fp32 value -> 0 and no tensor."""
    from paper_2505_19175_b200 import rasterizer as R
    a = np.random.default_rng(n).normal(size=n).astype(np.float32).astype(np.float64)
    t = R._staged_h2d_f32(a)
    assert t is not None and t.dtype == torch.float32
    np.testing.assert_array_equal(t.cpu().numpy(), a.astype(np.float32))
    b = a.copy()
    b[-1] += 1e-9
    assert R._staged_h2d_f32(b) is None
    t2 = R._staged_h2d_f32(a)  # the ring is reusable after a failed upload
    np.testing.assert_array_equal(t2.cpu().numpy(), a.astype(np.float32))
