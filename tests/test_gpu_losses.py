"""GPU parity of the on-device photometric loss (ts_loss.cu) against the
oracle (on the same fp32-rounded images) and the live reference's fixtures."""
import os

import numpy as np
import pytest

from oracle import losses as OL

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "loss.npz")


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def _check(x, y, lam, label):
    from paper_2505_19175_b200 import losses as DL
    xr, yr = f32(x), f32(y)
    want_l, want_g = OL.photometric_loss(xr, yr, lam)
    got_l, got_g = DL.photometric_loss(xr, yr, lam)
    assert abs(got_l - want_l) <= 1e-9 + 1e-6 * abs(want_l), f"{label} loss {got_l} vs {want_l}"
    scale = max(np.abs(want_g).max(), 1e-9)  # (identical images: gradient ~0)
    err = np.abs(got_g - want_g).max() / scale
    assert err <= 1e-5, f"{label} grad rel err {err}"
    if xr.shape[0] >= 11 and xr.shape[1] >= 11:
        assert abs(DL.ssim(xr, yr) - OL.ssim(xr, yr)) <= 1e-6, label


def test_against_reference_fixtures():
    from paper_2505_19175_b200 import losses as DL
    z = np.load(GOLD)
    for k in range(int(z["n"])):
        x, y, lam = z[f"x{k}"], z[f"y{k}"], float(z[f"lam{k}"])
        _check(x, y, lam, f"golden{k}")
        # fp32 inputs vs the reference's fp64 inputs: a few 1e-8
        got_l, _ = DL.photometric_loss(x, y, lam)
        assert abs(got_l - float(z[f"loss{k}"])) <= 1e-6, k


@pytest.mark.parametrize("shape", [(16, 16), (17, 33), (90, 70), (840, 1297)])
@pytest.mark.parametrize("lam", [0.0, 0.2, 1.0])
def test_random_images(shape, lam):
    rng = np.random.default_rng(shape[0] * 7 + int(lam * 10))
    x = rng.uniform(0, 1, shape + (3,))
    y = np.clip(x + rng.normal(0, 0.2, x.shape), 0, 1)
    _check(x, y, lam, f"{shape} lam {lam}")


def test_reference_cases_and_device_tensors():
    from paper_2505_19175_b200 import losses as DL
    x = f32(np.random.default_rng(3).uniform(0, 1, (16, 16, 3)))
    assert DL.photometric_loss(x, x, 0.2)[0] == pytest.approx(0.0, abs=1e-12)
    assert DL.photometric_loss(np.zeros((16, 16, 3)), np.ones((16, 16, 3)), 0.0)[0] == pytest.approx(1.0)
    assert DL.photometric_loss(np.full((4, 4, 3), 0.3), np.full((4, 4, 3), 0.7), 0.5)[0] == pytest.approx(0.2,
                                                                                                          abs=1e-7)
    assert DL.ssim(x, x) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        DL.ssim(np.zeros((16, 16, 3)), np.zeros((17, 16, 3)))
    with pytest.raises(ValueError):
        DL.photometric_loss(np.zeros((16, 16, 3)), np.zeros((17, 16, 3)), 0.2)
    # CUDA tensors in, CUDA gradient out (no host round trip)
    xt = torch.rand((64, 48, 3), device="cuda")
    yt = torch.rand((64, 48, 3), device="cuda")
    loss, g = DL.photometric_loss(xt, yt, 0.2)
    assert g.is_cuda and g.dtype == torch.float32 and g.shape == xt.shape
    wl, wg = OL.photometric_loss(xt.double().cpu().numpy(), yt.double().cpu().numpy(), 0.2)
    assert abs(loss - wl) <= 1e-6 * abs(wl)
    assert np.abs(g.double().cpu().numpy() - wg).max() <= 1e-5 * np.abs(wg).max()


def test_distortion_and_depth_against_fixtures():
    from paper_2505_19175_b200 import losses as DL
    from paper_2505_19175_b200.types import FragmentData
    z = np.load(GOLD)
    h, w = (int(v) for v in z["dist_hw"])
    for tag in "su":  # depth-sorted runs (prefix sums) and shuffled ones (pairwise)
        fr = FragmentData(z["dist_off"], np.zeros(len(z["dist_w"]), np.int64), z["dist_w"], z[f"dist_{tag}_z"])
        v, dw, dz = DL.distortion_loss(fr, image_size=h * w + 5)
        assert abs(v - float(z[f"dist_{tag}_val"])) <= 1e-12 * max(1.0, abs(v))
        assert np.abs(dw - z[f"dist_{tag}_dw"]).max() <= 1e-12
        assert np.abs(dz - z[f"dist_{tag}_dz"]).max() <= 1e-12
        d = DL.depth_from_fragments(fr, h, w)
        assert np.abs(d - z[f"depth_{tag}"]).max() <= 1e-12


def test_distortion_long_and_mixed_runs():
    # run lengths 0..140 (one, two and five 32-fragment chunks), sorted runs with ties,
    # and shuffled runs whose first out-of-order pair sits at a chunk or lane boundary
    from paper_2505_19175_b200 import losses as DL
    from paper_2505_19175_b200.types import FragmentData
    rng = np.random.default_rng(17)
    lens = np.concatenate([np.arange(0, 141), rng.integers(0, 70, 300)])
    rng.shuffle(lens)
    off = np.zeros(len(lens) + 1, np.int64)
    off[1:] = np.cumsum(lens)
    w = rng.random(off[-1]) * 0.5
    z = np.empty(off[-1])
    for i, n in enumerate(lens):
        zz = np.sort(np.round(rng.random(n) * 20.0, 1) + 1.0)  # sorted, with ties
        if n >= 2 and i % 3 == 0:  # out of order at a lane / chunk boundary or anywhere
            k = [4, 8, 32, 33, int(rng.integers(1, n))][i % 5]
            k = k if k < n else int(rng.integers(1, n))
            zz[k - 1], zz[k] = zz[k] + 0.5, zz[k - 1]
        z[off[i]:off[i + 1]] = zz
    fr = FragmentData(off, np.zeros(len(w), np.int64), w, z)
    v, dw, dz = DL.distortion_loss(fr, image_size=len(lens))
    wv, wdw, wdz = OL.distortion_loss(off, w, z, image_size=len(lens))
    assert abs(v - wv) <= 1e-12 * max(1.0, abs(wv))
    assert np.abs(dw - wdw).max() <= 1e-12 * max(1.0, np.abs(wdw).max())
    assert np.abs(dz - wdz).max() <= 1e-12 * max(1.0, np.abs(wdz).max())


def test_distortion_on_rendered_fragments():
    # fragments of a real frame stay on the device: loss and gradients vs the oracle
    from paper_2505_19175_b200 import losses as DL
    from paper_2505_19175_b200 import scenes
    from paper_2505_19175_b200.rasterizer import DeviceSoup, Rasterizer
    soup, intr, pose = scenes.make_scene("c1")
    r = Rasterizer()
    r.forward(DeviceSoup.from_soup(soup, dtype=torch.float32), intr, pose, keep_backward=True)
    fr = r.fragments()
    v, dw, dz = DL.distortion_loss(fr, rasterizer=r)
    assert dw.is_cuda and dw.shape == fr.weight.shape
    wv, wdw, wdz = OL.distortion_loss(fr.offsets.cpu().numpy(), fr.weight.cpu().numpy(), fr.depth.cpu().numpy())
    assert abs(v - wv) <= 1e-10 * max(1.0, abs(wv))
    assert np.abs(dw.cpu().numpy() - wdw).max() <= 1e-10 * max(1.0, np.abs(wdw).max())
    assert np.abs(dz.cpu().numpy() - wdz).max() <= 1e-10 * max(1.0, np.abs(wdz).max())
    d = DL.depth_from_fragments(fr, intr.height, intr.width, rasterizer=r)
    wd = OL.depth_from_fragments(fr.offsets.cpu().numpy(), fr.weight.cpu().numpy(), fr.depth.cpu().numpy(),
                                 intr.height, intr.width)
    assert np.abs(d.cpu().numpy() - wd).max() <= 1e-10 * max(1.0, np.abs(wd).max())


def test_normal_loss_against_fixture_and_rendered_fragments():
    from paper_2505_19175_b200 import losses as DL
    from paper_2505_19175_b200 import scenes
    from paper_2505_19175_b200.rasterizer import DeviceSoup, Rasterizer
    from paper_2505_19175_b200.types import CameraIntrinsics, CameraPose, FragmentData, TriangleSoup
    z = np.load(GOLD)
    h, w = (int(v) for v in z["dist_hw"])
    fx, fy, cx, cy = (float(a) for a in z["nl_intr"])
    n = len(z["nl_verts"])
    soup = TriangleSoup(z["nl_verts"], np.full(n, 0.5), np.ones(n), np.zeros((n, 16, 3)))
    intr = CameraIntrinsics(fx=fx, fy=fy, cx=cx, cy=cy, width=w, height=h)
    pose = CameraPose(rotation=z["nl_rot"], translation=z["nl_trans"])
    fr = FragmentData(z["dist_off"], z["nl_tri"], z["dist_w"], z["dist_u_z"])
    v, dv, dw = DL.normal_loss(soup, fr, z["nl_depth"], intr, pose)
    assert abs(v - float(z["nl_val"])) <= 1e-12
    assert np.abs(dv - z["nl_dv"]).max() <= 1e-12 * max(1.0, np.abs(z["nl_dv"]).max()) + 1e-15
    assert np.abs(dw - z["nl_dw"]).max() <= 1e-12
    # on a rendered frame, everything on the device
    s2, intr2, pose2 = scenes.make_scene("c1")
    r = Rasterizer()
    ds = DeviceSoup.from_soup(s2, dtype=torch.float32)
    r.forward(ds, intr2, pose2, keep_backward=True)
    frs = r.fragments()
    depth = DL.depth_from_fragments(frs, intr2.height, intr2.width, rasterizer=r)
    v, dv, dw = DL.normal_loss(ds, frs, depth, intr2, pose2, rasterizer=r)
    assert dv.is_cuda and dw.shape == frs.weight.shape
    wv, wdv, wdw = OL.normal_loss(ds.vertices.double().cpu().numpy(), frs.offsets.cpu().numpy(),
                                  frs.triangle.cpu().numpy(), frs.weight.cpu().numpy(), depth.cpu().numpy(),
                                  intr2.fx, intr2.fy, intr2.cx, intr2.cy, np.asarray(pose2.rotation),
                                  np.asarray(pose2.translation))
    assert abs(v - wv) <= 1e-10 * max(1.0, abs(wv))
    assert np.abs(dv.cpu().numpy() - wdv).max() <= 1e-9 * max(1e-6, np.abs(wdv).max())
    assert np.abs(dw.cpu().numpy() - wdw).max() <= 1e-10
