"""CPU: the photometric-loss oracle (oracle/losses.py) against the live
reference's fixtures (tests/golden/loss.npz, make_loss_golden.py) and the
reference's own loss tests (test_losses.py:68-120) re-run on the oracle."""
import os

import numpy as np
import pytest

from oracle import losses as OL

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "loss.npz")


def test_oracle_matches_reference_fixtures():
    z = np.load(GOLD)
    for k in range(int(z["n"])):
        loss, grad = OL.photometric_loss(z[f"x{k}"], z[f"y{k}"], float(z[f"lam{k}"]))
        assert abs(loss - float(z[f"loss{k}"])) <= 1e-12, k
        assert np.abs(grad - z[f"grad{k}"]).max() <= 1e-12, k
        assert abs(OL.ssim(z[f"x{k}"], z[f"y{k}"]) - float(z[f"ssim{k}"])) <= 1e-12, k


def test_reference_cases():
    x = np.random.default_rng(3).uniform(0, 1, (16, 16, 3))
    assert OL.photometric_loss(x, x, 0.2)[0] == pytest.approx(0.0, abs=1e-12)
    assert OL.photometric_loss(np.zeros((16, 16, 3)), np.ones((16, 16, 3)), 0.0)[0] == pytest.approx(1.0)
    rng = np.random.default_rng(4)
    a, b = rng.uniform(0, 1, (14, 14, 3)), rng.uniform(0, 1, (14, 14, 3))
    assert OL.photometric_loss(a, b, 0.0)[0] == pytest.approx(OL.photometric_loss(b, a, 0.0)[0])
    assert OL.photometric_loss(np.full((4, 4, 3), 0.3), np.full((4, 4, 3), 0.7), 0.5)[0] == pytest.approx(0.2)
    assert OL.ssim(x, x) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        OL.ssim(np.zeros((16, 16, 3)), np.zeros((17, 16, 3)))
    with pytest.raises(ValueError):
        OL.photometric_loss(np.zeros((16, 16, 3)), np.zeros((17, 16, 3)), 0.2)


def test_gradient_matches_finite_differences():
    rng = np.random.default_rng(5)
    x, y = rng.uniform(0.2, 0.8, (16, 16, 3)), rng.uniform(0.2, 0.8, (16, 16, 3))
    _, g = OL.photometric_loss(x, y, 0.2)
    h = 1e-6
    for _ in range(10):
        i, j, c = rng.integers(16), rng.integers(16), rng.integers(3)
        xp, xm = x.copy(), x.copy()
        xp[i, j, c] += h
        xm[i, j, c] -= h
        fd = (OL.photometric_loss(xp, y, 0.2)[0] - OL.photometric_loss(xm, y, 0.2)[0]) / (2 * h)
        assert g[i, j, c] == pytest.approx(fd, rel=1e-4, abs=1e-9)


def test_distortion_and_depth_match_reference_fixtures():
    z = np.load(GOLD)
    h, w = (int(v) for v in z["dist_hw"])
    for tag in "su":
        v, dw, dz = OL.distortion_loss(z["dist_off"], z["dist_w"], z[f"dist_{tag}_z"], image_size=h * w + 5)
        assert abs(v - float(z[f"dist_{tag}_val"])) <= 1e-12
        assert np.abs(dw - z[f"dist_{tag}_dw"]).max() <= 1e-12
        assert np.abs(dz - z[f"dist_{tag}_dz"]).max() <= 1e-12
        d = OL.depth_from_fragments(z["dist_off"], z["dist_w"], z[f"dist_{tag}_z"], h, w)
        assert np.abs(d - z[f"depth_{tag}"]).max() <= 1e-12


def test_normal_loss_matches_reference_fixture():
    z = np.load(GOLD)
    fx, fy, cx, cy = z["nl_intr"]
    v, dv, dw = OL.normal_loss(z["nl_verts"], z["dist_off"], z["nl_tri"], z["dist_w"], z["nl_depth"],
                               fx, fy, cx, cy, z["nl_rot"], z["nl_trans"])
    assert abs(v - float(z["nl_val"])) <= 1e-12
    assert np.abs(dv - z["nl_dv"]).max() <= 1e-12
    assert np.abs(dw - z["nl_dw"]).max() <= 1e-12
