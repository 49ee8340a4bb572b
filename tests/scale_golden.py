"""Checks against the at-scale live-reference digests (tests/golden/scale_*.npz,
made by tests/golden/make_golden_scale.py).  Shared by the CPU oracle pin
(test_oracle_scale.py) and the GPU parity tests (test_gpu_scale.py)."""
from __future__ import annotations

import os

import numpy as np

from conftest import GOLDEN, digest

RGB_TOL = 1e-5
MAXW_TOL = 1e-6
# gradients: |got - want| <= GRAD_RTOL * |want| + GRAD_ATOL per element (the
# reference's own criterion, test_backward.py:171, pytest.approx(rel=1e-4, abs=1e-7))
GRAD_RTOL = 1e-4
GRAD_ATOL = 1e-7
GROUPS = ("d_vertices", "d_opacity", "d_sigma", "d_sh")


def load(name):
    return np.load(os.path.join(GOLDEN, f"scale_{name}.npz"))


def check_inputs(z, soup):
    assert str(z["input_digest"]) == digest(soup.vertices, soup.opacity, soup.sigma, soup.sh), \
        "scene generator drifted from the golden inputs"


def check_forward(z, *, sorted_idx, tile_start, entry_tri, last_src, nfrag, pixcount, image, alpha, maxw,
                  area, label=""):
    """Discrete outputs bit-exact (digests), floats within the north_star tolerances."""
    assert len(sorted_idx) == int(z["n_visible"]), f"{label} visible count"
    assert len(entry_tri) == int(z["n_entries"]), f"{label} entry count"
    assert int(np.asarray(nfrag).sum()) == int(z["n_fragments"]), f"{label} fragment count"
    assert digest(np.asarray(sorted_idx, np.int64)) == str(z["sorted_idx_digest"]), f"{label} sort order"
    assert digest(np.asarray(tile_start, np.int64)) == str(z["tile_start_digest"]), f"{label} tile_start"
    assert digest(np.asarray(entry_tri, np.int64)) == str(z["entry_tri_digest"]), f"{label} tile lists"
    assert digest(np.asarray(last_src, np.int32).reshape(-1)) == str(z["last_src_digest"]), \
        f"{label} last contributor"
    assert digest(np.asarray(nfrag, np.int32).reshape(-1)) == str(z["nfrag_digest"]), f"{label} fragments/px"
    assert digest(np.asarray(pixcount, np.int64)) == str(z["pixcount_digest"]), f"{label} pixel counts"
    img = np.asarray(image, np.float64).reshape(-1, 3)
    ps, ts = z["pix_sample"], z["tri_sample"]
    assert np.abs(img[ps] - z["image_sample"]).max() <= RGB_TOL, f"{label} rgb sample"
    assert np.abs(img.sum(0) - z["image_sum"]).max() <= RGB_TOL * len(img), f"{label} rgb sum"
    a = np.asarray(alpha, np.float64).reshape(-1)
    assert np.abs(a[ps] - z["alpha_sample"]).max() <= RGB_TOL, f"{label} alpha sample"
    assert np.abs(np.asarray(maxw, np.float64)[ts] - z["maxw_sample"]).max() <= MAXW_TOL, f"{label} max weight"
    ar = np.asarray(area, np.float64)[ts]
    assert np.allclose(ar, z["area_sample"], rtol=1e-6, atol=1e-6), f"{label} area"


def grad_violations(got, want, rtol=GRAD_RTOL, atol=GRAD_ATOL):
    """Elements outside |got - want| <= rtol |want| + atol, and the worst ratio."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    tol = rtol * np.abs(want) + atol
    d = np.abs(got - want)
    bad = d > tol
    worst = float((d / tol).max()) if d.size else 0.0
    return int(bad.sum()), worst


def grad_rows(g):
    n = len(g.d_opacity)
    return np.concatenate([np.asarray(g.d_vertices).reshape(n, 9), np.asarray(g.d_opacity).reshape(n, 1),
                           np.asarray(g.d_sigma).reshape(n, 1), np.asarray(g.d_sh).reshape(n, 48)], axis=1)


def check_grad_sample(z, rows, label=""):
    """Sampled 59-value rows against the live reference's, plus group sums."""
    nb, worst = grad_violations(rows[z["tri_sample"]], z["grad_sample"])
    assert nb == 0, f"{label} {nb} sampled gradient values outside rtol 1e-4 + atol 1e-7 (worst {worst:.2f}x)"
    n = rows.shape[0]
    sums = [rows[:, :9].sum(), rows[:, 9].sum(), rows[:, 10].sum(), rows[:, 11:].sum()]
    abs_sums = [np.abs(rows[:, :9]).sum(), np.abs(rows[:, 9]).sum(), np.abs(rows[:, 10]).sum(),
                np.abs(rows[:, 11:]).sum()]
    for k in range(4):
        assert abs(abs_sums[k] - z["grad_abs_sum"][k]) <= 1e-6 * z["grad_abs_sum"][k] + 1e-7 * n, \
            f"{label} {GROUPS[k]} |sum|"
        assert abs(sums[k] - z["grad_sum"][k]) <= 1e-6 * z["grad_abs_sum"][k] + 1e-7 * n, f"{label} {GROUPS[k]} sum"
