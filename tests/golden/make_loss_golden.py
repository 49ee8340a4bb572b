"""Golden fixtures of the photometric loss from the LIVE reference
(trisplat/losses.py:122-142), run in the build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_loss_golden.py

Cases: random image pairs of several shapes (incl. below the 11x11 SSIM
window and non-multiples of 16), lam in {0, 0.2, 1}, identical images and a
constant pair; stores inputs, loss and gradient.
"""
from __future__ import annotations

import importlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
L = importlib.import_module("trisplat.losses")


def main():
    rng = np.random.default_rng(2024)
    out = {}
    cases = [((16, 16), 0.2), ((20, 23), 0.2), ((37, 29), 1.0), ((48, 40), 0.0), ((8, 9), 0.5),
             ((11, 11), 0.2), ((64, 50), 0.2)]
    for k, ((h, w), lam) in enumerate(cases):
        x = rng.uniform(0, 1, (h, w, 3))
        y = np.clip(x + rng.normal(0, 0.15, x.shape), 0, 1)
        loss, grad = L.photometric_loss(x, y, lam)
        out[f"x{k}"], out[f"y{k}"], out[f"lam{k}"] = x, y, np.float64(lam)
        out[f"loss{k}"], out[f"grad{k}"] = np.float64(loss), grad
        out[f"ssim{k}"] = np.float64(L.ssim(x, y))
    k = len(cases)
    x = rng.uniform(0, 1, (24, 24, 3))
    out[f"x{k}"], out[f"y{k}"], out[f"lam{k}"] = x, x.copy(), np.float64(0.2)
    loss, grad = L.photometric_loss(x, x, 0.2)
    out[f"loss{k}"], out[f"grad{k}"], out[f"ssim{k}"] = np.float64(loss), grad, np.float64(L.ssim(x, x))
    out["n"] = np.int64(k + 1)
    # distortion loss / depth map over fragment lists (losses.py:169-216):
    # a depth-sorted set (prefix-sum path) and a shuffled one (pairwise path)
    R = importlib.import_module("trisplat.render")
    h, w = 6, 7
    counts = rng.integers(0, 9, h * w)
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    nf = int(off[-1])
    wt = rng.uniform(0, 0.5, nf)
    z = rng.uniform(1, 5, nf)
    zs = z.copy()
    for p in range(h * w):
        zs[off[p]:off[p + 1]] = np.sort(zs[off[p]:off[p + 1]])
    for tag, zz in (("s", zs), ("u", z)):
        fr = R.FragmentData(offsets=off, triangle=np.zeros(nf, np.int64), weight=wt, depth=zz)
        val, dw, dz = L.distortion_loss(fr, image_size=h * w + 5)
        out[f"dist_{tag}_z"], out[f"dist_{tag}_val"], out[f"dist_{tag}_dw"], out[f"dist_{tag}_dz"] = zz, val, dw, dz
        out[f"depth_{tag}"] = L.depth_from_fragments(fr, h, w)
    out["dist_off"], out["dist_w"], out["dist_hw"] = off, wt, np.array([h, w])
    np.savez_compressed(os.path.join(HERE, "loss.npz"), **out)
    print("wrote", k + 1, "cases")


if __name__ == "__main__":
    main()
