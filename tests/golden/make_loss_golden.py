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
    # normal loss (losses.py:219-292): fp32-representable triangles seen by a
    # rotated camera, a smooth depth map and random fragment triangle ids
    G = importlib.import_module("trisplat.geometry")
    S = importlib.import_module("trisplat.soup")
    n_tri = 30
    r32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731
    verts = r32(rng.normal(0, 1, (n_tri, 1, 3)) + 0.3 * rng.normal(0, 1, (n_tri, 3, 3)))
    soup = S.TriangleSoup(verts, np.full(n_tri, 0.5), np.ones(n_tri), np.zeros((n_tri, 16, 3)))
    ang = 0.3
    rot = np.array([[np.cos(ang), 0, np.sin(ang)], [0, 1, 0], [-np.sin(ang), 0, np.cos(ang)]])
    pose = G.CameraPose(rotation=rot, translation=np.array([0.1, -0.2, 5.0]))
    intr = G.CameraIntrinsics(fx=9.0, fy=8.0, cx=3.4, cy=3.1, width=w, height=h)
    ys, xs = np.mgrid[0:h, 0:w]
    depth = 4.0 + 0.3 * np.sin(0.7 * xs) + 0.2 * np.cos(0.5 * ys) + 0.05 * rng.normal(0, 1, (h, w))
    ftri = rng.integers(0, n_tri, nf)
    fr = R.FragmentData(offsets=off, triangle=ftri, weight=wt, depth=z)
    val, dv, dw = L.normal_loss(soup, fr, depth, intr, pose)
    out.update(nl_verts=verts, nl_rot=rot, nl_trans=pose.translation, nl_intr=np.array([9.0, 8.0, 3.4, 3.1]),
               nl_depth=depth, nl_tri=ftri, nl_val=np.float64(val), nl_dv=dv, nl_dw=dw)
    np.savez_compressed(os.path.join(HERE, "loss.npz"), **out)
    print("wrote", k + 1, "cases")


if __name__ == "__main__":
    main()
