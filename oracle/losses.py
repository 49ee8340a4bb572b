"""CPU restatement of the reference's photometric loss (TEST INFRASTRUCTURE:
only tests/, __graft_entry__.smoke() and bench.py's CPU legs may use it).

Follows trisplat/losses.py:
  SSIM constants          :20-23   (11x11 window, sigma 1.5, K1 0.01, K2 0.03)
  _gaussian_1d            :48-52   normalised 1-D Gaussian
  _conv_same / _valid     :58-66   separable correlation, zero padding; valid crop
  _conv_adjoint           :69-73   zero-embedded gradient map, same correlation
  _ssim_channel           :76-107  per-window SSIM map, its partials, d(mean)/dx
  ssim                    :110-119 mean over channels, 1.0 below the window size
  photometric_loss        :122-142 (1-lam) L1 + lam (1-SSIM)/2 and its gradient
  distortion_loss         :153-203 pairwise w_i w_j |z_i - z_j| per pixel (prefix
                          sums for depth-sorted runs, pairwise otherwise)
  depth_from_fragments    :206-216 weight-normalised depth per pixel
  depth_normals / normal_loss :219-292 depth-map normals, triangle-normal alignment
in plain numpy, fp64.  Pinned to the live reference by tests/golden/loss.npz
(tests/golden/make_loss_golden.py).
"""
from __future__ import annotations

import numpy as np

WINDOW = 11
SIGMA = 1.5
K1 = 0.01
K2 = 0.03
HALF = WINDOW // 2


def gaussian_1d() -> np.ndarray:
    x = np.arange(-HALF, HALF + 1, dtype=np.float64)
    g = np.exp(-(x * x) / (2.0 * SIGMA * SIGMA))
    return g / g.sum()


_W = gaussian_1d()


def _corr1d(a: np.ndarray, axis: int) -> np.ndarray:
    """out[i] = sum_k w[k] a[i + k - HALF], zeros outside (correlate1d, mode=constant)."""
    a = np.moveaxis(a, axis, 0)
    n = a.shape[0]
    pad = np.zeros((n + 2 * HALF,) + a.shape[1:])
    pad[HALF:HALF + n] = a
    out = np.zeros_like(a, dtype=np.float64)
    for k in range(WINDOW):
        out += _W[k] * pad[k:k + n]
    return np.moveaxis(out, 0, axis)


def conv_same(x: np.ndarray) -> np.ndarray:
    return _corr1d(_corr1d(x, 0), 1)


def conv_valid(x: np.ndarray) -> np.ndarray:
    return conv_same(x)[HALF:-HALF, HALF:-HALF]


def conv_adjoint(g: np.ndarray, shape) -> np.ndarray:
    full = np.zeros(shape)
    full[HALF:-HALF, HALF:-HALF] = g
    return conv_same(full)


def ssim_channel(x: np.ndarray, y: np.ndarray):
    c1, c2 = K1 * K1, K2 * K2
    mx, my = conv_valid(x), conv_valid(y)
    exx, exy, eyy = conv_valid(x * x), conv_valid(x * y), conv_valid(y * y)
    vx, vy, cxy = exx - mx * mx, eyy - my * my, exy - mx * my
    a1, a2 = 2.0 * mx * my + c1, 2.0 * cxy + c2
    b1, b2 = mx * mx + my * my + c1, vx + vy + c2
    smap = (a1 * a2) / (b1 * b2)
    s = 1.0 / smap.size
    da1, da2 = a2 / (b1 * b2), a1 / (b1 * b2)
    db1, db2 = -smap / b1, -smap / b2
    g_mu = 2.0 * my * da1 + 2.0 * mx * db1 - 2.0 * my * da2 - 2.0 * mx * db2
    dx = conv_adjoint(g_mu * s, x.shape) + 2.0 * x * conv_adjoint(db2 * s, x.shape) \
        + y * conv_adjoint(2.0 * da2 * s, x.shape)
    return float(smap.mean()), dx


def ssim(x, y) -> float:
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if x.shape != y.shape:
        raise ValueError("image dimensions differ")
    if x.shape[0] < WINDOW or x.shape[1] < WINDOW:
        return 1.0
    return float(np.mean([ssim_channel(x[..., c], y[..., c])[0] for c in range(x.shape[2])]))


def photometric_loss(rendered, target, lam: float):
    r = np.asarray(rendered, dtype=np.float64)
    t = np.asarray(target, dtype=np.float64)
    if r.shape != t.shape:
        raise ValueError(f"image dimensions differ: {r.shape} vs {t.shape}")
    d = r - t
    l1 = float(np.abs(d).mean())
    g_l1 = np.sign(d) / d.size
    if lam == 0.0:
        return l1, g_l1
    if r.shape[0] < WINDOW or r.shape[1] < WINDOW:
        sv, g_s = 1.0, np.zeros_like(r)
    else:
        vals, g_s = [], np.zeros_like(r)
        for c in range(r.shape[2]):
            v, dx = ssim_channel(r[..., c], t[..., c])
            vals.append(v)
            g_s[..., c] = dx / r.shape[2]
        sv = float(np.mean(vals))
    return (1.0 - lam) * l1 + lam * (1.0 - sv) / 2.0, (1.0 - lam) * g_l1 - (lam / 2.0) * g_s


def distortion_loss(off, w, z, image_size=None):
    off = np.asarray(off, dtype=np.int64)
    w = np.asarray(w, dtype=np.float64)
    z = np.asarray(z, dtype=np.float64)
    npix = len(off) - 1
    scale = 1.0 / max(image_size if image_size is not None else npix, 1)
    if len(w) == 0:
        return 0.0, np.zeros(0), np.zeros(0)
    d_w, d_z = np.zeros_like(w), np.zeros_like(w)
    total = 0.0
    counts = np.diff(off)
    seg = np.repeat(np.arange(npix), counts)
    same = seg[1:] == seg[:-1]
    if (z[1:][same] >= z[:-1][same]).all():
        for p in range(npix):
            lo, hi = off[p], off[p + 1]
            ws, zs = w[lo:hi], z[lo:hi]
            wb = np.concatenate([[0.0], np.cumsum(ws)[:-1]]) if hi > lo else ws
            sb = np.concatenate([[0.0], np.cumsum(ws * zs)[:-1]]) if hi > lo else ws
            wa, sa = ws.sum() - wb - ws, (ws * zs).sum() - sb - ws * zs
            fwd = zs * wb - sb
            total += 2.0 * float((ws * fwd).sum())
            d_w[lo:hi] = 2.0 * (fwd + (sa - zs * wa))
            d_z[lo:hi] = 2.0 * ws * (wb - wa)
    else:
        for p in range(npix):
            lo, hi = off[p], off[p + 1]
            if hi - lo < 2:
                continue
            ws, zs = w[lo:hi], z[lo:hi]
            dz = np.abs(zs[:, None] - zs[None, :])
            total += float(ws @ dz @ ws)
            d_w[lo:hi] = 2.0 * dz @ ws
            d_z[lo:hi] = 2.0 * (np.sign(zs[:, None] - zs[None, :]) * ws[None, :]).sum(axis=1) * ws
    return total * scale, d_w * scale, d_z * scale


def depth_from_fragments(off, w, z, height, width):
    off = np.asarray(off, dtype=np.int64)
    d = np.zeros(height * width)
    ws = np.zeros(height * width)
    idx = np.repeat(np.arange(height * width), np.diff(off))
    np.add.at(d, idx, np.asarray(w) * np.asarray(z))
    np.add.at(ws, idx, np.asarray(w))
    return (d / np.maximum(ws, 1e-8)).reshape(height, width)


def depth_normals(depth, fx, fy, cx, cy):
    h, w = depth.shape
    ys, xs = np.mgrid[0:h, 0:w]
    p = np.stack([depth * (xs + 0.5 - cx) / fx, depth * (ys + 0.5 - cy) / fy, depth], axis=-1)
    q = np.pad(p, ((1, 1), (1, 1), (0, 0)), mode="edge")
    gx = (q[1:-1, 2:] - q[1:-1, :-2]) / 2.0
    gy = (q[2:, 1:-1] - q[:-2, 1:-1]) / 2.0
    n = np.cross(gx, gy)
    n = n / np.maximum(np.linalg.norm(n, axis=-1, keepdims=True), 1e-12)
    n[n[..., 2] > 0] *= -1.0
    return n


def normal_loss(vertices, off, tri, wgt, depth, fx, fy, cx, cy, rot, trans):
    v = np.asarray(vertices, dtype=np.float64)
    n_tri, nf = len(v), len(wgt)
    if nf == 0:
        return 0.0, np.zeros((n_tri, 3, 3)), np.zeros(0)
    h, w = depth.shape
    mw = depth_normals(depth, fx, fy, cx, cy).reshape(-1, 3)[np.repeat(np.arange(h * w), np.diff(off))] @ rot
    a, b = v[:, 1] - v[:, 0], v[:, 2] - v[:, 0]
    c = np.cross(a, b)
    cn = np.maximum(np.linalg.norm(c, axis=1), 1e-12)
    ch = c / cn[:, None]
    facing = ((ch @ rot.T) * (v.mean(axis=1) @ rot.T + trans)).sum(axis=1)
    fl = np.where(facing > 0, -1.0, 1.0)
    tri = np.asarray(tri, dtype=np.int64)
    cm = (ch[tri] * mw).sum(axis=1)
    dot = cm * fl[tri]
    value = float((wgt * (1.0 - dot)).sum() / nf)
    d_w = (1.0 - dot) / nf
    g = np.zeros((n_tri, 3))
    np.add.at(g, tri, (-wgt * fl[tri] / nf)[:, None] * (mw - ch[tri] * cm[:, None]) / cn[tri, None])
    da, db = np.cross(b, g), np.cross(g, a)
    dv = np.zeros((n_tri, 3, 3))
    dv[:, 1], dv[:, 2], dv[:, 0] = da, db, -(da + db)
    return value, dv, d_w
