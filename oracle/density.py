"""CPU restatement of the reference's adaptive density control (TEST
INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's CPU legs
may use it).

Follows trisplat/density.py:
  ViewStats aggregation   :42-71   per-view (max weight, covered, area), replaced
                                   views keep their first position; max / count / mean
  prune                   :74-94   low weight | few covering views | dead opacity
  sample_weights          :97-100  1 / max(sigma, 1e-12) or max(opacity, 0)
  sample_candidates       :103-120 exponential keys, stable argsort, first count
  midpoint_subdivide      :123-143 four children at the edge midpoints
  clone_with_noise        :146-171 per vertex: angle, radius draws; in-plane offset
  step_criterion          :174-177 alternating criterion per density step
  densify_step            :180-263 prune, then ceil(growth_rate * alive) additions
in plain numpy / Python loops over the picks, fp64.  Pinned to the live reference
by tests/golden/density.npz (tests/golden/make_density_golden.py).
"""
from __future__ import annotations

import math

import numpy as np

CFG_KEYS = ("tau_prune", "min_views", "min_pixels", "opacity_dead", "growth_rate", "tau_small",
            "max_noise_factor", "interval", "start_iter", "stop_iter")


def aggregate(per_view):
    """per_view: list of (max_weight, covered, area) in dict order."""
    n = len(per_view[0][0]) if per_view else 0
    mw = np.zeros(n)
    views = np.zeros(n, dtype=np.int64)
    area = np.zeros(n)
    for w, cov, a in per_view:
        mw = np.maximum(mw, w)
        views = views + cov
        area = area + a
    return mw, views, area / max(len(per_view), 1)


def record_views(view_ids, maxw, pix, area, min_pixels):
    """ViewStats.update sequence -> the per-view list in dict order."""
    d = {}
    for k, vid in enumerate(view_ids):
        d[int(vid)] = (np.asarray(maxw[k], np.float64), np.asarray(pix[k]) >= min_pixels,
                       np.asarray(area[k], np.float64))
    return list(d.values())


def _norm(x):
    return math.sqrt(float(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]))


def densify(v, o, s, h, per_view, iteration, cfg, rng):
    """Returns dict(v, o, s, h, origin, scheduled, masks (3,N), counts [n_add, n_split, n_clone, n_removed])."""
    c = dict(zip(CFG_KEYS, cfg))
    n0 = len(v)
    sched = (c["start_iter"] <= iteration <= c["stop_iter"]
             and (iteration - c["start_iter"]) % int(c["interval"]) == 0)
    if not sched or n0 == 0:
        return dict(v=v, o=o, s=s, h=h, origin=np.arange(n0), scheduled=False)
    mw, views, mean_area = aggregate(per_view)
    masks = np.stack([mw < c["tau_prune"], views < c["min_views"], o < c["opacity_dead"]])
    kept = np.nonzero(~masks.any(axis=0))[0]
    counts = [0, 0, 0, int(masks.any(axis=0).sum())]
    if len(kept) == 0:
        z = np.zeros(0, np.int64)
        return dict(v=v[z], o=o[z], s=s[z], h=h[z], origin=z, scheduled=True, masks=masks, counts=counts)
    sv, so, ss = v[kept], o[kept], s[kept]
    ma = mean_area[kept]
    inverse = ((iteration - c["start_iter"]) // int(c["interval"])) % 2 == 0
    n_add = math.ceil(c["growth_rate"] * len(kept))
    removed = np.zeros(len(kept), dtype=bool)
    child_v, child_src = [], []
    n_split = n_clone = 0
    remaining = n_add
    while remaining > 0:
        pool = np.nonzero(~removed)[0]
        if len(pool) == 0:
            break
        w = 1.0 / np.maximum(ss[pool], 1e-12) if inverse else np.maximum(so[pool], 0.0)
        tot = w.sum()
        if not np.isfinite(tot) or tot <= 0:
            w = np.ones(len(pool))
        keys = rng.exponential(size=len(pool)) / np.maximum(w, 1e-300)
        picks = np.argsort(keys, kind="stable")[:min(remaining, len(pool))]
        for loc in picks:
            if remaining <= 0:
                break
            i = int(pool[loc])
            p = sv[i]
            area2 = _norm(np.cross(p[1] - p[0], p[2] - p[0]))
            if ma[i] >= c["tau_small"] and remaining >= 3 and area2 >= 1e-12:
                m01, m12, m20 = (p[0] + p[1]) / 2.0, (p[1] + p[2]) / 2.0, (p[2] + p[0]) / 2.0
                child_v += [np.stack(q) for q in ((p[0], m01, m20), (m01, p[1], m12), (m20, m12, p[2]),
                                                  (m01, m12, m20))]
                child_src += [kept[i]] * 4
                removed[i] = True
                n_split += 1
                remaining -= 3
                continue
            q = p.copy()
            mean_edge = (_norm(p[1] - p[0]) + _norm(p[2] - p[1]) + _norm(p[0] - p[2])) / 3.0
            if area2 >= 1e-12 and mean_edge != 0.0:
                nrm = np.cross(p[1] - p[0], p[2] - p[0]) / area2
                b1 = (p[1] - p[0]) / _norm(p[1] - p[0])
                b2 = np.cross(nrm, b1)
                cap = c["max_noise_factor"] * mean_edge
                for j in range(3):
                    ang = rng.uniform(0.0, 2.0 * math.pi)
                    rad = rng.uniform(0.0, cap)
                    q[j] = q[j] + rad * (math.cos(ang) * b1 + math.sin(ang) * b2)
            child_v.append(q)
            child_src.append(kept[i])
            n_clone += 1
            remaining -= 1
    base = kept[~removed]
    origin = np.concatenate([base, np.asarray(child_src, dtype=np.int64)]).astype(np.int64)
    nv = np.concatenate([v[base], np.asarray(child_v).reshape(-1, 3, 3)]) if child_v else v[base]
    counts[:3] = [n_add, n_split, n_clone]
    return dict(v=nv, o=o[origin], s=s[origin], h=h[origin], origin=origin, scheduled=True, masks=masks,
                counts=counts)
