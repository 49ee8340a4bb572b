"""Golden fixtures of the reference's density control (trisplat/density.py:27-263),
run in the build container:  NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_density_golden.py

Each case: a soup with fp32-representable values (some degenerate and some
low-opacity triangles), per-view statistics fed to ViewStats.update in a fixed
order (one view re-recorded, which keeps its first position), a DensifyConfig,
an iteration and an rng seed; stored with densify_step's new soup, origin and
report counts."""
from __future__ import annotations

import dataclasses
import importlib
import os
import sys
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
D = importlib.import_module("trisplat.density")
S = importlib.import_module("trisplat.soup")
C = importlib.import_module("trisplat.config")

r32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731

CASES = [
    # name, n, n_views, iteration, cfg overrides, soup seed
    ("sigma", 300, 5, 500, {}, 1),
    ("opacity", 300, 5, 1000, {}, 2),
    ("unscheduled", 50, 3, 501, {}, 3),
    ("rounds", 120, 4, 500, {"growth_rate": 1.7, "tau_small": 10.0}, 4),
    ("all_pruned", 40, 3, 500, {"tau_prune": 2.0}, 5),
    ("few_adds", 60, 3, 1000, {"growth_rate": 0.05, "tau_small": 5.0}, 6),
]


def make_case(name, n, n_views, iteration, over, seed):
    rng = np.random.default_rng(seed)
    v = r32(rng.normal(0, 1, (n, 3, 3)))
    deg = rng.choice(n, size=max(n // 15, 1), replace=False)
    v[deg, 2] = v[deg, 0]  # degenerate: two equal vertices
    opacity = r32(rng.uniform(0.001, 0.9, n))
    sigma = r32(rng.uniform(0.05, 4.0, n))
    sh = r32(rng.normal(0, 0.3, (n, 16, 3)))
    soup = S.TriangleSoup(v, opacity, sigma, sh)
    stats = D.ViewStats.empty(n)
    views = []
    order = list(range(n_views)) + [1]  # view 1 is re-recorded last
    for vid in order:
        maxw = r32(rng.uniform(0, 0.1, n) * (rng.uniform(0, 1, n) < 0.9))
        pix = rng.integers(0, 6, n)
        area = r32(rng.uniform(0, 60, n))
        out = types.SimpleNamespace(per_triangle_max_weight=maxw, per_triangle_pixel_count=pix,
                                    per_triangle_area=area)
        stats.update(vid, out, min_pixels=2)
        views.append((vid, maxw, pix, area))
    cfg = dataclasses.replace(C.DensifyConfig(), **over)
    new, rep = D.densify_step(soup, stats, iteration, cfg, np.random.default_rng(100 + seed))
    out = {"v": v, "o": opacity, "s": sigma, "h": sh,
           "view_ids": np.array([x[0] for x in views]), "maxw": np.stack([x[1] for x in views]),
           "pix": np.stack([x[2] for x in views]), "area": np.stack([x[3] for x in views]),
           "iteration": np.array(iteration), "seed": np.array(100 + seed),
           "cfg": np.array([cfg.tau_prune, cfg.min_views, cfg.min_pixels, cfg.opacity_dead, cfg.growth_rate,
                            cfg.tau_small, cfg.max_noise_factor, cfg.interval, cfg.start_iter, cfg.stop_iter]),
           "nv": new.vertices, "no": new.opacity, "ns": new.sigma, "nh": new.sh, "origin": rep["origin"],
           "scheduled": np.array(rep["scheduled"])}
    if rep["scheduled"]:
        pr = rep["prune"]
        mask = np.zeros((3, n), dtype=bool)
        for i, k in enumerate(("low_weight", "few_views", "dead_opacity")):
            mask[i, pr[k]] = True
        out["prune_mask"] = mask
        out["counts"] = np.array([rep.get("n_add", 0), rep.get("n_split", 0), rep.get("n_clone", 0),
                                  pr["n_removed"]])
    return out


def main():
    out = {}
    for case in CASES:
        for k, a in make_case(*case).items():
            out[f"{case[0]}__{k}"] = a
    np.savez_compressed(os.path.join(HERE, "density.npz"), **out)
    print("wrote density.npz", sorted({k.split("__")[0] for k in out}))


if __name__ == "__main__":
    main()
