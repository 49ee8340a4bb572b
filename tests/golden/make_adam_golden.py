"""Golden fixtures of the reference's adam_step (trisplat/training.py:81-110),
run in the build container:  NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_adam_golden.py
A 40-triangle soup, 5 steps with seeded gradients and per-group rates (large
enough to hit both clamps); stores the initial parameters, every step's
gradients and the parameters after each step."""
from __future__ import annotations

import importlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
T = importlib.import_module("trisplat.training")
S = importlib.import_module("trisplat.soup")
B = importlib.import_module("trisplat.backward")


def main():
    rng = np.random.default_rng(77)
    n = 40
    r32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731
    soup = S.TriangleSoup(r32(rng.normal(0, 1, (n, 3, 3))), r32(rng.uniform(0.05, 0.95, n)),
                          r32(rng.uniform(0.01, 5.0, n)), r32(rng.normal(0, 0.3, (n, 16, 3))))
    out = {"v0": soup.vertices.copy(), "o0": soup.opacity.copy(), "s0": soup.sigma.copy(), "h0": soup.sh.copy()}
    lrs = {"vertices": 0.01, "opacity": 0.3, "sigma": 0.5, "sh": 0.02}
    state = T.AdamState.zeros(soup)
    for k in range(5):
        g = B.GradientSet(r32(rng.normal(0, 1, (n, 3, 3))), r32(rng.normal(0, 2, n)), r32(rng.normal(0, 2, n)),
                          r32(rng.normal(0, 0.1, (n, 16, 3))))
        T.adam_step(soup, g, state, lrs)
        for a, b in (("gv", g.d_vertices), ("go", g.d_opacity), ("gs", g.d_sigma), ("gh", g.d_sh),
                     ("v", soup.vertices), ("o", soup.opacity), ("s", soup.sigma), ("h", soup.sh)):
            out[f"{a}{k + 1}" if a in ("v", "o", "s", "h") else f"{a}{k}"] = np.array(b, copy=True)
    out["lrs"] = np.array([lrs["vertices"], lrs["opacity"], lrs["sigma"], lrs["sh"]])
    np.savez_compressed(os.path.join(HERE, "adam.npz"), **out)
    print("wrote adam.npz")


if __name__ == "__main__":
    main()
