"""CPU restatement of the reference's Adam step (TEST INFRASTRUCTURE: only
tests/ may use it).  Follows trisplat/training.py:22-28 (constants, groups),
:81-110 adam_step: finiteness check of every group first (the first offending
triangle of the first bad group is reported), then t += 1, bias-corrected
Adam per group with per-group learning rates, then the opacity / sigma clamps.
fp64 state; parameters are updated in place."""
from __future__ import annotations

import numpy as np

BETA1, BETA2, EPS = 0.9, 0.999, 1e-15
OPACITY_CLAMP = (1e-4, 1.0 - 1e-4)
SIGMA_CLAMP = (1e-3, 1e3)
GROUPS = ("vertices", "opacity", "sigma", "sh")


class State:
    def __init__(self, n):
        shapes = {"vertices": (n, 3, 3), "opacity": (n,), "sigma": (n,), "sh": (n, 16, 3)}
        self.m = {k: np.zeros(s) for k, s in shapes.items()}
        self.v = {k: np.zeros(s) for k, s in shapes.items()}
        self.t = 0


def adam_step(params: dict, grads: dict, state: State, lrs: dict):
    n = len(params["opacity"])
    for k in GROUPS:
        flat = np.asarray(grads[k]).reshape(n, -1) if n else np.zeros((0, 1))
        bad = ~np.isfinite(flat).all(axis=1)
        if bad.any():
            raise ValueError(f"non-finite {k} gradient for triangle {int(np.nonzero(bad)[0][0])}")
    state.t += 1
    c1, c2 = 1.0 - BETA1 ** state.t, 1.0 - BETA2 ** state.t
    for k in GROUPS:
        g = np.asarray(grads[k], dtype=np.float64)
        state.m[k] = BETA1 * state.m[k] + (1.0 - BETA1) * g
        state.v[k] = BETA2 * state.v[k] + (1.0 - BETA2) * g * g
        params[k] -= lrs[k] * (state.m[k] / c1) / (np.sqrt(state.v[k] / c2) + EPS)
    np.clip(params["opacity"], *OPACITY_CLAMP, out=params["opacity"])
    np.clip(params["sigma"], *SIGMA_CLAMP, out=params["sigma"])
