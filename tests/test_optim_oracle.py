"""CPU: the Adam oracle (oracle/optim.py) against the live reference's
adam_step fixtures (tests/golden/adam.npz, make_adam_golden.py)."""
import os

import numpy as np
import pytest

from oracle import optim as OP

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "adam.npz")


def _params(z):
    return {"vertices": z["v0"].copy(), "opacity": z["o0"].copy(), "sigma": z["s0"].copy(), "sh": z["h0"].copy()}


def _grads(z, k):
    return {"vertices": z[f"gv{k}"], "opacity": z[f"go{k}"], "sigma": z[f"gs{k}"], "sh": z[f"gh{k}"]}


def test_oracle_matches_reference_steps():
    z = np.load(GOLD)
    p, st = _params(z), OP.State(len(z["o0"]))
    lrs = dict(zip(OP.GROUPS, z["lrs"]))
    for k in range(5):
        OP.adam_step(p, _grads(z, k), st, lrs)
        for key, name in (("vertices", "v"), ("opacity", "o"), ("sigma", "s"), ("sh", "h")):
            assert np.array_equal(p[key], z[f"{name}{k + 1}"]), (k, key)


def test_non_finite_raises_before_any_change():
    z = np.load(GOLD)
    p, st = _params(z), OP.State(len(z["o0"]))
    g = {k: np.array(v, copy=True) for k, v in _grads(z, 0).items()}
    g["sh"][7, 3, 1] = np.nan
    g["sh"][2, 0, 0] = np.inf
    with pytest.raises(ValueError, match="non-finite sh gradient for triangle 2"):
        OP.adam_step(p, g, st, dict(zip(OP.GROUPS, z["lrs"])))
    assert st.t == 0 and np.array_equal(p["vertices"], z["v0"])
