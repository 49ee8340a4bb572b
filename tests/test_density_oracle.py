"""The density-control oracle (oracle/density.py) against the reference's
densify_step on the golden cases (tests/golden/density.npz): origin, prune
masks and counts exact; children vertices to rounding."""
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = ["sigma", "opacity", "unscheduled", "rounds", "all_pruned", "few_adds"]


def load_case(name):
    d = np.load(os.path.join(HERE, "golden", "density.npz"))
    return {k.split("__", 1)[1]: d[k] for k in d.files if k.startswith(name + "__")}


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference(name):
    from oracle import density as OD
    g = load_case(name)
    cfg = g["cfg"]
    per_view = OD.record_views(g["view_ids"], g["maxw"], g["pix"], g["area"], int(cfg[2]))
    r = OD.densify(g["v"], g["o"], g["s"], g["h"], per_view, int(g["iteration"]), cfg,
                   np.random.default_rng(int(g["seed"])))
    assert bool(r["scheduled"]) == bool(g["scheduled"])
    assert np.array_equal(r["origin"], g["origin"])
    if g["scheduled"]:
        assert np.array_equal(r["masks"], g["prune_mask"])
        assert list(r["counts"]) == list(g["counts"])
    assert np.array_equal(r["o"], g["no"]) and np.array_equal(r["s"], g["ns"]) and np.array_equal(r["h"], g["nh"])
    assert r["v"].shape == g["nv"].shape
    np.testing.assert_allclose(r["v"], g["nv"], rtol=0, atol=1e-12)
