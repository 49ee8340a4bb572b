"""GPU parity of the device density control (ts_density.cu via density.py)
with the reference's densify_step (golden cases, tests/golden/density.npz) and
with the oracle at a larger size: origin, prune report and counts exact, new
opacity / sigma / SH exact, children vertices to fp64 rounding (fp64 soup) or
fp32 rounding (fp32 soup); the Adam moment remap against numpy."""
import os
import types

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = ["sigma", "opacity", "unscheduled", "rounds", "all_pruned", "few_adds"]


def _load(name):
    d = np.load(os.path.join(HERE, "golden", "density.npz"))
    return {k.split("__", 1)[1]: d[k] for k in d.files if k.startswith(name + "__")}


def _cfg(c):
    from paper_2505_19175_b200.density import DensifyConfig
    return DensifyConfig(tau_prune=float(c[0]), min_views=int(c[1]), min_pixels=int(c[2]),
                         opacity_dead=float(c[3]), growth_rate=float(c[4]), tau_small=float(c[5]),
                         max_noise_factor=float(c[6]), interval=int(c[7]), start_iter=int(c[8]),
                         stop_iter=int(c[9]))


def _run(g, dtype):
    from paper_2505_19175_b200 import density as DD
    from paper_2505_19175_b200.rasterizer import DeviceSoup
    from paper_2505_19175_b200.types import TriangleSoup
    soup = DeviceSoup.from_soup(TriangleSoup(vertices=g["v"], opacity=g["o"], sigma=g["s"], sh=g["h"]), dtype=dtype)
    cfg = _cfg(g["cfg"])
    stats = DD.DeviceViewStats.empty(len(g["v"]))
    for k, vid in enumerate(g["view_ids"]):
        stats.update(int(vid), types.SimpleNamespace(per_triangle_max_weight=g["maxw"][k],
                                                     per_triangle_pixel_count=g["pix"][k],
                                                     per_triangle_area=g["area"][k]), cfg.min_pixels)
    new, rep = DD.densify_step(soup, stats, int(g["iteration"]), cfg, np.random.default_rng(int(g["seed"])))
    return new, rep


def _compare(new, rep, g, fp64, label):
    assert bool(rep["scheduled"]) == bool(g["scheduled"]), label
    assert np.array_equal(rep["origin"], g["origin"]), f"{label} origin"
    if g["scheduled"]:
        pr = rep["prune"]
        for i, k in enumerate(("low_weight", "few_views", "dead_opacity")):
            assert pr[k] == np.nonzero(g["prune_mask"][i])[0].tolist(), f"{label} {k}"
        c = g["counts"]
        assert (rep.get("n_add", 0), rep["n_split"], rep["n_clone"], pr["n_removed"]) == tuple(int(x) for x in c), label
    assert rep["n_after"] == len(g["origin"]) if g["scheduled"] else True
    for a, b in ((new.opacity, g["no"]), (new.sigma, g["ns"]), (new.sh, g["nh"])):
        assert np.array_equal(a.double().cpu().numpy(), b), f"{label} copied parameters"
    v = new.vertices.double().cpu().numpy()
    assert v.shape == g["nv"].shape
    if fp64:
        np.testing.assert_allclose(v, g["nv"], rtol=0, atol=1e-12, err_msg=label)
    else:
        np.testing.assert_allclose(v, g["nv"].astype(np.float32).astype(np.float64), rtol=2e-7, atol=1e-7,
                                   err_msg=label)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_densify_matches_reference(name, dtype):
    g = _load(name)
    new, rep = _run(g, torch.float64 if dtype == "f64" else torch.float32)
    _compare(new, rep, g, dtype == "f64", f"{name}/{dtype}")


def test_stats_aggregate_matches_oracle():
    from oracle import density as OD
    from paper_2505_19175_b200 import density as DD
    g = _load("sigma")
    stats = DD.DeviceViewStats.empty(len(g["v"]))
    for k, vid in enumerate(g["view_ids"]):
        stats.update(int(vid), types.SimpleNamespace(per_triangle_max_weight=g["maxw"][k],
                                                     per_triangle_pixel_count=g["pix"][k],
                                                     per_triangle_area=g["area"][k]), 2)
    mw, views, mean_area = OD.aggregate(OD.record_views(g["view_ids"], g["maxw"], g["pix"], g["area"], 2))
    assert stats.n_views == len(set(g["view_ids"].tolist()))
    assert np.array_equal(stats.max_weight().cpu().numpy(), mw)
    assert np.array_equal(stats.covering_views().cpu().numpy(), views)
    assert np.array_equal(stats.mean_area().cpu().numpy(), mean_area)


def test_densify_large_against_oracle():
    # 60k triangles, forward statistics of a real render, both criteria
    from oracle import density as OD
    from paper_2505_19175_b200 import density as DD
    from paper_2505_19175_b200 import scenes
    from paper_2505_19175_b200.rasterizer import DeviceSoup, Rasterizer
    soup = scenes.make_soup(60_000, seed=21, size=0.05, sigma=(0.5, 2.0))
    r = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731
    ds = DeviceSoup.from_soup(soup, dtype=torch.float32)
    rast = Rasterizer()
    stats = DD.DeviceViewStats.empty(len(ds))
    host = []
    for vid, f in enumerate((900.0, 1200.0, 700.0)):
        intr, pose = scenes.frontal_camera(320, 240, f)
        out = rast.forward(ds, intr, pose, keep_backward=False)
        torch.cuda.synchronize()
        stats.update(vid, out, 2)
        host.append((out.max_weight.double().cpu().numpy(), out.pixel_count.cpu().numpy(),
                     out.area.double().cpu().numpy()))
    cfg = DD.DensifyConfig(tau_prune=0.01, min_views=2, tau_small=3.0)
    v, o, s, h = (r(ds.vertices.double().cpu().numpy()), r(ds.opacity.double().cpu().numpy()),
                  r(ds.sigma.double().cpu().numpy()), r(ds.sh.double().cpu().numpy()))
    per_view = OD.record_views(range(3), [x[0] for x in host], [x[1] for x in host], [x[2] for x in host], 2)
    for it in (500, 1000):
        new, rep = DD.densify_step(ds, stats, it, cfg, np.random.default_rng(it))
        ref = OD.densify(v, o, s, h, per_view, it, [getattr(cfg, k) for k in OD.CFG_KEYS],
                         np.random.default_rng(it))
        assert np.array_equal(rep["origin"], ref["origin"]), it
        assert (rep["n_add"], rep["n_split"], rep["n_clone"]) == tuple(ref["counts"][:3]), it
        assert rep["n_split"] > 0 and rep["n_clone"] > 0
        np.testing.assert_allclose(new.vertices.double().cpu().numpy(),
                                   ref["v"].astype(np.float32).astype(np.float64), rtol=2e-7, atol=1e-7)
        assert np.array_equal(new.sh.double().cpu().numpy(), ref["h"])


def test_adam_remap():
    from paper_2505_19175_b200.optim import DeviceAdamState
    n = 37
    st = DeviceAdamState.zeros(n)
    st.m.copy_(torch.randn(59 * n, device="cuda"))
    st.v.copy_(torch.rand(59 * n, device="cuda"))
    st.t = 9
    origin = np.array([3, 0, -1, 36, 5, 5, 5, -1, 12], dtype=np.int64)
    new = st.remap(origin)
    assert new.n == len(origin) and new.t == 9
    for a, b in ((st.m, new.m), (st.v, new.v)):
        a, b = a.cpu().numpy(), b.cpu().numpy()
        o_old = o_new = 0
        for w in (9, 1, 1, 48):
            src = a[o_old:o_old + w * n].reshape(n, w)
            exp = np.where((origin >= 0)[:, None], src[np.maximum(origin, 0)], 0.0)
            assert np.array_equal(b[o_new:o_new + w * len(origin)].reshape(-1, w), exp)
            o_old += w * n
            o_new += w * len(origin)
