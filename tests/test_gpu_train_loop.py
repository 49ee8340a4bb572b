"""The device-resident training iteration of INTEGRATION.md (the reference's
training.py:121-231 composed from the drop-ins): forward, photometric loss,
backward, fused Adam, view statistics, a density step with the moment remap,
and model export -- the loss decreases over a few iterations on a fixed
target and every size stays consistent through the density step."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_device_training_loop(tmp_path):
    from paper_2505_19175_b200 import DeviceSoup, Rasterizer, density, losses, optim, scene_io, scenes
    r = Rasterizer()
    soup = DeviceSoup.from_soup(scenes.make_soup(3000, seed=7, size=0.15, sigma=(0.5, 3.0)), dtype=torch.float32)
    intr, _ = scenes.frontal_camera(96, 80, 110.0)
    poses = scenes.orbit_cameras(3, seed=4)
    gen = torch.Generator("cuda").manual_seed(0)
    targets = [torch.rand((80, 96, 3), device="cuda", generator=gen) * 0.2 + 0.4 for _ in poses]
    lrs = {"vertices": 1e-3, "opacity": 0.02, "sigma": 0.01, "sh": 0.02}
    cfg = density.DensifyConfig(tau_prune=1e-4, min_views=1, start_iter=6, interval=6, growth_rate=0.1,
                                tau_small=20.0)
    state = optim.DeviceAdamState.zeros(len(soup))
    stats = density.DeviceViewStats.empty(len(soup))
    rng = np.random.default_rng(3)
    first = last = None
    for it in range(12):
        v = it % len(poses)
        f = r.forward(soup, intr, poses[v])
        loss, d_img = losses.photometric_loss(f.image, targets[v], 0.2, rasterizer=r)
        if v == 0:
            first = loss if first is None else first
            last = loss
        g = r.backward(d_img)
        optim.adam_step(soup, g, state, lrs, rasterizer=r)
        stats.update(v, f, cfg.min_pixels)
        if it + 1 == 6:
            n0 = len(soup)
            soup, rep = density.densify_step(soup, stats, it + 1, cfg, rng, rasterizer=r)
            assert rep["scheduled"] and rep["n_after"] == len(soup) == len(rep["origin"])
            alive = n0 - rep["prune"]["n_removed"]
            assert rep["n_after"] == alive + 3 * rep["n_split"] + rep["n_clone"]
            state = state.remap(rep["origin"])
            assert state.n == len(soup) and state.m.numel() == 59 * len(soup)
            stats = density.DeviceViewStats.empty(len(soup))
    assert last < first, (first, last)
    scene_io.save_model(tmp_path / "m.npz", soup)
    back, views = scene_io.load_model(tmp_path / "m.npz")
    assert views is None and torch.equal(back.vertices, soup.vertices)


def test_chunked_backward_matches_backward():
    """ts_backward_chunked (the chain in triangle ranges, an event after each:
    the all-reduce overlap of the view-parallel step) gives the same gradient
    as ts_backward, accumulating or not, and fires every event."""
    from paper_2505_19175_b200 import parallel, scenes
    from paper_2505_19175_b200.rasterizer import DeviceGrads, DeviceSoup, Rasterizer
    rast = Rasterizer()
    soup = scenes.make_soup(5000, seed=21, size=0.1, sigma=(0.5, 3.0))
    intr, pose = scenes.frontal_camera(96, 80, 110.0)
    ds = DeviceSoup.from_soup(soup, dtype=torch.float32)
    d = torch.randn((80, 96, 3), device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    rast.forward(ds, intr, pose)
    ref = rast.backward(d)
    for k in (1, 3, 8):
        b = parallel.chunk_bounds(len(ds), k)
        ev = [torch.cuda.Event() for _ in range(k)]
        g = DeviceGrads.zeros(len(ds))
        rast.forward(ds, intr, pose)
        rast.backward(d, g, chunks=(b, ev))
        torch.cuda.synchronize()
        assert all(e.query() for e in ev)
        assert torch.equal(g.flat, ref.flat), k
        rast.forward(ds, intr, pose)
        rast.backward(d, g, accumulate=True, chunks=(b, ev))
        assert torch.allclose(g.flat, 2 * ref.flat, rtol=1e-6, atol=1e-12)


def test_reserve_then_no_allocation():
    """ts_reserve sizes the per-frame buffers up front (two-phase allocation):
    a training forward + backward of that size allocates nothing more, and the
    results equal those of a context that grew on demand."""
    from paper_2505_19175_b200 import DeviceSoup, Rasterizer, scenes
    soup = DeviceSoup.from_soup(scenes.make_soup(200_000, seed=3, size=0.02, sigma=(1.0, 1.0)), dtype=torch.float32)
    intr, pose = scenes.frontal_camera(640, 360, 550.0)
    d_img = torch.randn((360, 640, 3), device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    grow = Rasterizer()
    f0 = grow.forward(soup, intr, pose, keep_backward=True)
    g0 = grow.backward(d_img)
    r = Rasterizer()
    b = r.reserve(len(soup), 640, 360, entries=f0.n_entries, keep_backward=True)
    assert b > 0 and b == r.workspace_bytes()
    f1 = r.forward(soup, intr, pose, keep_backward=True)
    g1 = r.backward(d_img)
    torch.cuda.synchronize()
    assert r.workspace_bytes() == b
    assert torch.equal(f0.image, f1.image) and torch.equal(f0.pixel_count, f1.pixel_count)
    # (fp64 atomics: the summation order, and so the last bits, may differ between runs)
    torch.testing.assert_close(g1.flat, g0.flat, rtol=1e-6, atol=1e-6 * float(g0.flat.abs().max()))
