"""GPU parity of the fragment-collection path: render(collect_fragments=True)
(render.py:383-399, 420-425; _kernels.py:107-116, 135-178) against the
reference's own fragment lists stored in the golden fixtures, and
render_backward(frag_grads=...) (backward.py:122-142; _kernels.py:262-272)
against the oracle.  Bar: offsets and triangle ids bit-exact, depths exact,
weights within 1e-9, gradients within 1e-4 relative."""
import numpy as np
import pytest

from conftest import golden_paths, GoldenScene, rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GRAD_RTOL = 1e-4


@pytest.fixture(scope="module")
def rast():
    from paper_2505_19175_b200.rasterizer import Rasterizer
    return Rasterizer()


def _dev(soup):
    from paper_2505_19175_b200.rasterizer import DeviceSoup
    return DeviceSoup.from_soup(soup, dtype=torch.float64 if np.asarray(soup.vertices).dtype == np.float64
                                else torch.float32)


def _fg(offsets, seed):
    rng = np.random.default_rng(seed)
    f = int(offsets[-1])
    return offsets, rng.normal(size=f), rng.normal(size=f) * 0.1


@pytest.mark.parametrize("path", golden_paths(), ids=lambda p: p.split("/")[-1])
def test_golden_fragment_lists(rast, path):
    g = GoldenScene(path)
    rast.forward(_dev(g.soup), g.intr, g.pose, mode=g.mode, background=g.background)
    fr = rast.fragments().to_fragment_data()
    assert np.array_equal(fr.offsets, g["frag_offsets"])
    assert np.array_equal(fr.triangle, g["frag_triangle"])
    assert np.array_equal(fr.depth, g["frag_depth"])
    assert np.abs(fr.weight - g["frag_weight"]).max(initial=0.0) <= 1e-9


def _weights(rast, backward):
    """The stream backward takes the fragments' weights of the same forward."""
    return rast.fragments().weight if backward == "stream" else None


@pytest.mark.parametrize("backward", ["tile", "stream"])
@pytest.mark.parametrize("path", golden_paths()[:6], ids=lambda p: p.split("/")[-1])
def test_golden_fragment_gradients(rast, path, backward):
    from oracle import oracle as O
    g = GoldenScene(path)
    rast.forward(_dev(g.soup), g.intr, g.pose, mode=g.mode, background=g.background)
    off, dw, dz = _fg(g["frag_offsets"], 7)
    gr = rast.backward_fragments(torch.as_tensor(g.d_image, dtype=torch.float32, device="cuda"),
                                 torch.from_numpy(off), torch.from_numpy(dw), torch.from_numpy(dz),
                                 weight=_weights(rast, backward))
    ref = O.render_backward(g.soup, g.intr, g.pose, mode=g.mode, background=g.background,
                            d_image=g.d_image, frag_grads=(off, dw, dz))
    for k in ("d_vertices", "d_opacity", "d_sigma", "d_sh"):
        err = rel_err(getattr(gr, k).double().cpu().numpy(), getattr(ref, k))
        assert err < GRAD_RTOL, f"{g.name} {k} rel err {err}"


@pytest.mark.parametrize("backward", ["tile", "stream"])
@pytest.mark.parametrize("mode", ["normalized", "sigmoid"])
def test_mid_scene_fragments_and_gradients(rast, mode, backward):
    from oracle import oracle as O
    from paper_2505_19175_b200 import scenes
    soup = scenes.make_soup(20000, seed=5, size=0.08, sigma=(0.5, 3.0))
    intr, pose = scenes.frontal_camera(192, 144, 200.0)
    rast.forward(_dev(soup), intr, pose, mode=mode)
    fr = rast.fragments().to_fragment_data()
    ref = O.render(soup, intr, pose, mode=mode, collect_fragments=True)
    assert np.array_equal(fr.offsets, ref.fragments.offsets)
    assert np.array_equal(fr.triangle, ref.fragments.triangle)
    assert np.array_equal(fr.depth, ref.fragments.depth)
    assert np.abs(fr.weight - ref.fragments.weight).max(initial=0.0) <= 1e-9
    d_image = scenes.make_d_image(5, intr.height, intr.width)
    off, dw, dz = _fg(fr.offsets, 9)
    gr = rast.backward_fragments(torch.as_tensor(d_image, dtype=torch.float32, device="cuda"),
                                 torch.from_numpy(off), torch.from_numpy(dw), torch.from_numpy(dz),
                                 weight=_weights(rast, backward))
    gref = O.render_backward(soup, intr, pose, mode=mode, d_image=d_image, frag_grads=(off, dw, dz))
    for k in ("d_vertices", "d_opacity", "d_sigma", "d_sh"):
        err = rel_err(getattr(gr, k).double().cpu().numpy(), getattr(gref, k))
        assert err < GRAD_RTOL, f"{mode} {k} rel err {err}"


def test_drop_in_collect_and_frag_grads(rast):
    """The reference's Python surface: FragmentData out of render(), frag_grads
    into render_backward(), and its layout error (backward.py:134-136)."""
    from oracle import oracle as O
    from paper_2505_19175_b200 import rasterizer as R
    from paper_2505_19175_b200 import scenes
    soup = scenes.make_soup(3000, seed=11, size=0.15, sigma=(0.5, 4.0))
    intr, pose = scenes.frontal_camera(96, 80, 110.0)
    out = R.render(soup, intr, pose, collect_fragments=True)
    ref = O.render(soup, intr, pose, collect_fragments=True)
    assert out.fragments.count() == len(ref.fragments.triangle)
    assert np.array_equal(out.fragments.triangle, ref.fragments.triangle)
    d_image = scenes.make_d_image(11, intr.height, intr.width)
    fg = _fg(out.fragments.offsets, 3)
    gs = R.render_backward(soup, intr, pose, d_image=d_image, frag_grads=fg)
    gref = O.render_backward(soup, intr, pose, d_image=d_image, frag_grads=fg)
    assert rel_err(gs.d_vertices, gref.d_vertices) < GRAD_RTOL
    bad = fg[0].copy()
    bad[5:] += 1
    with pytest.raises(ValueError, match="fragment gradients do not match this scene/camera"):
        R.render_backward(soup, intr, pose, d_image=d_image, frag_grads=(bad, fg[1], fg[2]))
    with pytest.raises(ValueError, match="fragment gradients do not match this scene/camera"):
        R.render_backward(soup, intr, pose, d_image=d_image, frag_grads=(fg[0], fg[1][:-1], fg[2]))
