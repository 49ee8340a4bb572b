"""install() rebinds every name the reference's callers import by value
(training.py:12,19, synthetic.py:14, cli.py:21, backward.py:16-17,
render.py's own project_scene / build_tile_lists) -- checked against the live
reference package in the build container (skipped where it is absent, e.g.
on the GPU box).  CPU only: nothing is rendered."""
import importlib
import os
import sys

import pytest

REF_SRC = "/root/reference/pkg/src"


@pytest.fixture()
def trisplat_modules():
    if not os.path.isdir(os.path.join(REF_SRC, "trisplat")):
        pytest.skip("reference package not present")
    sys.path.insert(0, REF_SRC)
    names = ["trisplat", "trisplat.render", "trisplat.backward", "trisplat.training", "trisplat.synthetic",
             "trisplat.cli"]
    try:
        mods = {n: importlib.import_module(n) for n in names}
    except Exception as ex:  # numba / PIL missing
        sys.path.remove(REF_SRC)
        pytest.skip(f"reference not importable: {ex}")
    saved = {(n, a): getattr(m, a) for n, m in mods.items()
             for a in ("render", "render_backward", "project_scene", "build_tile_lists") if hasattr(m, a)}
    yield mods
    for (n, a), v in saved.items():
        setattr(mods[n], a, v)
    sys.path.remove(REF_SRC)


def test_install_rebinds_reference_callers(trisplat_modules):
    from paper_2505_19175_b200 import rasterizer as R
    patched = set(R.install())
    want = {"trisplat.training.render", "trisplat.training.render_backward", "trisplat.synthetic.render",
            "trisplat.cli.render", "trisplat.backward.render", "trisplat.backward.render_backward",
            "trisplat.backward.project_scene", "trisplat.backward.build_tile_lists", "trisplat.render.render",
            "trisplat.render.project_scene", "trisplat.render.build_tile_lists", "trisplat.render",
            "trisplat.render_backward"}
    assert want <= patched, sorted(want - patched)
    m = trisplat_modules
    assert m["trisplat.training"].render is R.render
    assert m["trisplat.training"].render_backward is R.render_backward
    assert m["trisplat.synthetic"].render is R.render
    assert m["trisplat.cli"].render is R.render
    assert m["trisplat.backward"].project_scene is R.project_scene
    assert m["trisplat.backward"].build_tile_lists is R.build_tile_lists
    assert m["trisplat.render"].build_tile_lists is R.build_tile_lists
