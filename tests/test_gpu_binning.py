"""GPU parity of the tile-first binning (ts_bin.cu) in its corner cases:
equal depths (one run of equal keys per tile), clustered depths (long runs
of distinct keys that share a range-reduced key), tiles longer than the
tile sort's register / shared-memory staging (2048 / 8192 entries; the
global-scratch path beyond), and the legacy
global-sort binning on the same scenes.  Tile lists, last contributors and
images must equal the oracle's (render.py:275-361 order: np.lexsort((idx, z))
then stable by tile)."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _soup(n, seed, z_of, spread=0.25, size=0.03):
    from paper_2505_19175_b200.types import TriangleSoup
    rng = np.random.default_rng(seed)
    c = np.zeros((n, 1, 3))
    c[:, 0, :2] = rng.uniform(-spread, spread, (n, 2))
    v = c + size * rng.normal(size=(n, 3, 3))
    v[:, :, 2] = z_of(rng, n)[:, None]  # every vertex of a triangle at its depth
    r = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731
    return TriangleSoup(vertices=r(v), opacity=r(rng.uniform(0.05, 0.3, n)), sigma=r(np.full(n, 1.0)),
                        sh=r(rng.normal(0, 0.3, (n, 16, 3))))


def _check(rast, soup, intr, pose, label, precision="fast"):
    from oracle import oracle as O
    from paper_2505_19175_b200.rasterizer import DeviceSoup
    ds = DeviceSoup.from_soup(soup, dtype=torch.float32)
    f = rast.forward(ds, intr, pose, precision=precision, keep_backward=False, debug=True)
    ref = O.render(soup, intr, pose)
    ntiles = ((intr.width + 15) // 16) * ((intr.height + 15) // 16)
    ts = rast.dump_tile_start(ntiles)
    assert np.array_equal(ts, ref.tile_start), f"{label} tile_start"
    assert np.array_equal(rast.dump_entry_rank(f.n_entries), ref.entry_tri), f"{label} tile lists"
    assert np.array_equal(rast.dump_sorted_idx(f.n_visible), ref.proj.sorted_idx), f"{label} sort order"
    assert np.array_equal(f.last_src.cpu().numpy(), ref.last_src), f"{label} last contributor"
    err = np.abs(f.image.double().cpu().numpy() - ref.image).max()
    assert err <= 1e-5, f"{label} rgb {err}"
    return int(np.diff(ts).max())


@pytest.fixture(scope="module")
def rast():
    from paper_2505_19175_b200.rasterizer import Rasterizer
    return Rasterizer()


def _cam(w=48, h=48, f=90.0):
    from paper_2505_19175_b200 import scenes
    return scenes.frontal_camera(w, h, f)


def test_equal_depths_long_runs(rast):
    # all centroids at exactly the same camera depth: the whole tile is one run
    soup = _soup(3000, 1, lambda rng, n: np.zeros(n))
    intr, pose = _cam()
    longest = _check(rast, soup, intr, pose, "equal")
    assert longest > 64


def test_clustered_depths_with_outlier(rast):
    # depths within 1e-6 of each other plus a far outlier: distinct keys that
    # collide after the 16-bit range reduction
    def z(rng, n):
        d = 1e-6 * rng.uniform(0, 1, n)
        d[0] = -3.0
        return d
    soup = _soup(3000, 2, z)
    intr, pose = _cam()
    _check(rast, soup, intr, pose, "clustered")


def test_tiles_longer_than_shared_memory(rast):
    # > 2048 entries per tile: the tile sort runs on global scratch
    soup = _soup(9000, 3, lambda rng, n: rng.uniform(-1, 1, n), spread=0.08, size=0.02)
    intr, pose = _cam(32, 32, 90.0)
    longest = _check(rast, soup, intr, pose, "long tiles")
    assert longest > 2048


def test_tiles_longer_than_staging(rast):
    # > 8192 entries per tile: the stable LSD path on global scratch
    soup = _soup(24000, 5, lambda rng, n: rng.uniform(-1, 1, n), spread=0.08, size=0.02)
    intr, pose = _cam(32, 32, 90.0)
    longest = _check(rast, soup, intr, pose, "very long tiles")
    assert longest > 8192


def test_long_tiles_with_equal_depths(rast):
    soup = _soup(7000, 4, lambda rng, n: np.round(rng.uniform(-1, 1, n), 1), spread=0.08, size=0.02)
    intr, pose = _cam(32, 32, 90.0)
    longest = _check(rast, soup, intr, pose, "long tiles, ties")
    assert longest > 2048


def test_legacy_binning_matches():
    # TS_BIN_LEGACY (global depth sort + stable tile sort) on the same scenes, in a
    # fresh process (the switch is read once per process)
    code = (
        "import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import test_gpu_binning as T\n"
        "from paper_2505_19175_b200.rasterizer import Rasterizer\n"
        "import numpy as np\n"
        "r = Rasterizer()\n"
        "T._check(r, T._soup(3000, 1, lambda rng, n: np.zeros(n)), *T._cam(), 'legacy equal')\n"
        "T._check(r, T._soup(9000, 3, lambda rng, n: rng.uniform(-1, 1, n), spread=0.08, size=0.02),"
        " *T._cam(32, 32, 90.0), 'legacy long')\n"
        "print('ok')\n" % (ROOT, HERE))
    env = dict(os.environ, TS_BIN_LEGACY="1")
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and "ok" in p.stdout, p.stdout[-2000:] + p.stderr[-2000:]


def test_many_tiles_uses_tile_ranges(rast):
    # 3840x2160 = 32400 tiles: the chunk x tile counting runs in several
    # shared-memory tile ranges (12288 tiles each)
    from paper_2505_19175_b200 import scenes
    soup = scenes.make_soup(60_000, seed=9, size=0.03, sigma=(0.5, 2.0))
    intr, pose = scenes.frontal_camera(3840, 2160, 3300.0)
    longest = _check(rast, soup, intr, pose, "4k")
    assert longest > 0
