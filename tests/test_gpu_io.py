"""GPU parity of the model I/O drop-ins (scene_io.py in this package, ts_io.cu)
with the reference's files (tests/golden/io/): PLY and OBJ bytes identical,
import_ply arrays identical, reference .npz models load; the reference's error
cases; a 2M-triangle PLY round trip against the oracle's quantisation."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")


def _soup(dtype=torch.float64):
    from paper_2505_19175_b200.rasterizer import DeviceSoup
    from paper_2505_19175_b200.types import TriangleSoup
    g = np.load(os.path.join(GOLD, "soup.npz"))
    return DeviceSoup.from_soup(TriangleSoup(vertices=g["v"], opacity=g["o"], sigma=g["s"], sh=g["h"]), dtype=dtype), g


def test_export_ply_bytes(tmp_path):
    from paper_2505_19175_b200 import scene_io as IO
    ds, _ = _soup()
    p = IO.export_mesh(ds, tmp_path / "mesh.ply")
    assert open(p, "rb").read() == open(os.path.join(GOLD, "mesh.ply"), "rb").read()


def test_export_obj_bytes(tmp_path):
    from paper_2505_19175_b200 import scene_io as IO
    ds, _ = _soup()
    IO.export_mesh(ds, tmp_path / "mesh.obj", "OBJ")
    for f in ("mesh.obj", "mesh.mtl"):
        assert open(tmp_path / f, "rb").read() == open(os.path.join(GOLD, f), "rb").read(), f


def test_unknown_format(tmp_path):
    from paper_2505_19175_b200 import scene_io as IO
    ds, _ = _soup()
    with pytest.raises(ValueError, match="unsupported mesh format"):
        IO.export_mesh(ds, tmp_path / "x.stl", "stl")


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_import_ply(dtype):
    from paper_2505_19175_b200 import scene_io as IO
    _, g = _soup()
    s = IO.import_ply(os.path.join(GOLD, "mesh.ply"), sigma=0.07, dtype=dtype)
    assert s.solid
    cast = (lambda a: a) if dtype == torch.float64 else (lambda a: a.astype(np.float32).astype(np.float64))
    for t, ref in ((s.vertices, g["iv"]), (s.opacity, g["io"]), (s.sigma, g["is_"]), (s.sh, g["ih"])):
        assert np.array_equal(t.double().cpu().numpy(), cast(ref))


def test_import_errors(tmp_path):
    from paper_2505_19175_b200 import scene_io as IO
    raw = open(os.path.join(GOLD, "mesh.ply"), "rb").read()
    hdr_end = raw.index(b"end_header\n") + len(b"end_header\n")
    (tmp_path / "a.ply").write_bytes(b"plx\n" + raw[4:])
    with pytest.raises(ValueError, match="not a PLY file"):
        IO.import_ply(tmp_path / "a.ply")
    (tmp_path / "b.ply").write_bytes(raw[:hdr_end - len(b"end_header\n")])
    with pytest.raises(ValueError, match="unterminated PLY header"):
        IO.import_ply(tmp_path / "b.ply")
    (tmp_path / "c.ply").write_bytes(raw.replace(b"element vertex 72", b"element vertex 71"))
    with pytest.raises(ValueError, match="unshared triangle-soup"):
        IO.import_ply(tmp_path / "c.ply")
    body = bytearray(raw[hdr_end:])
    bad = bytearray(body)
    bad[45 * 24 + 16 * 5:45 * 24 + 16 * 5 + 4] = (4).to_bytes(4, "little")
    (tmp_path / "d.ply").write_bytes(raw[:hdr_end] + bytes(bad))
    with pytest.raises(ValueError, match="non-triangle face"):
        IO.import_ply(tmp_path / "d.ply")
    bad = bytearray(body)
    bad[45 * 24 + 16 * 7 + 8:45 * 24 + 16 * 7 + 12] = (500).to_bytes(4, "little")
    (tmp_path / "e.ply").write_bytes(raw[:hdr_end] + bytes(bad))
    with pytest.raises(IndexError):
        IO.import_ply(tmp_path / "e.ply")


def test_models_interchange(tmp_path):
    from paper_2505_19175_b200 import scene_io as IO
    ds, g = _soup()
    s, views = IO.load_model(os.path.join(GOLD, "model.npz"), dtype=torch.float64)
    assert views is None and not s.solid
    for t, ref in ((s.vertices, g["v"]), (s.opacity, g["o"]), (s.sigma, g["s"]), (s.sh, g["h"])):
        assert np.array_equal(t.cpu().numpy(), ref)
    IO.save_model(tmp_path / "m.npz", ds)
    a, b = np.load(tmp_path / "m.npz"), np.load(os.path.join(GOLD, "model.npz"))
    assert sorted(a.files) == sorted(b.files)
    for k in b.files:
        assert np.array_equal(a[k], b[k]), k


def test_large_round_trip(tmp_path):
    from oracle import scene_io as OI
    from paper_2505_19175_b200 import scene_io as IO
    from paper_2505_19175_b200 import scenes
    from paper_2505_19175_b200.rasterizer import DeviceSoup
    soup = scenes.make_soup(2_000_000, seed=3, size=0.02, sigma=1.0)
    ds = DeviceSoup.from_soup(soup, dtype=torch.float32)
    p = IO.export_mesh(ds, tmp_path / "big.ply")
    raw = open(p, "rb").read()
    n = len(ds)
    hl = len(OI.header(n))
    assert raw[:hl] == OI.header(n) and len(raw) == hl + 61 * n
    rng = np.random.default_rng(0)
    sample = rng.choice(n, 5000, replace=False)
    vb = np.frombuffer(raw[hl:hl + 45 * n], OI.VDT).reshape(n, 3)
    ref = np.frombuffer(OI.pack(soup.vertices[sample], soup.sh[sample])[len(OI.header(len(sample))):
                                                                         len(OI.header(len(sample))) + 45 * len(sample)],
                        OI.VDT).reshape(-1, 3)
    assert np.array_equal(vb[sample], ref)
    back = IO.import_ply(p, sigma=1.0)
    assert np.array_equal(back.vertices.cpu().numpy(), ds.vertices.cpu().numpy())
