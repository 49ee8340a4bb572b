"""The PLY oracle (oracle/scene_io.py) against the reference's export_mesh /
import_ply files and arrays (tests/golden/io/): bytes and values exact."""
import os

import numpy as np

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")


def test_pack_matches_reference_file():
    from oracle import scene_io as OI
    g = np.load(os.path.join(GOLD, "soup.npz"))
    ref = open(os.path.join(GOLD, "mesh.ply"), "rb").read()
    assert OI.pack(g["v"], g["h"]) == ref


def test_unpack_matches_reference_import():
    from oracle import scene_io as OI
    g = np.load(os.path.join(GOLD, "soup.npz"))
    n = len(g["v"])
    raw = open(os.path.join(GOLD, "mesh.ply"), "rb").read()
    body = raw[len(OI.header(n)):]
    v, o, s, h = OI.unpack(body[:45 * n], body[45 * n:], 0.07)
    assert np.array_equal(v, g["iv"]) and np.array_equal(o, g["io"])
    assert np.array_equal(s, g["is_"]) and np.array_equal(h, g["ih"])
