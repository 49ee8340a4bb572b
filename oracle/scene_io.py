"""CPU restatement of the reference's binary PLY body (TEST INFRASTRUCTURE:
only tests/, __graft_entry__.smoke() and bench.py's CPU legs may use it).

Follows trisplat/scene_io.py:
  _quantize / soup_colors  :356-363  floor(clip(C0 sh0 + 0.5, 0, 1) * 255 + 0.5)
  _export_ply              :382-414  header, 3N 15-byte vertex records, N faces
  import_ply               :417-455  positions by face index, DC from vertex 0
in numpy.  Pinned to the live reference by tests/golden/io/ (make_io_golden.py).
"""
from __future__ import annotations

import numpy as np

C0 = 0.28209479177387814
VDT = np.dtype([("x", "<f4"), ("y", "<f4"), ("z", "<f4"), ("r", "u1"), ("g", "u1"), ("b", "u1")])
FDT = np.dtype([("c", "<i4"), ("a", "<i4"), ("b", "<i4"), ("d", "<i4")])


def header(n: int) -> bytes:
    props = "".join(f"property float {a}\n" for a in "xyz") + "".join(
        f"property uchar {c}\n" for c in ("red", "green", "blue"))
    return (f"ply\nformat binary_little_endian 1.0\nelement vertex {3 * n}\n{props}"
            f"element face {n}\nproperty list int int vertex_indices\nend_header\n").encode("ascii")


def quantise(sh0: np.ndarray) -> np.ndarray:
    c = np.clip(C0 * np.asarray(sh0, np.float64) + 0.5, 0.0, 1.0)
    return np.floor(c * 255.0 + 0.5).astype(np.uint8)


def pack(vertices, sh) -> bytes:
    v = np.asarray(vertices, np.float64).reshape(-1, 3, 3)
    n = len(v)
    rec = np.zeros(3 * n, VDT)
    p = v.reshape(-1, 3).astype(np.float32)
    rec["x"], rec["y"], rec["z"] = p[:, 0], p[:, 1], p[:, 2]
    q = np.repeat(quantise(np.asarray(sh)[:, 0, :]), 3, axis=0)
    rec["r"], rec["g"], rec["b"] = q[:, 0], q[:, 1], q[:, 2]
    f = np.zeros(n, FDT)
    f["c"] = 3
    f["a"], f["b"], f["d"] = 3 * np.arange(n), 3 * np.arange(n) + 1, 3 * np.arange(n) + 2
    return header(n) + rec.tobytes() + f.tobytes()


def unpack(body_vertices: bytes, body_faces: bytes, sigma: float):
    rec = np.frombuffer(body_vertices, VDT)
    f = np.frombuffer(body_faces, FDT)
    idx = np.stack([f["a"], f["b"], f["d"]], axis=1)
    pos = np.stack([rec["x"], rec["y"], rec["z"]], axis=1).astype(np.float64)
    rgb = np.stack([rec["r"], rec["g"], rec["b"]], axis=1)[idx[:, 0]].astype(np.float64) / 255.0
    sh = np.zeros((len(f), 16, 3))
    sh[:, 0] = (rgb - 0.5) / C0
    return pos[idx], np.ones(len(f)), np.full(len(f), sigma), sh
