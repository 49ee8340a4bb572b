"""Golden fixtures of the reference's model I/O (trisplat/scene_io.py:365-527),
run in the build container:  NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_io_golden.py
A 24-triangle soup (fp64 values, SH DC spanning the clip range) exported as PLY
and OBJ (+ .mtl) by export_mesh, the PLY re-imported by import_ply, and the
soup saved by save_model; the files and the imported arrays are stored under
tests/golden/io/."""
from __future__ import annotations

import importlib
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "io")
sys.path.insert(0, "/root/reference/pkg/src")
IO = importlib.import_module("trisplat.scene_io")
S = importlib.import_module("trisplat.soup")


def main():
    rng = np.random.default_rng(11)
    n = 24
    v = rng.normal(0, 1, (n, 3, 3))
    sh = rng.normal(0, 0.6, (n, 16, 3))
    sh[0, 0] = [-5.0, 5.0, 0.0]  # both clip bounds and mid grey
    soup = S.TriangleSoup(v, rng.uniform(0.05, 0.95, n), rng.uniform(0.1, 3.0, n), sh)
    os.makedirs(OUT, exist_ok=True)
    with tempfile.TemporaryDirectory() as td:
        IO.export_mesh(soup, os.path.join(td, "mesh.ply"), "ply")
        IO.export_mesh(soup, os.path.join(td, "mesh.obj"), "obj")
        IO.save_model(os.path.join(td, "model.npz"), soup)
        for f in ("mesh.ply", "mesh.obj", "mesh.mtl", "model.npz"):
            shutil.copy(os.path.join(td, f), os.path.join(OUT, f))
        back = IO.import_ply(os.path.join(td, "mesh.ply"), sigma=0.07)
    np.savez_compressed(os.path.join(OUT, "soup.npz"), v=v, o=soup.opacity, s=soup.sigma, h=sh,
                        iv=back.vertices, io=back.opacity, is_=back.sigma, ih=back.sh)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
