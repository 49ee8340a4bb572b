"""Shared fixtures: golden-scene loading and the GPU marker.

Tests marked ``gpu`` run on a B200 (driver: ``pytest -m gpu``); everything
else runs on CPU (``pytest -m "not gpu"``).
"""
from __future__ import annotations

import glob
import hashlib
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")

from paper_2505_19175_b200.types import (CameraIntrinsics, CameraPose,  # noqa: E402
                                         TriangleSoup, WindowMode)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")


def golden_paths():
    return sorted(glob.glob(os.path.join(GOLDEN, "rs_*.npz")))


class GoldenScene:
    def __init__(self, path):
        z = np.load(path, allow_pickle=False)
        self.name = os.path.basename(path)
        self.z = z
        self.soup = TriangleSoup(z["vertices"], z["opacity"], z["sigma"], z["sh"])
        cam = z["cam"]
        w, h = (int(x) for x in z["size"])
        self.intr = CameraIntrinsics(fx=float(cam[0]), fy=float(cam[1]), cx=float(cam[2]),
                                     cy=float(cam[3]), width=w, height=h, z_near=float(cam[4]))
        self.pose = CameraPose(rotation=z["rotation"], translation=z["translation"])
        self.mode = WindowMode.NORMALIZED if int(z["mode"]) == 0 else WindowMode.SIGMOID
        self.background = tuple(float(x) for x in z["background"])
        self.d_image = np.random.default_rng(int(z["d_image_seed"])).normal(size=(h, w, 3))

    def __getitem__(self, k):
        return self.z[k]


@pytest.fixture(params=golden_paths(), ids=lambda p: os.path.basename(p))
def golden_scene(request):
    return GoldenScene(request.param)


def rel_err(got, ref, floor=None):
    """max |got-ref| / max(|ref|) with an absolute floor (fraction of the
    largest reference magnitude) so near-zero sums do not dominate."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    scale = np.abs(ref).max() if ref.size else 0.0
    if scale == 0.0:
        return float(np.abs(got).max()) if got.size else 0.0
    denom = np.maximum(np.abs(ref), (floor if floor is not None else 1e-3) * scale)
    return float((np.abs(got - ref) / denom).max())


def digest(*arrays) -> str:
    """Same digest as tests/golden/make_golden.py."""
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()
