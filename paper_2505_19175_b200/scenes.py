"""Synthetic benchmark / parity scenes.

All parameters are drawn in fp64 and rounded to fp32, so the fp32 device
copy and the fp64 oracle copy hold identical values.  Camera convention is
the reference's (``synthetic.look_at``, synthetic.py:78-87).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .types import CameraIntrinsics, CameraPose, TriangleSoup


@dataclass(frozen=True)
class SceneConfig:
    name: str
    n: int
    seed: int
    size: float
    sigma: float | tuple  # constant, or (lo, hi) uniform range
    width: int
    height: int
    f: float
    sh_degree: int = 3


CONFIGS = {
    # configs[0]: 10k, 128x128, fwd+bwd vs CPU reference
    "c1": SceneConfig("c1", 10_000, 1, 0.17, (0.5, 5.0), 128, 128, 140.8),
    # configs[1]: 500k, 1280x720, forward only
    "c2": SceneConfig("c2", 500_000, 3, 0.02, 1.0, 1280, 720, 1100.0),
    # north-star headline: 2M, 1280x720, forward
    "ns": SceneConfig("ns", 2_000_000, 3, 0.02, 1.0, 1280, 720, 1100.0),
    # configs[2]: 2M, 1297x840, fwd+bwd training step
    "c3": SceneConfig("c3", 2_000_000, 3, 0.02, 1.0, 1297, 840, 1150.0),
    # configs[4]: 5M, 1920x1080, sharp window
    "c5": SceneConfig("c5", 5_000_000, 3, 0.02, 0.1, 1920, 1080, 2100.0),
}


def make_soup(n: int, seed: int, size: float, sigma, dtype=np.float32) -> TriangleSoup:
    """centers ~ U(-2,2)^3, verts = centers + size*N(0,1), opacity ~ U(0.1,0.9),
    sigma constant or U(lo,hi), sh ~ N(0,0.3); rounded to fp32."""
    rng = np.random.default_rng(seed)
    centers = rng.uniform(-2.0, 2.0, (n, 1, 3))
    verts = centers + size * rng.normal(size=(n, 3, 3))
    opacity = rng.uniform(0.1, 0.9, n)
    if isinstance(sigma, tuple):
        sig = rng.uniform(sigma[0], sigma[1], n)
    else:
        sig = np.full(n, float(sigma))
    sh = rng.normal(0.0, 0.3, (n, 16, 3))
    r = lambda a: np.asarray(a, dtype=dtype).astype(np.float64)  # noqa: E731
    return TriangleSoup(vertices=r(verts), opacity=r(opacity), sigma=r(sig), sh=r(sh))


def frontal_camera(width: int, height: int, f: float):
    intr = CameraIntrinsics(fx=f, fy=f, cx=width / 2.0, cy=height / 2.0, width=width,
                            height=height)
    pose = CameraPose(rotation=np.eye(3), translation=np.array([0.0, 0.0, 6.0]))
    return intr, pose


def make_scene(cfg: SceneConfig | str):
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    soup = make_soup(cfg.n, cfg.seed, cfg.size, cfg.sigma)
    intr, pose = frontal_camera(cfg.width, cfg.height, cfg.f)
    return soup, intr, pose


def make_d_image(seed: int, height: int, width: int, fp32: bool = False) -> np.ndarray:
    """Upstream image gradient N(0,1); ``fp32=True`` rounds it to fp32 values
    (held in fp64) so the device's fp32 d_image and the fp64 oracle see the
    same numbers, as the scene parameters do."""
    d = np.random.default_rng(seed + 100).normal(size=(height, width, 3))
    return d.astype(np.float32).astype(np.float64) if fp32 else d


def look_at(center, target) -> CameraPose:
    """synthetic.py:78-87: +z toward the target, y-down."""
    center = np.asarray(center, dtype=np.float64)
    target = np.asarray(target, dtype=np.float64)
    z = target - center
    z = z / np.linalg.norm(z)
    up = np.array([0.0, -1.0, 0.0])
    x = np.cross(up, z)
    x = x / np.linalg.norm(x)
    y = np.cross(z, x)
    r = np.stack([x, y, z])
    return CameraPose(rotation=r, translation=-r @ center)


def orbit_cameras(n_views: int, seed: int = 4, radius: float = 6.0):
    """C4: eye = r*(cos el cos az, sin el, cos el sin az), az~U(0,2pi),
    el~U(-0.5,0.5), looking at the origin."""
    rng = np.random.default_rng(seed)
    az = rng.uniform(0.0, 2 * np.pi, n_views)
    el = rng.uniform(-0.5, 0.5, n_views)
    poses = []
    for a, e in zip(az, el):
        eye = radius * np.array([np.cos(e) * np.cos(a), np.sin(e), np.cos(e) * np.sin(a)])
        poses.append(look_at(eye, np.zeros(3)))
    return poses
