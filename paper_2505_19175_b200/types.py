"""Host-side data types mirroring the reference package's public surface.

Each class restates the reference type of the same name (same fields, same
validation and error messages), so code written against ``trisplat`` runs
unchanged against this package.  The renderer itself duck-types its inputs:
a reference ``trisplat.TriangleSoup`` / ``CameraIntrinsics`` / ``CameraPose``
is accepted just as well as these.

  WindowMode, CameraIntrinsics, CameraPose, Triangle3D   geometry.py:25-99
  TriangleSoup, PARAMS_PER_TRIANGLE                      soup.py:14-77
  ImageBuffer, FragmentData, RenderOutput                render.py:46-91
  GradientSet                                            backward.py:24-56
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

PARAMS_PER_TRIANGLE = 59  # 9 vertex coords + opacity + sigma + 48 SH (soup.py:14)
DEGENERATE_AREA = 1e-8       # geometry.py:18
DEGENERATE_INRADIUS = 1e-6   # geometry.py:19
DEFAULT_TAU_CUTOFF = 1.0 / 255.0  # geometry.py:22
DEFAULT_TILE_SIZE = 16       # render.py:26
TAU_CONTRIB = 1.0 / 255.0    # render.py:27


class WindowMode(Enum):
    NORMALIZED = "normalized"
    SIGMOID = "sigmoid"


def mode_flag(mode) -> int:
    """0 = NORMALIZED, 1 = SIGMOID; accepts this enum, the reference enum,
    its string value or the integer flag."""
    if isinstance(mode, (int, np.integer)):
        return int(mode)
    val = getattr(mode, "value", mode)
    return 0 if str(val).lower() == "normalized" else 1


@dataclass(frozen=True)
class CameraIntrinsics:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    z_near: float = 0.01

    def __post_init__(self):
        if not (self.fx > 0 and self.fy > 0):
            raise ValueError("focal lengths must be positive")
        if self.width < 1 or self.height < 1:
            raise ValueError("image size must be at least 1x1")
        if not self.z_near > 0:
            raise ValueError("z_near must be positive")


@dataclass(frozen=True)
class CameraPose:
    """World-to-camera rigid transform: x_cam = R @ x_world + t."""

    rotation: np.ndarray
    translation: np.ndarray

    def __post_init__(self):
        r = np.asarray(self.rotation, dtype=np.float64)
        t = np.asarray(self.translation, dtype=np.float64).reshape(3)
        if r.shape != (3, 3):
            raise ValueError("rotation must be 3x3")
        if not np.allclose(r.T @ r, np.eye(3), atol=1e-9):
            raise ValueError("rotation is not orthonormal")
        if abs(np.linalg.det(r) - 1.0) > 1e-9:
            raise ValueError("rotation must have determinant +1")
        object.__setattr__(self, "rotation", r)
        object.__setattr__(self, "translation", t)

    def camera_center(self) -> np.ndarray:
        return -self.rotation.T @ self.translation


@dataclass
class Triangle3D:
    vertices: np.ndarray
    opacity: float
    sigma: float
    sh: np.ndarray

    def __post_init__(self):
        self.vertices = np.asarray(self.vertices, dtype=np.float64).reshape(3, 3)
        self.sh = np.asarray(self.sh, dtype=np.float64).reshape(16, 3)
        if not 0.0 < self.opacity < 1.0:
            raise ValueError(f"opacity must be in (0,1), got {self.opacity}")
        if not self.sigma > 0:
            raise ValueError(f"sigma must be positive, got {self.sigma}")


@dataclass
class TriangleSoup:
    vertices: np.ndarray  # (N,3,3)
    opacity: np.ndarray   # (N,)
    sigma: np.ndarray     # (N,)
    sh: np.ndarray        # (N,16,3)
    solid: bool = False

    def __post_init__(self):
        self.vertices = np.ascontiguousarray(self.vertices, dtype=np.float64).reshape(-1, 3, 3)
        n = len(self.vertices)
        self.opacity = np.ascontiguousarray(self.opacity, dtype=np.float64).reshape(n)
        self.sigma = np.ascontiguousarray(self.sigma, dtype=np.float64).reshape(n)
        self.sh = np.ascontiguousarray(self.sh, dtype=np.float64).reshape(n, 16, 3)

    def __len__(self) -> int:
        return len(self.vertices)

    @classmethod
    def empty(cls) -> "TriangleSoup":
        return cls(np.zeros((0, 3, 3)), np.zeros(0), np.zeros(0), np.zeros((0, 16, 3)))

    @classmethod
    def from_triangles(cls, triangles) -> "TriangleSoup":
        tris = list(triangles)
        if not tris:
            return cls.empty()
        return cls(vertices=np.stack([t.vertices for t in tris]),
                   opacity=np.array([t.opacity for t in tris]),
                   sigma=np.array([t.sigma for t in tris]),
                   sh=np.stack([t.sh for t in tris]))

    def copy(self) -> "TriangleSoup":
        return TriangleSoup(self.vertices.copy(), self.opacity.copy(), self.sigma.copy(),
                            self.sh.copy(), solid=self.solid)

    def validate_finite(self):
        validate_finite(self)


def as_soup(triangles):
    """soup.py:80-83: a soup-like object passes through, an iterable of
    Triangle3D-likes is stacked."""
    if hasattr(triangles, "vertices") and hasattr(triangles, "sh") and not isinstance(
            triangles, (list, tuple)):
        return triangles
    return TriangleSoup.from_triangles(triangles)


def validate_finite(soup):
    """soup.py:67-77: raise naming the first offending triangle, groups in the
    order vertices, opacity, sigma, sh."""
    n = len(soup.vertices)
    if n == 0:
        return
    for name, arr in (("vertices", soup.vertices), ("opacity", soup.opacity),
                      ("sigma", soup.sigma), ("sh", soup.sh)):
        flat = np.asarray(arr).reshape(n, -1)
        bad = ~np.isfinite(flat).all(axis=1)
        if bad.any():
            raise ValueError(f"non-finite {name} in triangle {int(np.nonzero(bad)[0][0])}")


@dataclass
class ImageBuffer:
    rgb: np.ndarray

    def __post_init__(self):
        self.rgb = np.asarray(self.rgb, dtype=np.float64)
        if self.rgb.ndim != 3 or self.rgb.shape[2] != 3:
            raise ValueError("image must be HxWx3")
        if not np.isfinite(self.rgb).all():
            raise ValueError("image contains non-finite values")

    @classmethod
    def trusted(cls, rgb: np.ndarray) -> "ImageBuffer":
        """An (H, W, 3) fp64 image the device produced clipped to [0, 1] (fmin /
        fmax return the non-NaN operand, so it is finite by construction): the
        same object without the O(HW) validation pass."""
        buf = cls.__new__(cls)
        buf.rgb = rgb
        return buf

    @property
    def height(self) -> int:
        return self.rgb.shape[0]

    @property
    def width(self) -> int:
        return self.rgb.shape[1]


@dataclass
class FragmentData:
    offsets: np.ndarray
    triangle: np.ndarray
    weight: np.ndarray
    depth: np.ndarray

    def count(self) -> int:
        return len(self.triangle)


@dataclass
class SceneProjection:
    """project_scene's result (render.py:128-156): depth-sorted screen-space data
    of the accepted triangles of one view (M of them), fp64 / int64."""

    n_total: int
    sorted_idx: np.ndarray  # (M,) source indices, depth order
    z: np.ndarray           # (M,) sort depth
    xc: np.ndarray          # (M,3,3) camera-space vertices
    q: np.ndarray           # (M,3,2)
    nrm: np.ndarray         # (M,3,2)
    doff: np.ndarray        # (M,3)
    esign: np.ndarray       # (M,3)
    phis: np.ndarray        # (M,)
    area: np.ndarray        # (M,)
    sig: np.ndarray
    opa: np.ndarray
    rgb: np.ndarray         # (M,3) clamped
    raw_rgb: np.ndarray     # (M,3) pre-clamp
    basis: np.ndarray       # (M,16)
    viewdir: np.ndarray     # (M,3) unit
    u_norm: np.ndarray      # (M,)
    bbox: np.ndarray        # (M,4) int64: x0,x1,y0,y1
    area_full: np.ndarray   # (N,) projected area for every source triangle


@dataclass
class RenderOutput:
    image: ImageBuffer
    alpha_map: np.ndarray
    per_triangle_max_weight: np.ndarray
    per_triangle_pixel_count: np.ndarray
    per_triangle_area: np.ndarray
    fragments: FragmentData | None = None


@dataclass
class GradientSet:
    d_vertices: np.ndarray  # (N,3,3)
    d_opacity: np.ndarray   # (N,)
    d_sigma: np.ndarray     # (N,)
    d_sh: np.ndarray        # (N,16,3)

    @classmethod
    def zeros(cls, n: int) -> "GradientSet":
        return cls(np.zeros((n, 3, 3)), np.zeros(n), np.zeros(n), np.zeros((n, 16, 3)))

    def param(self, index: int) -> float:
        tri, off = divmod(index, PARAMS_PER_TRIANGLE)
        if off < 9:
            return float(self.d_vertices[tri].reshape(9)[off])
        if off == 9:
            return float(self.d_opacity[tri])
        if off == 10:
            return float(self.d_sigma[tri])
        return float(self.d_sh[tri].reshape(48)[off - 11])

    def scaled(self, factor: float) -> "GradientSet":
        return GradientSet(self.d_vertices * factor, self.d_opacity * factor,
                           self.d_sigma * factor, self.d_sh * factor)

    def add(self, other: "GradientSet"):
        self.d_vertices += other.d_vertices
        self.d_opacity += other.d_opacity
        self.d_sigma += other.d_sigma
        self.d_sh += other.d_sh
