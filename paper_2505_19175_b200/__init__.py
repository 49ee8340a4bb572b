"""B200-native differentiable rasterizer for Triangle Splatting (arXiv 2505.19175).

Drop-in replacement for the reference package's render() / render_backward()
path: every stage runs as hand-written sm_100a CUDA behind the C ABI in
include/trisplat_b200.h.  See DESIGN.md.
"""
__version__ = "0.1.0"

from .types import (CameraIntrinsics, CameraPose, FragmentData, GradientSet,  # noqa: F401
                    ImageBuffer, RenderOutput, SceneProjection, Triangle3D, TriangleSoup, WindowMode)


def __getattr__(name):
    # torch-dependent API is imported lazily so the types stay importable
    # without a GPU stack.
    if name in ("render", "render_backward", "project_scene", "build_tile_lists", "install", "Rasterizer", "DeviceSoup",
                "DeviceGrads", "ForwardResult", "default_rasterizer"):
        from . import rasterizer
        return getattr(rasterizer, name)
    raise AttributeError(name)
