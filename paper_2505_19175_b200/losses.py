"""On-device losses: drop-ins for the reference's
``photometric_loss`` / ``ssim`` (trisplat/losses.py:110-142),
``distortion_loss`` (:169-203), ``depth_from_fragments`` (:206-216) and
``normal_loss`` (:219-292).

Same signatures, return types and errors as the reference:
  photometric_loss(rendered, target, lam) -> (loss: float, grad)
  ssim(x, y) -> float
Inputs may be numpy arrays / ``ImageBuffer`` (H x W x 3; the result gradient is
then a numpy fp64 array, like the reference's) or CUDA tensors (no host round
trip: the gradient stays a CUDA fp32 tensor, ready for ``Rasterizer.backward``).
The computation runs in ts_loss.cu (fp64 window statistics); images enter as
fp32, the rasterizer's output precision.
"""
from __future__ import annotations

import ctypes

import numpy as np

SSIM_WINDOW = 11


def _as_image(a):
    rgb = getattr(a, "rgb", a)  # ImageBuffer
    return rgb


def _to_dev(a):
    import torch
    if isinstance(a, torch.Tensor):
        return a.detach().to(device="cuda", dtype=torch.float32).contiguous(), True
    return torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=np.float64)), dtype=torch.float32,
                           device="cuda").contiguous(), False


def _shape(a):
    return tuple(a.shape)


def _run(x, y, lam, want_grad, ssim_only=False, rasterizer=None, stream=None):
    import torch
    from . import _lib
    from .rasterizer import default_rasterizer
    r = rasterizer or default_rasterizer()
    h, w = int(x.shape[0]), int(x.shape[1])
    out = torch.empty(2, dtype=torch.float64, device="cuda")
    grad = torch.empty_like(x) if want_grad else None
    st = (stream or torch.cuda.current_stream()).cuda_stream
    if ssim_only:
        rc = r.lib.ts_ssim(r._ctx, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), h, w,
                           ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st))
        _lib.check(rc, "ssim")
    else:
        rc = r.lib.ts_photometric_loss(r._ctx, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), h, w,
                                       float(lam), ctypes.c_void_p(out.data_ptr()),
                                       ctypes.c_void_p(grad.data_ptr() if grad is not None else 0),
                                       ctypes.c_void_p(st))
        _lib.check(rc, "photometric_loss")
    return out, grad


def photometric_loss(rendered, target, lam: float, rasterizer=None, stream=None):
    """(1-lambda) * L1 + lambda * (1 - SSIM)/2, with gradient w.r.t. rendered
    (losses.py:122-142)."""
    r, t = _as_image(rendered), _as_image(target)
    if _shape(r) != _shape(t):
        raise ValueError(f"image dimensions differ: {_shape(r)} vs {_shape(t)}")
    x, dev_in = _to_dev(r)
    y, _ = _to_dev(t)
    if x.ndim != 3 or x.shape[2] != 3:
        raise ValueError("image must be HxWx3")
    out, grad = _run(x, y, lam, True, rasterizer=rasterizer, stream=stream)
    if dev_in:
        return float(out[0].item()), grad
    return float(out[0].item()), grad.double().cpu().numpy()


def ssim(x, y, rasterizer=None, stream=None) -> float:
    """Mean SSIM over channels (11x11 Gaussian window, sigma 1.5; losses.py:110-119)."""
    a, b = _as_image(x), _as_image(y)
    if _shape(a) != _shape(b):
        raise ValueError("image dimensions differ")
    if a.shape[0] < SSIM_WINDOW or a.shape[1] < SSIM_WINDOW:
        return 1.0
    xa, _ = _to_dev(a)
    yb, _ = _to_dev(b)
    out, _ = _run(xa, yb, 1.0, False, ssim_only=True, rasterizer=rasterizer, stream=stream)
    return float(out[1].item())


def _frag_dev(fragments):
    """(offsets int64, weight f64, depth f64) CUDA tensors and whether the input was on the device."""
    import torch
    off = fragments.offsets
    if isinstance(off, torch.Tensor):
        return (off.to(device="cuda", dtype=torch.int64).contiguous(),
                fragments.weight.to(device="cuda", dtype=torch.float64).contiguous(),
                fragments.depth.to(device="cuda", dtype=torch.float64).contiguous(), True)
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")  # noqa: E731
    return (t(np.asarray(off, dtype=np.int64), torch.int64), t(np.asarray(fragments.weight, np.float64), torch.float64),
            t(np.asarray(fragments.depth, np.float64), torch.float64), False)


def distortion_loss(fragments, image_size: int | None = None, rasterizer=None, stream=None):
    """Pairwise blend-weighted depth spread averaged over pixels (losses.py:169-203).
    Returns (value, d_weight, d_depth) aligned with the fragment arrays (CUDA
    tensors for DeviceFragments input, numpy for FragmentData)."""
    import torch
    from . import _lib
    from .rasterizer import default_rasterizer
    off, w, z, dev_in = _frag_dev(fragments)
    npix = off.numel() - 1
    nf = w.numel()
    if nf == 0:
        zero = torch.zeros(0, dtype=torch.float64, device="cuda")
        return (0.0, zero, zero) if dev_in else (0.0, np.zeros(0), np.zeros(0))
    r = rasterizer or default_rasterizer()
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    d_w = torch.empty_like(w)
    d_z = torch.empty_like(z)
    st = (stream or torch.cuda.current_stream()).cuda_stream
    rc = r.lib.ts_distortion_loss(r._ctx, ctypes.c_void_p(off.data_ptr()), ctypes.c_void_p(w.data_ptr()),
                                  ctypes.c_void_p(z.data_ptr()), npix,
                                  int(image_size) if image_size is not None else npix,
                                  ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(d_w.data_ptr()),
                                  ctypes.c_void_p(d_z.data_ptr()), ctypes.c_void_p(st))
    _lib.check(rc, "distortion_loss")
    if dev_in:
        return float(out.item()), d_w, d_z
    return float(out.item()), d_w.cpu().numpy(), d_z.cpu().numpy()


def depth_from_fragments(fragments, height: int, width: int, rasterizer=None, stream=None):
    """Blend-weight-normalised expected depth per pixel, 0 where empty (losses.py:206-216)."""
    import torch
    from . import _lib
    from .rasterizer import default_rasterizer
    off, w, z, dev_in = _frag_dev(fragments)
    r = rasterizer or default_rasterizer()
    d = torch.empty(height * width, dtype=torch.float64, device="cuda")
    st = (stream or torch.cuda.current_stream()).cuda_stream
    rc = r.lib.ts_fragment_depth(r._ctx, ctypes.c_void_p(off.data_ptr()), ctypes.c_void_p(w.data_ptr()),
                                 ctypes.c_void_p(z.data_ptr()), height * width, ctypes.c_void_p(d.data_ptr()),
                                 ctypes.c_void_p(st))
    _lib.check(rc, "fragment_depth")
    d = d.view(height, width)
    return d if dev_in else d.cpu().numpy()


def normal_loss(triangles, fragments, depth, intr, pose, rasterizer=None, stream=None):
    """Blend-weighted misalignment of the camera-facing triangle normals with
    the depth-map normals (losses.py:219-292, depth normals held fixed).
    Returns (value, d_vertices (N,3,3) fp64, d_weight (F,) fp64): CUDA tensors
    for device inputs (DeviceSoup / DeviceFragments), numpy otherwise."""
    import torch
    from . import _lib
    from .rasterizer import default_rasterizer, make_camera
    from .types import as_soup
    dev_in = isinstance(getattr(triangles, "vertices", None), torch.Tensor)
    if dev_in:
        v = triangles.vertices.to(device="cuda", dtype=torch.float32).contiguous()
    else:
        v = torch.as_tensor(np.asarray(as_soup(triangles).vertices, dtype=np.float32), device="cuda").contiguous()
    n = v.shape[0]
    off, w, _, _ = _frag_dev(fragments)
    tri = fragments.triangle
    tri = (tri if isinstance(tri, torch.Tensor) else torch.as_tensor(np.asarray(tri))).to(
        device="cuda", dtype=torch.int32).contiguous()
    d = depth if isinstance(depth, torch.Tensor) else torch.as_tensor(np.asarray(depth, dtype=np.float64))
    d = d.to(device="cuda", dtype=torch.float64).contiguous()
    nf = w.numel()
    if nf == 0:
        z = torch.zeros((n, 3, 3), dtype=torch.float64, device="cuda")
        e = torch.zeros(0, dtype=torch.float64, device="cuda")
        return (0.0, z, e) if dev_in else (0.0, z.cpu().numpy(), e.cpu().numpy())
    r = rasterizer or default_rasterizer()
    cam = make_camera(intr, pose)
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    dv = torch.empty((n, 3, 3), dtype=torch.float64, device="cuda")
    dw = torch.empty(nf, dtype=torch.float64, device="cuda")
    st = (stream or torch.cuda.current_stream()).cuda_stream
    rc = r.lib.ts_normal_loss(r._ctx, ctypes.c_void_p(v.data_ptr()), n, ctypes.c_void_p(off.data_ptr()),
                              ctypes.c_void_p(tri.data_ptr()), ctypes.c_void_p(w.data_ptr()), nf,
                              ctypes.c_void_p(d.data_ptr()), ctypes.byref(cam), ctypes.c_void_p(out.data_ptr()),
                              ctypes.c_void_p(dv.data_ptr()), ctypes.c_void_p(dw.data_ptr()), ctypes.c_void_p(st))
    _lib.check(rc, "normal_loss")
    if dev_in:
        return float(out.item()), dv, dw
    return float(out.item()), dv.cpu().numpy(), dw.cpu().numpy()


def install(trisplat_module=None):
    """Rebind the reference's photometric_loss / ssim (imported by name in
    training.py:16-17, scene_io.py:23, __init__.py:18-19) to this path."""
    import importlib
    import sys
    patched = []
    targets = {"trisplat": ("photometric_loss", "ssim", "distortion_loss", "normal_loss"),
               "trisplat.losses": ("photometric_loss", "ssim", "distortion_loss", "depth_from_fragments",
                                   "normal_loss"),
               "trisplat.training": ("photometric_loss", "distortion_loss", "depth_from_fragments", "normal_loss"),
               "trisplat.scene_io": ("_ssim",)}
    repl = {"photometric_loss": photometric_loss, "ssim": ssim, "_ssim": ssim, "distortion_loss": distortion_loss,
            "depth_from_fragments": depth_from_fragments, "normal_loss": normal_loss}
    for mod_name, names in targets.items():
        try:
            mod = sys.modules.get(mod_name) or importlib.import_module(mod_name)
        except Exception:
            continue
        for nm in names:
            if hasattr(mod, nm):
                setattr(mod, nm, repl[nm])
                patched.append(f"{mod_name}.{nm}")
    return patched
