"""B200 rasterizer: device-resident API plus the reference's drop-in functions.

Device-resident API (the hot path; no host copies)::

    rast = Rasterizer()
    soup = DeviceSoup.from_soup(cpu_soup, dtype=torch.float32)
    fwd = rast.forward(soup, intr, pose)          # torch tensors on cuda
    grads = rast.backward(d_image)                # DeviceGrads (fp32)

Drop-in functions with the reference signatures and error behaviour:

    render(triangles, intr, pose, mode, background, collect_fragments,
           tau_cutoff, tile_size, active_sh_degree) -> RenderOutput     render.py:364-432
    render_backward(triangles, intr, pose, mode, background, d_image,
                    frag_grads, tau_cutoff, tile_size, active_sh_degree) -> GradientSet
                                                                        backward.py:93-211

Both run every stage on the GPU through the C ABI (include/trisplat_b200.h);
numpy inputs are uploaded (fp64 kept as fp64 so the drop-in sees exactly the
reference's parameter values) and numpy outputs returned.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .types import (DEFAULT_TAU_CUTOFF, DEFAULT_TILE_SIZE, TAU_CONTRIB, FragmentData,
                    GradientSet, ImageBuffer, RenderOutput, SceneProjection, as_soup, mode_flag)

PRECISION = {"fast": 0, "exact": 1}


def _require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("trisplat_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


# host -> device uploads of large numpy arrays: chunks copied (multi-threaded)
# into a small ring of pinned buffers while the previous chunk's DMA runs, about
# 4x the rate of a pageable copy (the drop-in render() uploads the reference's
# 944 MB fp64 soup every call)
_STAGE_CHUNK = 16 << 20  # 6 buffers, DMA alternating over 2 streams (measured: 49 GB/s)
_STAGE_NBUF = 6
_STAGE: dict = {}  # device index -> ([(pinned buffer, event)], [copy streams])


def _staged_h2d(a: np.ndarray, device="cuda") -> torch.Tensor:
    src = torch.from_numpy(a)
    out = torch.empty(src.shape, dtype=src.dtype, device=device)
    nbytes = a.nbytes
    if nbytes < (4 << 20):
        out.copy_(src)
        return out
    dev = out.device.index if out.device.index is not None else torch.cuda.current_device()
    if dev not in _STAGE:
        with torch.cuda.device(dev):
            _STAGE[dev] = ([(torch.empty(_STAGE_CHUNK, dtype=torch.uint8).pin_memory(), torch.cuda.Event())
                            for _ in range(_STAGE_NBUF)], [torch.cuda.Stream(dev) for _ in range(2)])
    ring, streams = _STAGE[dev]
    sb = src.reshape(-1).view(torch.uint8)
    ob = out.reshape(-1).view(torch.uint8)
    cur = torch.cuda.current_stream(out.device)
    for st in streams:
        st.wait_stream(cur)  # (out is allocated on the current stream)
    for i, off in enumerate(range(0, nbytes, _STAGE_CHUNK)):
        buf, ev = ring[i % len(ring)]
        st = streams[i % len(streams)]
        c = min(_STAGE_CHUNK, nbytes - off)
        ev.synchronize()  # the slot's previous DMA is done
        buf[:c].copy_(sb[off:off + c])
        with torch.cuda.stream(st):
            ob[off:off + c].copy_(buf[:c], non_blocking=True)
            ev.record(st)
    for st in streams:
        cur.wait_stream(st)
    return out


# lossless fp32 upload (ts_upload_f32): chunk bytes, ring slots, flags (bit 0: streaming stores)
_UPLOAD_F32 = (16 << 20, 4, 1)  # (tools/upload_probe.py: 12.7 ms for the north-star soup; 4 MB x 4 regular stores 15.8)


def _staged_h2d_f32(a: np.ndarray, device="cuda") -> "torch.Tensor | None":
    """fp64 array -> fp32 device tensor when every value is an fp32 value
    (ts_upload_f32: each chunk converted on the host's threads into a
    page-locked ring slot while the previous chunk's DMA runs), else None."""
    lib = _lib.load()
    src = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    out = torch.empty(a.shape, dtype=torch.float32, device=device)
    with torch.cuda.device(out.device):
        st = torch.cuda.current_stream(out.device)
        chunk, nslot, flags = _UPLOAD_F32
        rc = lib.ts_upload_f32(ctypes.c_void_p(src.ctypes.data), src.size, ctypes.c_void_p(out.data_ptr()),
                               ctypes.c_void_p(st.cuda_stream), chunk, nslot, flags)
    if rc < 0:
        _lib.check(rc, "upload_f32")
    return out if rc == 1 else None


@dataclass
class DeviceSoup:
    """Triangle parameters resident on the GPU (SoA, soup.py:17-30)."""

    vertices: torch.Tensor  # (N,3,3)
    opacity: torch.Tensor   # (N,)
    sigma: torch.Tensor     # (N,)
    sh: torch.Tensor        # (N,16,3)
    solid: bool = False

    @classmethod
    def from_soup(cls, soup, dtype=torch.float32, device="cuda") -> "DeviceSoup":
        soup = as_soup(soup)
        n = len(soup.vertices)

        def up(a, shape):
            a = np.ascontiguousarray(np.asarray(a).reshape(shape))
            if torch.from_numpy(a[:0]).dtype == dtype and torch.device(device).type == "cuda":
                return _staged_h2d(a, device)
            return torch.as_tensor(a, dtype=dtype).to(device)

        return cls(up(soup.vertices, (n, 3, 3)), up(soup.opacity, (n,)), up(soup.sigma, (n,)),
                   up(soup.sh, (n, 16, 3)), bool(getattr(soup, "solid", False)))

    def __len__(self):
        return self.vertices.shape[0]

    @classmethod
    def from_soup_f32_exact(cls, soup, device="cuda") -> "DeviceSoup | None":
        """The fp64 soup as fp32 device tensors if every parameter is an fp32
        value (half the upload, the same values), else None."""
        soup = as_soup(soup)
        n = len(soup.vertices)
        if n == 0:
            return None
        parts = []
        for a, shape in ((soup.vertices, (n, 3, 3)), (soup.opacity, (n,)), (soup.sigma, (n,)),
                         (soup.sh, (n, 16, 3))):
            a = np.asarray(a)
            if a.dtype != np.float64:
                return None
            t = _staged_h2d_f32(a.reshape(shape), device)
            if t is None:
                return None
            parts.append(t)
        return cls(*parts, bool(getattr(soup, "solid", False)))


    @property
    def dtype(self):
        return self.vertices.dtype

    def _ts(self):
        for t in (self.vertices, self.opacity, self.sigma, self.sh):
            if not t.is_cuda or not t.is_contiguous() or t.dtype != self.vertices.dtype:
                raise ValueError("DeviceSoup tensors must be contiguous CUDA tensors of one dtype")
        n = len(self)
        shapes = {"vertices": (tuple(self.vertices.shape), (n, 3, 3)),
                  "opacity": (tuple(self.opacity.shape), (n,)),
                  "sigma": (tuple(self.sigma.shape), (n,)),
                  "sh": (tuple(self.sh.shape), (n, 16, 3))}
        for name, (got, want) in shapes.items():
            if got != want:
                raise ValueError(f"DeviceSoup.{name} must have shape {want}, got {got}")
        return _lib.TsSoup(self.vertices.data_ptr(), self.opacity.data_ptr(),
                           self.sigma.data_ptr(), self.sh.data_ptr(), len(self))


@dataclass
class DeviceGrads:
    """GradientSet on the GPU (backward.py:24-56), fp32, one flat buffer
    [d_vertices (N*9) | d_opacity (N) | d_sigma (N) | d_sh (N*48)] so a
    single all-reduce covers all 59 parameters."""

    flat: torch.Tensor
    n: int

    @classmethod
    def zeros(cls, n: int, device="cuda") -> "DeviceGrads":
        return cls(torch.zeros(n * 59, dtype=torch.float32, device=device), n)

    @property
    def d_vertices(self):
        return self.flat[: self.n * 9].view(self.n, 3, 3)

    @property
    def d_opacity(self):
        return self.flat[self.n * 9: self.n * 10]

    @property
    def d_sigma(self):
        return self.flat[self.n * 10: self.n * 11]

    @property
    def d_sh(self):
        return self.flat[self.n * 11:].view(self.n, 16, 3)

    def _ts(self):
        return _lib.TsGrads(self.d_vertices.data_ptr(), self.d_opacity.data_ptr(),
                            self.d_sigma.data_ptr(), self.d_sh.data_ptr())

    def to_gradient_set(self) -> GradientSet:
        return GradientSet(self.d_vertices.double().cpu().numpy(),
                           self.d_opacity.double().cpu().numpy(),
                           self.d_sigma.double().cpu().numpy(),
                           self.d_sh.double().cpu().numpy())


@dataclass
class DeviceFragments:
    """FragmentData (render.py:68-81) on the GPU."""

    offsets: torch.Tensor   # (H*W+1,) int64
    triangle: torch.Tensor  # (F,) int32 source ids
    weight: torch.Tensor    # (F,) float64 T*alpha
    depth: torch.Tensor     # (F,) float64 camera-space z

    def to_fragment_data(self) -> FragmentData:
        return FragmentData(offsets=self.offsets.cpu().numpy(),
                            triangle=self.triangle.cpu().numpy().astype(np.int64),
                            weight=self.weight.cpu().numpy(), depth=self.depth.cpu().numpy())


@dataclass
class ForwardResult:
    image: torch.Tensor        # (H,W,3) float32, clipped
    alpha_map: torch.Tensor    # (H,W)
    max_weight: torch.Tensor   # (N,)
    pixel_count: torch.Tensor  # (N,) int32
    area: torch.Tensor         # (N,)
    last_src: torch.Tensor | None  # (H,W) int32
    n_frag: torch.Tensor | None    # (H,W) int32
    n_visible: int
    n_entries: int
    n_flagged: int


def make_camera(intr, pose) -> _lib.TsCamera:
    r = np.asarray(pose.rotation, dtype=np.float64).reshape(9)
    t = np.asarray(pose.translation, dtype=np.float64).reshape(3)
    return _lib.TsCamera(float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy),
                         float(getattr(intr, "z_near", 0.01)), (ctypes.c_double * 9)(*r),
                         (ctypes.c_double * 3)(*t), int(intr.width), int(intr.height))


def make_options(mode=0, background=(0.0, 0.0, 0.0), tau_cutoff=DEFAULT_TAU_CUTOFF,
                 tile_size=DEFAULT_TILE_SIZE, active_sh_degree=3, solid=False, precision="fast",
                 param_dtype=torch.float32, validate=True,
                 keep_backward=True) -> _lib.TsOptions:
    bg = np.asarray(background, dtype=np.float64).reshape(3)
    if not 0 <= int(active_sh_degree) <= 3:
        raise ValueError("SH degree must be in [0,3]")
    check_tile_size(tile_size)
    # every output of render / render_backward is independent of the tile size
    # (each pixel composites the triangles whose bbox holds it, in depth order);
    # the kernels always work on 16x16 tiles
    return _lib.TsOptions(mode_flag(mode), int(active_sh_degree), 16, int(bool(solid)),
                          float(tau_cutoff), float(TAU_CONTRIB), (ctypes.c_double * 3)(*bg),
                          PRECISION[precision] if isinstance(precision, str) else int(precision),
                          1 if param_dtype == torch.float64 else 0, int(bool(validate)),
                          int(bool(keep_backward)))


_NONFINITE_GROUPS = ("vertices", "opacity", "sigma", "sh")


def check_tile_size(tile_size):
    """The reference divides by the tile size (render.py:352-353): 0 raises
    ZeroDivisionError there; negative sizes are rejected here."""
    ts = int(tile_size)
    if ts == 0:
        raise ZeroDivisionError("integer division or modulo by zero")
    if ts < 0:
        raise ValueError(f"tile_size must be positive, got {ts}")
    return ts


def _check_grads(grads: "DeviceGrads", n: int):
    """The kernels write 59 * n floats of the last forward's soup: the buffer
    must be sized for exactly that soup (a DeviceGrads kept across a densify
    step would otherwise be written past its end)."""
    if grads.n != n or grads.flat.numel() != 59 * n or not grads.flat.is_contiguous() \
            or grads.flat.dtype != torch.float32 or not grads.flat.is_cuda:
        raise ValueError(f"gradient buffer is for {grads.n} triangles ({grads.flat.numel()} floats), "
                         f"the last forward had {n} (needs {59 * n} contiguous float32 on the GPU)")


class Rasterizer:
    """One C-ABI context (scratch memory + last forward state) on one device."""

    def __init__(self, device: int | None = None):
        _require_cuda()
        self.lib = _lib.load()
        self.device = torch.cuda.current_device() if device is None else int(device)
        h = ctypes.c_void_p()
        _lib.check(self.lib.ts_context_create(ctypes.byref(h), self.device), "context_create")
        self._ctx = h
        self._last = None  # (n, H, W)
        self._last_soup = None

    def __del__(self):
        try:
            if getattr(self, "_ctx", None):
                self.lib.ts_context_destroy(self._ctx)
        except Exception:
            pass

    def set_option(self, option: int, value: int):
        """Cross-check paths for tests (_lib.TS_OPT_LEGACY_BINNING, TS_OPT_TILE_BACKWARD)."""
        _lib.check(self.lib.ts_set_option(self._ctx, int(option), int(value)), "set_option")

    def launch_count(self) -> int:
        return int(self.lib.ts_launch_count(self._ctx))

    def profile(self, enable: bool = True):
        """Record CUDA events around every pipeline stage (on the call's stream)."""
        _lib.check(self.lib.ts_profile(self._ctx, int(bool(enable))), "profile")

    def set_async(self, enable: bool = True):
        """Asynchronous forwards: forward() enqueues the frame and returns without
        waiting for the GPU (ForwardResult counts are then -1); status() waits and
        reports the last frame."""
        _lib.check(self.lib.ts_set_async(self._ctx, int(bool(enable))), "set_async")
        self._async = bool(enable)

    @property
    def is_async(self) -> bool:
        return bool(getattr(self, "_async", False))

    def status(self, stream=None) -> dict:
        """Wait for the last forward and return its counts; raises on non-finite
        input or if an asynchronous frame outgrew the tile-entry buffer (repeat it)."""
        res = _lib.TsForwardResult()
        dev = torch.device("cuda", self.device)
        st = (stream or torch.cuda.current_stream(dev)).cuda_stream
        rc = self.lib.ts_forward_status(self._ctx, ctypes.byref(res), ctypes.c_void_p(st))
        if rc != _lib.TS_OK:
            self._last = None
            self._last_soup = None
        if rc == _lib.TS_ERR_NONFINITE:
            for g, idx in zip(_NONFINITE_GROUPS, res.err_index):
                if idx >= 0:
                    raise ValueError(f"non-finite {g} in triangle {int(idx)}")
        _lib.check(rc, "forward_status")
        return {"n_visible": int(res.n_visible), "n_entries": int(res.n_entries),
                "n_flagged": int(res.n_flagged)}

    def flagged_pixels(self) -> int:
        """Pixels of the last fast forward re-resolved by the exact fix-up."""
        torch.cuda.synchronize()
        v = ctypes.c_int64()
        _lib.check(self.lib.ts_flagged_pixels(self._ctx, ctypes.byref(v)), "flagged_pixels")
        return int(v.value)

    def stage_times(self) -> dict:
        """Device milliseconds of each stage of the last forward/backward."""
        buf = (ctypes.c_float * len(_lib.STAGES))()
        _lib.check(self.lib.ts_stage_times(self._ctx, buf, len(_lib.STAGES)), "stage_times")
        return {k: float(v) for k, v in zip(_lib.STAGES, buf)}

    def forward(self, soup: DeviceSoup, intr, pose, mode=0, background=(0.0, 0.0, 0.0),
                tau_cutoff=DEFAULT_TAU_CUTOFF, tile_size=DEFAULT_TILE_SIZE, active_sh_degree=3,
                precision="fast", validate=True, debug=False, out: ForwardResult | None = None,
                stream=None, keep_backward=True) -> ForwardResult:
        n = len(soup)
        h, w = int(intr.height), int(intr.width)
        dev = soup.vertices.device
        if out is None:
            out = ForwardResult(
                image=torch.empty((h, w, 3), dtype=torch.float32, device=dev),
                alpha_map=torch.empty((h, w), dtype=torch.float32, device=dev),
                max_weight=torch.empty(n, dtype=torch.float32, device=dev),
                pixel_count=torch.empty(n, dtype=torch.int32, device=dev),
                area=torch.empty(n, dtype=torch.float32, device=dev),
                last_src=torch.empty((h, w), dtype=torch.int32, device=dev) if debug else None,
                n_frag=torch.empty((h, w), dtype=torch.int32, device=dev) if debug else None,
                n_visible=0, n_entries=0, n_flagged=0)
        cam = make_camera(intr, pose)
        opt = make_options(mode, background, tau_cutoff, tile_size, active_sh_degree, soup.solid,
                           precision, soup.dtype, validate, keep_backward)
        fo = _lib.TsForwardOut(_ptr(out.image), _ptr(out.alpha_map), _ptr(out.max_weight),
                               _ptr(out.pixel_count), _ptr(out.area), _ptr(out.last_src),
                               _ptr(out.n_frag))
        res = _lib.TsForwardResult()
        st = (stream or torch.cuda.current_stream(dev)).cuda_stream
        ts = soup._ts()
        rc = self.lib.ts_forward(self._ctx, ctypes.byref(cam), ctypes.byref(opt),
                                 ctypes.byref(ts), ctypes.byref(fo), ctypes.byref(res),
                                 ctypes.c_void_p(st))
        if rc != _lib.TS_OK:  # the context keeps no state of a failed frame
            self._last = None
            self._last_soup = None
        if rc == _lib.TS_ERR_NONFINITE:
            for g, idx in zip(_NONFINITE_GROUPS, res.err_index):
                if idx >= 0:
                    raise ValueError(f"non-finite {g} in triangle {int(idx)}")
        _lib.check(rc, "forward")
        out.n_visible, out.n_entries, out.n_flagged = (int(res.n_visible), int(res.n_entries),
                                                       int(res.n_flagged))
        self._last = (n, h, w)
        self._last_soup = soup  # ts_backward reads these parameters: keep them alive
        return out

    def backward(self, d_image: torch.Tensor, grads: DeviceGrads | None = None,
                 accumulate: bool = False, stream=None, chunks=None) -> DeviceGrads:
        """Gradient of sum(d_image * C) into ``grads`` (+= when accumulating).
        ``chunks = (bounds, events)``: the final chain to the parameter
        gradients runs in triangle ranges [bounds[k], bounds[k+1]) and
        torch.cuda.Event events[k] is recorded once range k is final
        (ts_backward_chunked; parallel.chunk_bounds gives valid bounds)."""
        if self._last is None:
            raise RuntimeError("backward() needs a preceding forward()")
        n, h, w = self._last
        if tuple(d_image.shape) != (h, w, 3):
            raise ValueError(f"d_image must be {(h, w, 3)}, got {tuple(d_image.shape)}")
        d_image = d_image.to(dtype=torch.float32).contiguous()
        if grads is None:
            grads = DeviceGrads(torch.empty(n * 59, dtype=torch.float32, device=d_image.device), n)
            accumulate = False
        _check_grads(grads, n)
        stream = stream or torch.cuda.current_stream(d_image.device)
        st = stream.cuda_stream
        g = grads._ts()
        if chunks is None:
            _lib.check(self.lib.ts_backward(self._ctx, _ptr(d_image), ctypes.byref(g),
                                            int(bool(accumulate)), ctypes.c_void_p(st)), "backward")
            return grads
        bounds, events = chunks
        k = len(bounds) - 1
        if len(events) != k:
            raise ValueError("one event per chunk")
        for ev in events:  # (torch creates the CUDA event at its first record)
            ev.record(stream)
        b = (ctypes.c_int64 * (k + 1))(*[int(x) for x in bounds])
        evp = (ctypes.c_void_p * k)(*[ctypes.c_void_p(ev.cuda_event) for ev in events])
        _lib.check(self.lib.ts_backward_chunked(self._ctx, _ptr(d_image), ctypes.byref(g), int(bool(accumulate)),
                                                k, b, evp, ctypes.c_void_p(st)), "backward_chunked")
        return grads

    def reserve(self, n: int, width: int, height: int, entries: int = 0, keep_backward: bool = False) -> int:
        """Size every per-frame buffer for scenes of up to n triangles at
        width x height (ts_reserve), so later forwards / backwards of that size
        allocate nothing; returns the device bytes the context holds."""
        _lib.check(self.lib.ts_reserve(self._ctx, int(n), int(width), int(height), int(entries),
                                       int(bool(keep_backward))), "reserve")
        return self.workspace_bytes()

    def workspace_bytes(self) -> int:
        return int(self.lib.ts_workspace_bytes(self._ctx))

    MAX_PENDING_VIEWS = 8

    def backward_screen(self, d_image: torch.Tensor, stream=None) -> int:
        """Blend backward of the last (training) forward into the next pending-view
        slot (ts_backward_screen); ``chain_views`` later turns every pending view
        into parameter gradients in one pass.  Returns the number of pending views."""
        if self._last is None:
            raise RuntimeError("backward_screen() needs a preceding forward()")
        _, h, w = self._last
        if tuple(d_image.shape) != (h, w, 3):
            raise ValueError(f"d_image must be {(h, w, 3)}, got {tuple(d_image.shape)}")
        d_image = d_image.to(dtype=torch.float32).contiguous()
        st = (stream or torch.cuda.current_stream(d_image.device)).cuda_stream
        _lib.check(self.lib.ts_backward_screen(self._ctx, _ptr(d_image), ctypes.c_void_p(st)), "backward_screen")
        return int(self.lib.ts_pending_views(self._ctx))

    def chain_views(self, grads: DeviceGrads, accumulate: bool = False, stream=None, chunks=None) -> DeviceGrads:
        """Parameter gradients of every pending view (ts_chain_views): ``grads``
        gets their sum (+= when accumulating), as ``backward`` on each view in
        turn would; ``chunks = (bounds, events)`` as in ``backward``."""
        _check_grads(grads, self._last[0] if self._last is not None else grads.n)
        dev = torch.device("cuda", self.device)
        stream = stream or torch.cuda.current_stream(dev)
        st = stream.cuda_stream
        g = grads._ts()
        if chunks is None:
            _lib.check(self.lib.ts_chain_views(self._ctx, ctypes.byref(g), int(bool(accumulate)), 0, None, None,
                                               ctypes.c_void_p(st)), "chain_views")
            return grads
        bounds, events = chunks
        k = len(bounds) - 1
        if len(events) != k:
            raise ValueError("one event per chunk")
        for ev in events:
            ev.record(stream)
        b = (ctypes.c_int64 * (k + 1))(*[int(x) for x in bounds])
        evp = (ctypes.c_void_p * k)(*[ctypes.c_void_p(ev.cuda_event) for ev in events])
        _lib.check(self.lib.ts_chain_views(self._ctx, ctypes.byref(g), int(bool(accumulate)), k, b, evp,
                                           ctypes.c_void_p(st)), "chain_views")
        return grads

    def pending_views(self) -> int:
        return int(self.lib.ts_pending_views(self._ctx))

    def fragments(self, stream=None) -> "DeviceFragments":
        """Fragment lists of the last forward (render(collect_fragments=True),
        render.py:383-399, 420-425): CSR offsets (int64, H*W+1), source ids,
        blend weights T*alpha (fp64) and depths (fp64), in compositing order."""
        if self._last is None:
            raise RuntimeError("fragments() needs a preceding forward()")
        _, h, w = self._last
        dev = torch.device("cuda", self.device)
        st = (stream or torch.cuda.current_stream(dev)).cuda_stream
        off = torch.empty(h * w + 1, dtype=torch.int64, device=dev)
        nf = ctypes.c_int64()
        _lib.check(self.lib.ts_fragment_offsets(self._ctx, _ptr(off), ctypes.byref(nf), ctypes.c_void_p(st)),
                   "fragment_offsets")
        f = int(nf.value)
        tri = torch.empty(max(f, 1), dtype=torch.int32, device=dev)
        wgt = torch.empty(max(f, 1), dtype=torch.float64, device=dev)
        dep = torch.empty(max(f, 1), dtype=torch.float64, device=dev)
        _lib.check(self.lib.ts_collect_fragments(self._ctx, _ptr(off), _ptr(tri), _ptr(wgt), _ptr(dep),
                                                 ctypes.c_void_p(st)), "collect_fragments")
        return DeviceFragments(off, tri[:f], wgt[:f], dep[:f])

    def backward_fragments(self, d_image: torch.Tensor, offsets: torch.Tensor, d_weight: torch.Tensor,
                           d_depth: torch.Tensor, grads: DeviceGrads | None = None, accumulate: bool = False,
                           stream=None, weight: torch.Tensor | None = None) -> DeviceGrads:
        """backward() plus upstream gradients on the blend weight and depth of
        every fragment (render_backward(frag_grads=...), backward.py:122-142).
        ``weight``: the fragments' blend weights of this forward
        (``fragments().weight``); with it the gradient streams over the
        forward's fragment records instead of replaying every pixel."""
        if self._last is None:
            raise RuntimeError("backward_fragments() needs a preceding forward()")
        n, h, w = self._last
        if tuple(d_image.shape) != (h, w, 3):
            raise ValueError(f"d_image must be {(h, w, 3)}, got {tuple(d_image.shape)}")
        dev = torch.device("cuda", self.device)
        d_image = d_image.to(device=dev, dtype=torch.float32).contiguous()
        offsets = offsets.to(device=dev, dtype=torch.int64).contiguous()
        d_weight = d_weight.to(device=dev, dtype=torch.float64).contiguous()
        d_depth = d_depth.to(device=dev, dtype=torch.float64).contiguous()
        if grads is None:
            grads = DeviceGrads(torch.empty(n * 59, dtype=torch.float32, device=dev), n)
            accumulate = False
        _check_grads(grads, n)
        st = (stream or torch.cuda.current_stream(dev)).cuda_stream
        g = grads._ts()
        if weight is not None:
            weight = weight.to(device=dev, dtype=torch.float64).contiguous()
            if weight.numel() != d_weight.numel():
                raise ValueError("fragment gradients do not match this scene/camera")
        rc = self.lib.ts_backward_fragments(self._ctx, _ptr(d_image), _ptr(offsets), _ptr(weight), _ptr(d_weight),
                                            _ptr(d_depth), ctypes.byref(g), int(bool(accumulate)),
                                            ctypes.c_void_p(st))
        if rc == _lib.TS_ERR_FRAGMENTS:
            raise ValueError("fragment gradients do not match this scene/camera")
        _lib.check(rc, "backward_fragments")
        return grads

    # ---- parity dumps (project_scene / build_tile_lists internals) ----
    def _dump(self, what, numel, dtype):
        buf = torch.empty(max(numel, 1), dtype=dtype, device="cuda")
        _lib.check(self.lib.ts_debug_copy(self._ctx, what, _ptr(buf), buf.numel() * buf.element_size(),
                                          ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
                   "debug_copy")
        return buf[:numel].cpu().numpy()

    def dump_sorted_idx(self, m):
        return self._dump(_lib.TS_DUMP_SORTED_IDX, m, torch.int32).astype(np.int64)

    def dump_tile_start(self, ntiles):
        return self._dump(_lib.TS_DUMP_TILE_START, ntiles + 1, torch.int32).astype(np.int64)

    def dump_entry_rank(self, e):
        return self._dump(_lib.TS_DUMP_ENTRY_RANK, e, torch.int32).astype(np.int64)

    def dump_bbox(self, n):
        return self._dump(_lib.TS_DUMP_BBOX, n * 4, torch.int32).reshape(n, 4).astype(np.int64)

    def dump_depth(self, n):
        return self._dump(_lib.TS_DUMP_DEPTH, n, torch.float64)

    def dump_fragment_records(self, max_records):
        """Fragment records of the last training forward (streaming backward input)."""
        raw = self._dump(_lib.TS_DUMP_FRAGREC, 8 + 48 * max_records, torch.uint8)
        cnt = int(raw[:8].view(np.uint64)[0])
        rec = raw[8:8 + 48 * cnt].reshape(cnt, 48)
        tc = rec[:, :32].copy().view(np.float64).reshape(cnt, 4)
        ids = rec[:, 32:].copy().view(np.uint32).reshape(cnt, 4)
        return tc, ids

    def dump_sgrad(self, n):
        return self._dump(_lib.TS_DUMP_SGRAD, n * 16, torch.float64).reshape(n, 16)


_DEFAULT: Rasterizer | None = None


def default_rasterizer() -> Rasterizer:
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = Rasterizer()
    return _DEFAULT


def _param_dtype(soup):
    v = np.asarray(soup.vertices)
    return torch.float32 if v.dtype == np.float32 else torch.float64


def project_scene(soup, intr, pose, mode=0, tau_cutoff: float = DEFAULT_TAU_CUTOFF,
                  active_sh_degree: int = 3) -> SceneProjection:
    """Drop-in for trisplat.render.project_scene (render.py:253-312): the
    projection, cull, depth order, edges, tight bboxes and SH colour of every
    accepted triangle, in fp64, from the device (a forward on the default
    rasterizer, then the TS_DUMP_PROJECTION dump in the reference's operation
    order)."""
    _require_cuda()
    soup = as_soup(soup)
    rast = default_rasterizer()
    ds = DeviceSoup.from_soup(soup, dtype=_param_dtype(soup))
    fwd = rast.forward(ds, intr, pose, mode, (0.0, 0.0, 0.0), tau_cutoff, DEFAULT_TILE_SIZE,
                       active_sh_degree, keep_backward=False)
    n, m = len(ds), fwd.n_visible
    sidx = rast.dump_sorted_idx(m)
    raw = torch.empty(_lib.PROJ_ROW * m + n + 1, dtype=torch.float64, device="cuda")
    _lib.check(rast.lib.ts_debug_copy(rast._ctx, _lib.TS_DUMP_PROJECTION, _ptr(raw), raw.numel() * 8,
                                      ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "debug_copy")
    host = raw.cpu().numpy()
    rows = host[:_lib.PROJ_ROW * m].reshape(m, _lib.PROJ_ROW)
    col = iter(np.cumsum([0, 9, 6, 1, 1, 1, 6, 3, 3, 1, 1, 3, 3, 16, 3, 1, 4]))
    lo = next(col)

    def take(shape):
        nonlocal lo
        hi = next(col)
        a = np.ascontiguousarray(rows[:, lo:hi]).reshape((m,) + shape)
        lo = hi
        return a

    xc, q = take((3, 3)), take((3, 2))
    z, area, phis = take(()), take(()), take(())
    nrm, doff, esign = take((3, 2)), take((3,)), take((3,))
    sig, opa = take(()), take(())
    rgb, raw_rgb, basis, viewdir, u_norm = take((3,)), take((3,)), take((16,)), take((3,)), take(())
    bbox = take((4,)).astype(np.int64)
    return SceneProjection(n_total=n, sorted_idx=sidx, z=z, xc=xc, q=q, nrm=nrm, doff=doff, esign=esign,
                           phis=phis, area=area, sig=sig, opa=opa, rgb=rgb, raw_rgb=raw_rgb, basis=basis,
                           viewdir=viewdir, u_norm=u_norm, bbox=bbox,
                           area_full=np.ascontiguousarray(host[_lib.PROJ_ROW * m:_lib.PROJ_ROW * m + n]))


def build_tile_lists(proj, intr, tile_size: int = DEFAULT_TILE_SIZE):
    """Drop-in for trisplat.render.build_tile_lists (render.py:349-361): CSR
    per-tile lists of depth ranks (each tile's list in rank order) for any tile
    size, built on the device (ts_tile_lists) from ``proj.bbox``.
    Returns (ntx, nty, tile_start int64[ntx*nty+1], entry_tri int64[E])."""
    _require_cuda()
    ts = check_tile_size(tile_size)
    ntx = (int(intr.width) + ts - 1) // ts
    nty = (int(intr.height) + ts - 1) // ts
    bbox = np.ascontiguousarray(np.asarray(proj.bbox, dtype=np.int64).reshape(-1, 4))
    m = bbox.shape[0]
    rast = default_rasterizer()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    bb = torch.from_numpy(bbox).to("cuda") if m else torch.zeros((1, 4), dtype=torch.int64, device="cuda")
    e = ctypes.c_int64()
    _lib.check(rast.lib.ts_tile_lists(rast._ctx, _ptr(bb), m, ts, int(intr.width), int(intr.height), None, None,
                                      ctypes.byref(e), st), "tile_lists")
    start = torch.empty(ntx * nty + 1, dtype=torch.int64, device="cuda")
    entry = torch.empty(max(int(e.value), 1), dtype=torch.int64, device="cuda")
    _lib.check(rast.lib.ts_tile_lists(rast._ctx, _ptr(bb), m, ts, int(intr.width), int(intr.height), _ptr(start),
                                      _ptr(entry), ctypes.byref(e), st), "tile_lists")
    return ntx, nty, start.cpu().numpy(), entry[:int(e.value)].cpu().numpy()


# bytes the last render() copied device -> host and the wall-clock split of
# that call (bench.py's e2e accounting)
LAST_RENDER_D2H_BYTES = 0
LAST_RENDER_TIMES: dict = {}


class _PinnedPool:
    """Page-locked host buffers for render()'s outputs, reused once every array
    handed out from a buffer is gone (a fresh cudaHostAlloc of the ~77 MB of
    outputs costs ~2.5 ms, a pageable array page-faults while it is written).
    The caller's arrays are numpy views of one ndarray per buffer; a weak
    reference to that ndarray tells when the last of them has been dropped."""

    def __init__(self):
        self.entries = []  # [base uint8 pinned tensor, weakref to the ndarray handed out or None]

    def get(self, count: int, dtype: torch.dtype):
        """(device-copyable host tensor, numpy array on the same memory) of ``count`` items."""
        import weakref
        nbytes = count * torch.empty(0, dtype=dtype).element_size()
        free = [e for e in self.entries if e[1] is None or e[1]() is None]
        ent = next((e for e in free if e[0].numel() >= nbytes), None)
        if ent is None:
            # free buffers too small for this request are released (scene sizes change)
            free_ids = {id(e) for e in free}
            self.entries = [e for e in self.entries if id(e) not in free_ids]
            ent = [torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True), None]
            self.entries.append(ent)
        host = ent[0][:nbytes].view(dtype)
        arr = host.numpy()
        ent[1] = weakref.ref(arr)
        return host, arr


_PINNED = _PinnedPool()


def render(triangles, intr, pose, mode=0, background=(0.0, 0.0, 0.0),
           collect_fragments: bool = False, tau_cutoff: float = DEFAULT_TAU_CUTOFF,
           tile_size: int = DEFAULT_TILE_SIZE, active_sh_degree: int = 3,
           precision: str = "fast") -> RenderOutput:
    """Drop-in for trisplat.render.render (render.py:364-432)."""
    global LAST_RENDER_D2H_BYTES, LAST_RENDER_TIMES
    import time
    t0 = time.perf_counter()
    _require_cuda()
    soup = as_soup(triangles)
    if collect_fragments and precision != "fast":
        raise ValueError("collect_fragments needs precision='fast'")
    rast = default_rasterizer()
    # an fp64 soup of fp32 values (the reference's synthetic scenes) crosses PCIe
    # as fp32 and renders through the fp32-parameter kernels with the same values
    ds = DeviceSoup.from_soup_f32_exact(soup) if precision == "fast" and _param_dtype(soup) == torch.float64 \
        else None
    if ds is None:
        ds = DeviceSoup.from_soup(soup, dtype=_param_dtype(soup))
    t1 = time.perf_counter()

    def frame_and_outputs(asynchronous: bool):
        # asynchronous: the frame, the output packing and the copies are enqueued
        # back to back and the host waits once (ts_forward_status checks the frame)
        was = rast.is_async
        rast.set_async(asynchronous)
        try:
            f = rast.forward(ds, intr, pose, mode, background, tau_cutoff, tile_size, active_sh_degree,
                             precision=precision)
            # the fp64 outputs converted and packed on the device, one copy each for the
            # fp64 block and the int64 pixel counts into cached page-locked host memory
            pk = torch.cat([f.image.reshape(-1).double(), f.alpha_map.reshape(-1).double(),
                            f.max_weight.double(), f.area.double()])
            pk_h, flat = _PINNED.get(pk.numel(), torch.float64)
            pk_h.copy_(pk, non_blocking=True)
            pc_h, pixc = _PINNED.get(f.max_weight.numel(), torch.int64)
            pc_h.copy_(f.pixel_count.long(), non_blocking=True)
            if asynchronous:
                rast.status()  # waits for the frame and the copies; raises like a synchronous forward
            torch.cuda.current_stream().synchronize()
            return f, flat, pixc
        finally:
            rast.set_async(was)

    if collect_fragments:
        fwd, flat, pixc = frame_and_outputs(False)
    else:
        try:
            fwd, flat, pixc = frame_and_outputs(True)
        except RuntimeError:
            # an asynchronous frame that outgrew the tile-entry buffer (the status
            # grew it): the synchronous forward redoes it
            fwd, flat, pixc = frame_and_outputs(False)
    t2 = time.perf_counter()
    frags = rast.fragments().to_fragment_data() if collect_fragments else None
    h, w = fwd.alpha_map.shape
    n = fwd.max_weight.numel()
    o1, o2, o3 = h * w * 3, h * w * 4, h * w * 4 + n
    image, alpha = flat[:o1].reshape(h, w, 3), flat[o1:o2].reshape(h, w)
    maxw, area = flat[o2:o3], flat[o3:o3 + n]
    t3 = time.perf_counter()
    LAST_RENDER_D2H_BYTES = image.nbytes + alpha.nbytes + maxw.nbytes + pixc.nbytes + area.nbytes
    if frags is not None:
        LAST_RENDER_D2H_BYTES += sum(np.asarray(a).nbytes for a in (frags.offsets, frags.triangle,
                                                                      frags.weight, frags.depth))
    out = RenderOutput(image=ImageBuffer.trusted(image), alpha_map=alpha, per_triangle_max_weight=maxw,
                       per_triangle_pixel_count=pixc, per_triangle_area=area, fragments=frags)
    LAST_RENDER_TIMES = {"upload": "f32" if ds.vertices.dtype == torch.float32 else "f64",
                         "upload_bytes": sum(t.numel() * t.element_size() for t in
                                             (ds.vertices, ds.opacity, ds.sigma, ds.sh)),
                         "upload_ms": (t1 - t0) * 1e3, "forward_ms": (t2 - t1) * 1e3,
                         "download_ms": (t3 - t2) * 1e3, "total_ms": (time.perf_counter() - t0) * 1e3}
    return out


def render_backward(triangles, intr, pose, mode=0, background=(0.0, 0.0, 0.0), d_image=None,
                    frag_grads=None, tau_cutoff: float = DEFAULT_TAU_CUTOFF,
                    tile_size: int = DEFAULT_TILE_SIZE, active_sh_degree: int = 3,
                    precision: str = "fast") -> GradientSet:
    """Drop-in for trisplat.backward.render_backward (backward.py:93-211)."""
    _require_cuda()
    soup = as_soup(triangles)
    h, w = intr.height, intr.width
    d_np = np.ascontiguousarray(d_image, dtype=np.float64)
    if d_np.shape != (h, w, 3):
        raise ValueError(f"d_image must be {(h, w, 3)}, got {d_np.shape}")
    if not np.isfinite(d_np).all():
        raise ValueError("d_image contains non-finite values")
    rast = default_rasterizer()
    ds = DeviceSoup.from_soup(soup, dtype=_param_dtype(soup))
    rast.forward(ds, intr, pose, mode, background, tau_cutoff, tile_size, active_sh_degree,
                 precision=precision)
    d_dev = torch.as_tensor(d_np, dtype=torch.float32, device="cuda")
    if frag_grads is None:
        return rast.backward(d_dev).to_gradient_set()
    if precision != "fast":
        raise ValueError("frag_grads needs precision='fast'")
    # backward.py:122-136: the layout must be this scene's fragment CSR
    frag_off, fg_dw, fg_dz = frag_grads
    frag_off = np.ascontiguousarray(frag_off, dtype=np.int64)
    fg_dw = np.ascontiguousarray(fg_dw, dtype=np.float64)
    fg_dz = np.ascontiguousarray(fg_dz, dtype=np.float64)
    nf = ctypes.c_int64()
    _lib.check(rast.lib.ts_fragment_offsets(rast._ctx, None, ctypes.byref(nf),
                                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
               "fragment_offsets")
    if frag_off.shape != (h * w + 1,) or len(fg_dw) != nf.value or len(fg_dz) != nf.value:
        raise ValueError("fragment gradients do not match this scene/camera")
    g = rast.backward_fragments(d_dev, torch.from_numpy(frag_off), torch.from_numpy(fg_dw),
                                torch.from_numpy(fg_dz))
    return g.to_gradient_set()


def install(trisplat_module=None):
    """Rebind the reference's render / render_backward to this path.

    The reference imports them by name in several modules (training.py:12,19,
    synthetic.py:14, cli.py:21, backward.py:17), so each binding is patched.
    Returns the list of patched attributes."""
    import importlib
    import sys
    patched = []
    targets = {
        "trisplat": ("render", "render_backward", "project_scene", "build_tile_lists"),
        "trisplat.render": ("render", "project_scene", "build_tile_lists"),
        "trisplat.backward": ("render", "render_backward", "project_scene", "build_tile_lists"),
        "trisplat.training": ("render", "render_backward"),
        "trisplat.synthetic": ("render",),
        "trisplat.cli": ("render",),
    }
    repl = {"render": render, "render_backward": render_backward, "project_scene": project_scene,
            "build_tile_lists": build_tile_lists}
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
