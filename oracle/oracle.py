"""CPU parity oracle for the trisplat rasterizer path (TEST INFRASTRUCTURE ONLY).

Python orchestration over ``liboracle.so`` (``trisplat_oracle.c``), mirroring
the reference call stacks stage by stage:

* ``project_scene``      -- render.py:253-312
* ``build_tile_lists``   -- render.py:349-361
* ``render``             -- render.py:364-432 (+ per-pixel last contributor / count)
* ``render_backward``    -- backward.py:93-211

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module; the product path (``paper_2505_19175_b200``)
never does.  Parity of the C restatement against the live reference is
pinned by the fixtures in ``tests/golden/``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from types import SimpleNamespace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

ALPHA_CLAMP = 0.99
ALPHA_MIN = 1.0 / 255.0
T_MIN = 1e-4
TAU_CONTRIB = 1.0 / 255.0
DEFAULT_TAU_CUTOFF = 1.0 / 255.0

_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int64)
_i64 = ctypes.c_int64
_int = ctypes.c_int
_dbl = ctypes.c_double


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        src = os.path.join(_HERE, "trisplat_oracle.c")
        if not os.path.exists(path) or (os.path.exists(src)
                                         and os.path.getmtime(src) > os.path.getmtime(path)):
            build()
        lib = ctypes.CDLL(path)
        lib.or_project.restype = _i64
        lib.or_project.argtypes = [_i64, _D, _D, _D, _D, _int, _D, _i64, _i64, _D, _D, _int,
                                   _dbl, _int, _I, _D, _D, _D, _D, _D, _D, _D, _D, _D, _D,
                                   _D, _D, _D, _D, _D, _I, _D]
        lib.or_tile_count.restype = _i64
        lib.or_tile_count.argtypes = [_i64, _I, _i64, _i64, _i64, _I]
        lib.or_tile_fill.restype = None
        lib.or_tile_fill.argtypes = [_i64, _I, _i64, _i64, _i64, _I, _I]
        lib.or_rasterize_forward.restype = None
        lib.or_rasterize_forward.argtypes = [_i64, _i64, _i64, _i64, _i64, _I, _I, _D, _D, _D,
                                             _D, _D, _D, _I, _int, _D, _dbl, _int, _I, _D, _D,
                                             _D, _I, _I, _D, _I, _I]
        lib.or_count_fragments.restype = None
        lib.or_count_fragments.argtypes = [_i64, _i64, _i64, _i64, _i64, _I, _I, _D, _D, _D,
                                           _D, _D, _I, _int, _I]
        lib.or_reduce_stats.restype = None
        lib.or_reduce_stats.argtypes = [_i64, _I, _I, _D, _I, _D, _I]
        lib.or_rasterize_backward.restype = None
        lib.or_rasterize_backward.argtypes = [_i64, _i64, _i64, _i64, _i64, _I, _I, _D, _D, _D,
                                              _D, _D, _D, _D, _D, _I, _int, _D, _D, _int, _I,
                                              _D, _D, _D, _D, _D, _D, _D, _D]
        lib.or_backward_chain.restype = None
        lib.or_backward_chain.argtypes = [_i64, _i64, _I, _I, _D, _D, _D, _D, _D, _D, _int, _D,
                                          _D, _D, _D, _D, _D, _D, _D, _D, _int, _D, _D, _D, _D]
        lib.or_set_threads.argtypes = [_int]
        lib.or_get_threads.restype = _int
        _LIB = lib
    return _LIB


def set_threads(n: int):
    _lib().or_set_threads(int(n))


def get_threads() -> int:
    return int(_lib().or_get_threads())


def _p(a):
    if a.dtype == np.int64:
        return a.ctypes.data_as(_I)
    return a.ctypes.data_as(_D)


def mode_flag(mode) -> int:
    """0 = normalized window, 1 = sigmoid (geometry.py:25-29)."""
    if isinstance(mode, (int, np.integer)):
        return int(mode)
    val = getattr(mode, "value", mode)
    return 0 if str(val).lower() == "normalized" else 1


def _f64(a, shape):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(shape))


def _soup_arrays(soup):
    n = len(soup.vertices)
    return (n, _f64(soup.vertices, (n, 3, 3)), _f64(soup.opacity, (n,)),
            _f64(soup.sigma, (n,)), _f64(soup.sh, (n, 16, 3)), bool(getattr(soup, "solid", False)))


def validate_finite(soup):
    """soup.py:67-77 -- first offending triangle per group, groups in order."""
    n, v, o, s, sh, _ = _soup_arrays(soup)
    if n == 0:
        return
    for name, arr in (("vertices", v), ("opacity", o), ("sigma", s), ("sh", sh)):
        bad = ~np.isfinite(arr.reshape(n, -1)).all(axis=1)
        if bad.any():
            raise ValueError(f"non-finite {name} in triangle {int(np.nonzero(bad)[0][0])}")


def _cam(intr):
    return np.array([intr.fx, intr.fy, intr.cx, intr.cy, getattr(intr, "z_near", 0.01)],
                    dtype=np.float64)


def project_scene(soup, intr, pose, mode=0, tau_cutoff=DEFAULT_TAU_CUTOFF, active_sh_degree=3):
    n, v, o, s, sh, solid = _soup_arrays(soup)
    r = _f64(pose.rotation, (3, 3))
    t = _f64(pose.translation, (3,))
    nn = max(n, 1)
    out = SimpleNamespace(
        n_total=n,
        sorted_idx=np.zeros(nn, np.int64), z=np.zeros(nn), xc=np.zeros((nn, 3, 3)),
        q=np.zeros((nn, 3, 2)), nrm=np.zeros((nn, 3, 2)), doff=np.zeros((nn, 3)),
        esign=np.zeros((nn, 3)), phis=np.zeros(nn), area=np.zeros(nn), sig=np.zeros(nn),
        opa=np.zeros(nn), rgb=np.zeros((nn, 3)), raw_rgb=np.zeros((nn, 3)),
        basis=np.zeros((nn, 16)), viewdir=np.zeros((nn, 3)), u_norm=np.zeros(nn),
        bbox=np.zeros((nn, 4), np.int64), area_full=np.zeros(nn))
    cam = _cam(intr)
    m = _lib().or_project(n, _p(v), _p(o), _p(s), _p(sh), int(solid), _p(cam), intr.width,
                          intr.height, _p(r), _p(t), mode_flag(mode), float(tau_cutoff),
                          int(active_sh_degree), _p(out.sorted_idx), _p(out.z), _p(out.xc),
                          _p(out.q), _p(out.nrm), _p(out.doff), _p(out.esign), _p(out.phis),
                          _p(out.area), _p(out.sig), _p(out.opa), _p(out.rgb), _p(out.raw_rgb),
                          _p(out.basis), _p(out.viewdir), _p(out.u_norm), _p(out.bbox),
                          _p(out.area_full))
    for k in ("sorted_idx", "z", "xc", "q", "nrm", "doff", "esign", "phis", "area", "sig",
              "opa", "rgb", "raw_rgb", "basis", "viewdir", "u_norm", "bbox"):
        setattr(out, k, np.ascontiguousarray(getattr(out, k)[:m]))
    out.area_full = out.area_full[:n]
    return out


def build_tile_lists(proj, intr, tile_size=16):
    ntx = (intr.width + tile_size - 1) // tile_size
    nty = (intr.height + tile_size - 1) // tile_size
    counts = np.zeros(ntx * nty, np.int64)
    m = len(proj.sorted_idx)
    bbox = np.ascontiguousarray(proj.bbox, dtype=np.int64).reshape(max(m, 0), 4)
    if m == 0:
        bbox = np.zeros((1, 4), np.int64)
    _lib().or_tile_count(m, _p(bbox), tile_size, ntx, nty, _p(counts))
    start = np.zeros(ntx * nty + 1, np.int64)
    np.cumsum(counts, out=start[1:])
    entry_tri = np.zeros(max(int(start[-1]), 1), np.int64)
    _lib().or_tile_fill(m, _p(bbox), tile_size, ntx, nty, _p(start), _p(entry_tri))
    return ntx, nty, start, entry_tri[:int(start[-1])]


def _nz(a, shape_tail=(), dtype=np.float64):
    """Non-empty buffer (ctypes needs a valid pointer even for zero-length)."""
    if len(a) == 0:
        return np.zeros((1,) + shape_tail, dtype)
    return np.ascontiguousarray(a)


def render(triangles, intr, pose, mode=0, background=(0.0, 0.0, 0.0), collect_fragments=False,
           tau_cutoff=DEFAULT_TAU_CUTOFF, tile_size=16, active_sh_degree=3):
    """render.py:364-432.  Returns a namespace with the RenderOutput fields
    plus ``proj``/``tile_start``/``entry_tri`` and per-pixel ``last_src``
    (source id of the last composited fragment, -1 if none) and ``nfrag``."""
    validate_finite(triangles)
    h, w = intr.height, intr.width
    bg = np.asarray(background, dtype=np.float64).reshape(3).copy()
    mf = mode_flag(mode)
    proj = project_scene(triangles, intr, pose, mf, tau_cutoff, active_sh_degree)
    ntx, nty, tile_start, entry_tri = build_tile_lists(proj, intr, tile_size)
    n_tiles = ntx * nty
    m = len(proj.sorted_idx)
    lib = _lib()
    nrm, doff, phis = _nz(proj.nrm, (3, 2)), _nz(proj.doff, (3,)), _nz(proj.phis)
    sig, opa, rgb = _nz(proj.sig), _nz(proj.opa), _nz(proj.rgb, (3,))
    bbox = _nz(proj.bbox, (4,), np.int64)
    et = _nz(entry_tri, (), np.int64)
    if collect_fragments:
        frag_count = np.zeros((h, w), np.int64)
        lib.or_count_fragments(h, w, tile_size, ntx, n_tiles, _p(tile_start), _p(et), _p(nrm),
                               _p(doff), _p(phis), _p(sig), _p(opa), _p(bbox), mf,
                               _p(frag_count))
        frag_off = np.zeros(h * w + 1, np.int64)
        np.cumsum(frag_count.reshape(-1), out=frag_off[1:])
        nf = int(frag_off[-1])
        frag_m = np.zeros(max(nf, 1), np.int64)
        frag_w = np.zeros(max(nf, 1))
        collect = 1
    else:
        frag_off = np.zeros(1, np.int64)
        frag_m = np.zeros(1, np.int64)
        frag_w = np.zeros(1)
        nf = 0
        collect = 0
    image = np.zeros((h, w, 3))
    alpha_map = np.zeros((h, w))
    ne = len(entry_tri)
    ent_maxw = np.zeros(max(ne, 1))
    ent_pix = np.zeros(max(ne, 1), np.int64)
    last_m = np.zeros(h * w, np.int64)
    nfrag = np.zeros(h * w, np.int64)
    lib.or_rasterize_forward(h, w, tile_size, ntx, n_tiles, _p(tile_start), _p(et), _p(nrm),
                             _p(doff), _p(phis), _p(sig), _p(opa), _p(rgb), _p(bbox), mf, _p(bg),
                             TAU_CONTRIB, collect, _p(frag_off), _p(image), _p(alpha_map),
                             _p(ent_maxw), _p(ent_pix), _p(frag_m), _p(frag_w), _p(last_m),
                             _p(nfrag))
    n = proj.n_total
    maxw = np.zeros(max(n, 1))
    pix = np.zeros(max(n, 1), np.int64)
    if ne:
        lib.or_reduce_stats(ne, _p(et), _p(_nz(proj.sorted_idx, (), np.int64)), _p(ent_maxw),
                            _p(ent_pix), _p(maxw), _p(pix))
    sidx = proj.sorted_idx
    last_src = np.where(last_m >= 0, sidx[np.maximum(last_m, 0)] if m else -1, -1)
    fragments = None
    if collect_fragments:
        fragments = SimpleNamespace(offsets=frag_off, triangle=sidx[frag_m[:nf]],
                                    weight=frag_w[:nf], depth=proj.z[frag_m[:nf]])
    return SimpleNamespace(
        image=np.clip(image, 0.0, 1.0), image_unclipped=image, alpha_map=alpha_map,
        per_triangle_max_weight=maxw[:n], per_triangle_pixel_count=pix[:n],
        per_triangle_area=proj.area_full, fragments=fragments, proj=proj,
        tile_start=tile_start, entry_tri=entry_tri, ent_maxw=ent_maxw[:ne], ent_pix=ent_pix[:ne],
        last_src=last_src.reshape(h, w), last_m=last_m.reshape(h, w),
        nfrag=nfrag.reshape(h, w))


def render_backward(triangles, intr, pose, mode=0, background=(0.0, 0.0, 0.0), d_image=None,
                    frag_grads=None, tau_cutoff=DEFAULT_TAU_CUTOFF, tile_size=16,
                    active_sh_degree=3, return_screen=False):
    """backward.py:93-211.  Returns a namespace with d_vertices (N,3,3),
    d_opacity (N,), d_sigma (N,), d_sh (N,16,3)."""
    validate_finite(triangles)
    h, w = intr.height, intr.width
    d_image = np.ascontiguousarray(d_image, dtype=np.float64)
    if d_image.shape != (h, w, 3):
        raise ValueError(f"d_image must be {(h, w, 3)}, got {d_image.shape}")
    if not np.isfinite(d_image).all():
        raise ValueError("d_image contains non-finite values")
    bg = np.asarray(background, dtype=np.float64).reshape(3).copy()
    mf = mode_flag(mode)
    n, v, o, s, sh, solid = _soup_arrays(triangles)
    proj = project_scene(triangles, intr, pose, mf, tau_cutoff, active_sh_degree)
    ntx, nty, tile_start, entry_tri = build_tile_lists(proj, intr, tile_size)
    n_tiles = ntx * nty
    lib = _lib()
    nrm, doff, phis = _nz(proj.nrm, (3, 2)), _nz(proj.doff, (3,)), _nz(proj.phis)
    sig, opa, rgb = _nz(proj.sig), _nz(proj.opa), _nz(proj.rgb, (3,))
    q = _nz(proj.q, (3, 2))
    esign = _nz(proj.esign, (3,))
    bbox = _nz(proj.bbox, (4,), np.int64)
    et = _nz(entry_tri, (), np.int64)
    if frag_grads is not None:
        frag_off, fg_dw, fg_dz = frag_grads
        frag_off = np.ascontiguousarray(frag_off, dtype=np.int64)
        fg_dw = np.ascontiguousarray(fg_dw, dtype=np.float64)
        fg_dz = np.ascontiguousarray(fg_dz, dtype=np.float64)
        count = np.zeros((h, w), np.int64)
        lib.or_count_fragments(h, w, tile_size, ntx, n_tiles, _p(tile_start), _p(et), _p(nrm),
                               _p(doff), _p(phis), _p(sig), _p(opa), _p(bbox), mf, _p(count))
        expect = np.zeros(h * w + 1, np.int64)
        np.cumsum(count.reshape(-1), out=expect[1:])
        if frag_off.shape != expect.shape or not np.array_equal(frag_off, expect) \
                or len(fg_dw) != expect[-1] or len(fg_dz) != expect[-1]:
            raise ValueError("fragment gradients do not match this scene/camera")
        has_fg = 1
        fg_dw, fg_dz = _nz(fg_dw), _nz(fg_dz)
    else:
        frag_off = np.zeros(1, np.int64)
        fg_dw = np.zeros(1)
        fg_dz = np.zeros(1)
        has_fg = 0
    ne = len(entry_tri)
    gq_e = np.zeros((max(ne, 1), 3, 2))
    go_e = np.zeros(max(ne, 1))
    gsig_e = np.zeros(max(ne, 1))
    grgb_e = np.zeros((max(ne, 1), 3))
    gphis_e = np.zeros(max(ne, 1))
    gz_e = np.zeros(max(ne, 1))
    lib.or_rasterize_backward(h, w, tile_size, ntx, n_tiles, _p(tile_start), _p(et), _p(q),
                              _p(nrm), _p(doff), _p(esign), _p(phis), _p(sig), _p(opa), _p(rgb),
                              _p(bbox), mf, _p(bg), _p(d_image), has_fg, _p(frag_off), _p(fg_dw),
                              _p(fg_dz), _p(gq_e), _p(go_e), _p(gsig_e), _p(grgb_e), _p(gphis_e),
                              _p(gz_e))
    m = len(proj.sorted_idx)
    if return_screen:
        sg = np.zeros((n, 13))
        src = proj.sorted_idx[entry_tri] if ne else np.zeros(0, np.int64)
        for j, arr in enumerate((gq_e.reshape(-1, 6)[:ne], go_e[:ne, None], gsig_e[:ne, None],
                                 grgb_e.reshape(-1, 3)[:ne], gphis_e[:ne, None], gz_e[:ne, None])):
            off = (0, 6, 7, 8, 11, 12)[j]
            np.add.at(sg[:, off:off + arr.shape[1]], src, arr)
        return sg
    grads = SimpleNamespace(d_vertices=np.zeros((n, 3, 3)), d_opacity=np.zeros(n),
                            d_sigma=np.zeros(n), d_sh=np.zeros((n, 16, 3)))
    if m == 0:
        return grads
    cam = _cam(intr)
    r = _f64(pose.rotation, (3, 3))
    lib.or_backward_chain(m, ne, _p(et), _p(proj.sorted_idx), _p(gq_e), _p(go_e), _p(gsig_e),
                          _p(grgb_e), _p(gphis_e), _p(gz_e), mf, _p(cam), _p(r), _p(proj.q),
                          _p(proj.xc), _p(proj.raw_rgb), _p(proj.basis), _p(proj.viewdir),
                          _p(proj.u_norm), _p(sh), int(active_sh_degree),
                          _p(grads.d_vertices), _p(grads.d_opacity), _p(grads.d_sigma),
                          _p(grads.d_sh))
    return grads
