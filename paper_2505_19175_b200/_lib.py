"""ctypes binding of the C ABI declared in include/trisplat_b200.h.

The shared library is built in-tree (``python -m paper_2505_19175_b200.build``
or ``__graft_entry__.build()``).  There is no CPU fallback: if the library is
missing or no CUDA device is present, loading fails loudly.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TRISPLAT_B200_LIB") or os.path.join(HERE, "libtrisplat_b200.so")

TS_OK = 0
TS_ERR_INVALID_ARG = -1
TS_ERR_NONFINITE = -5
TS_ERR_FRAGMENTS = -7
TS_ERR_CAPACITY = -9
TS_DUMP_SORTED_IDX = 1
TS_DUMP_TILE_START = 2
TS_DUMP_ENTRY_RANK = 3
TS_DUMP_BBOX = 4
TS_DUMP_DEPTH = 5
TS_DUMP_SGRAD = 6
TS_DUMP_FRAGREC = 7
TS_DUMP_PROJECTION = 8
PROJ_ROW = 64


class TsCamera(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_double), ("fy", ctypes.c_double), ("cx", ctypes.c_double),
                ("cy", ctypes.c_double), ("z_near", ctypes.c_double),
                ("R", ctypes.c_double * 9), ("t", ctypes.c_double * 3),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class TsOptions(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("sh_degree", ctypes.c_int32),
                ("tile_size", ctypes.c_int32), ("solid", ctypes.c_int32),
                ("tau_cutoff", ctypes.c_double), ("tau_contrib", ctypes.c_double),
                ("background", ctypes.c_double * 3), ("precision", ctypes.c_int32),
                ("param_dtype", ctypes.c_int32), ("validate", ctypes.c_int32),
                ("keep_backward", ctypes.c_int32)]


class TsSoup(ctypes.Structure):
    _fields_ = [("vertices", ctypes.c_void_p), ("opacity", ctypes.c_void_p),
                ("sigma", ctypes.c_void_p), ("sh", ctypes.c_void_p), ("n", ctypes.c_int64)]


class TsForwardOut(ctypes.Structure):
    _fields_ = [("image", ctypes.c_void_p), ("alpha_map", ctypes.c_void_p),
                ("max_weight", ctypes.c_void_p), ("pixel_count", ctypes.c_void_p),
                ("area", ctypes.c_void_p), ("last_src", ctypes.c_void_p),
                ("n_frag", ctypes.c_void_p)]


class TsForwardResult(ctypes.Structure):
    _fields_ = [("n_visible", ctypes.c_int64), ("n_entries", ctypes.c_int64),
                ("n_flagged", ctypes.c_int64), ("err_index", ctypes.c_int64 * 4)]


class TsGrads(ctypes.Structure):
    _fields_ = [("d_vertices", ctypes.c_void_p), ("d_opacity", ctypes.c_void_p),
                ("d_sigma", ctypes.c_void_p), ("d_sh", ctypes.c_void_p)]


EXPORTS = ["ts_context_create", "ts_context_destroy", "ts_error_string", "ts_version",
           "ts_forward", "ts_backward", "ts_debug_copy", "ts_launch_count", "ts_profile",
           "ts_stage_times", "ts_flagged_pixels", "ts_fragment_offsets", "ts_collect_fragments",
           "ts_backward_fragments", "ts_set_async", "ts_forward_status", "ts_set_option", "ts_photometric_loss",
           "ts_ssim", "ts_adam_step", "ts_distortion_loss", "ts_fragment_depth",
           "ts_normal_loss", "ts_view_stats_accumulate", "ts_prune_mark", "ts_sample_candidates",
           "ts_pick_info", "ts_gather_rows", "ts_child_vertices", "ts_ply_pack", "ts_ply_unpack",
           "ts_tile_lists", "ts_backward_chunked", "ts_backward_screen", "ts_chain_views",
           "ts_pending_views", "ts_pack_f32", "ts_upload_f32", "ts_reserve", "ts_workspace_bytes"]
TS_OPT_LEGACY_BINNING = 1
TS_OPT_TILE_BACKWARD = 2
STAGES = ["preprocess", "depth_sort", "binning", "blend", "fixup", "blend_bwd", "chain_bwd"]

_LIB = None


def load(path: str = LIB_PATH):
    """Load the library and declare every exported signature."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is not built; run __graft_entry__.build() "
                           "(python -m paper_2505_19175_b200.build)")
    lib = ctypes.CDLL(path)
    P = ctypes.POINTER
    lib.ts_context_create.argtypes = [P(ctypes.c_void_p), ctypes.c_int]
    lib.ts_context_create.restype = ctypes.c_int
    lib.ts_context_destroy.argtypes = [ctypes.c_void_p]
    lib.ts_context_destroy.restype = ctypes.c_int
    lib.ts_error_string.argtypes = [ctypes.c_int]
    lib.ts_error_string.restype = ctypes.c_char_p
    lib.ts_version.argtypes = []
    lib.ts_version.restype = ctypes.c_char_p
    lib.ts_forward.argtypes = [ctypes.c_void_p, P(TsCamera), P(TsOptions), P(TsSoup),
                               P(TsForwardOut), P(TsForwardResult), ctypes.c_void_p]
    lib.ts_forward.restype = ctypes.c_int
    lib.ts_backward.argtypes = [ctypes.c_void_p, ctypes.c_void_p, P(TsGrads), ctypes.c_int,
                                ctypes.c_void_p]
    lib.ts_backward.restype = ctypes.c_int
    lib.ts_fragment_offsets.argtypes = [ctypes.c_void_p, ctypes.c_void_p, P(ctypes.c_int64), ctypes.c_void_p]
    lib.ts_fragment_offsets.restype = ctypes.c_int
    lib.ts_collect_fragments.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_void_p]
    lib.ts_collect_fragments.restype = ctypes.c_int
    lib.ts_backward_fragments.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p, P(TsGrads), ctypes.c_int,
                                          ctypes.c_void_p]
    lib.ts_backward_fragments.restype = ctypes.c_int
    lib.ts_set_async.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.ts_set_async.restype = ctypes.c_int
    lib.ts_forward_status.argtypes = [ctypes.c_void_p, P(TsForwardResult), ctypes.c_void_p]
    lib.ts_forward_status.restype = ctypes.c_int
    lib.ts_set_option.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64]
    lib.ts_set_option.restype = ctypes.c_int
    lib.ts_debug_copy.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                  ctypes.c_size_t, ctypes.c_void_p]
    lib.ts_debug_copy.restype = ctypes.c_int
    lib.ts_photometric_loss.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p]
    lib.ts_photometric_loss.restype = ctypes.c_int
    lib.ts_ssim.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                            ctypes.c_void_p, ctypes.c_void_p]
    lib.ts_ssim.restype = ctypes.c_int
    lib.ts_adam_step.argtypes = [ctypes.c_void_p] + [ctypes.c_void_p] * 4 + [ctypes.c_int64, P(TsGrads),
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                 P(ctypes.c_double), ctypes.c_void_p, ctypes.c_void_p]
    lib.ts_adam_step.restype = ctypes.c_int
    lib.ts_distortion_loss.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_int64] + \
        [ctypes.c_void_p] * 4
    lib.ts_distortion_loss.restype = ctypes.c_int
    lib.ts_fragment_depth.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
    lib.ts_fragment_depth.restype = ctypes.c_int
    lib.ts_normal_loss.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, P(TsCamera),
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    lib.ts_normal_loss.restype = ctypes.c_int
    V, I64, I, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    lib.ts_view_stats_accumulate.argtypes = [V, I64, V, V, V, I, I, V, V, V, V]
    lib.ts_prune_mark.argtypes = [V, I64, V, V, V, I, D, I, D, V, V, V, V]
    lib.ts_sample_candidates.argtypes = [V, I64, V, V, V, I, I, V, I64, V, V]
    lib.ts_pick_info.argtypes = [V, I64, V, V, V, V, I64, V, I, V, V, V, V]
    lib.ts_gather_rows.argtypes = [V, I64, V, V, V, I, I, V]
    lib.ts_child_vertices.argtypes = [V, I64, V, V, V, D, V, V, I, V]
    lib.ts_ply_pack.argtypes = [V, V, V, I, I64, V, V, V]
    lib.ts_ply_unpack.argtypes = [V, V, I64, V, I64, D, I, V, V, V, V, V, V]
    lib.ts_tile_lists.argtypes = [V, V, I64, I, I, I, V, V, P(ctypes.c_int64), V]
    lib.ts_tile_lists.restype = ctypes.c_int
    lib.ts_backward_chunked.argtypes = [V, V, P(TsGrads), I, I, P(ctypes.c_int64), P(ctypes.c_void_p), V]
    lib.ts_backward_chunked.restype = ctypes.c_int
    lib.ts_backward_screen.argtypes = [V, V, V]
    lib.ts_backward_screen.restype = ctypes.c_int
    lib.ts_chain_views.argtypes = [V, P(TsGrads), I, I, P(ctypes.c_int64), P(ctypes.c_void_p), V]
    lib.ts_chain_views.restype = ctypes.c_int
    lib.ts_pack_f32.argtypes = [V, V, ctypes.c_int64, I]
    lib.ts_pack_f32.restype = ctypes.c_int
    lib.ts_upload_f32.argtypes = [V, ctypes.c_int64, V, V, ctypes.c_int64, I, I]
    lib.ts_upload_f32.restype = ctypes.c_int
    lib.ts_reserve.argtypes = [V, ctypes.c_int64, I, I, ctypes.c_int64, I]
    lib.ts_reserve.restype = ctypes.c_int
    lib.ts_workspace_bytes.argtypes = [V]
    lib.ts_workspace_bytes.restype = ctypes.c_int64
    lib.ts_pending_views.argtypes = [V]
    lib.ts_pending_views.restype = ctypes.c_int
    for nm in ("ts_ply_pack", "ts_ply_unpack", "ts_view_stats_accumulate", "ts_prune_mark", "ts_sample_candidates", "ts_pick_info",
               "ts_gather_rows", "ts_child_vertices"):
        getattr(lib, nm).restype = ctypes.c_int
    lib.ts_launch_count.argtypes = [ctypes.c_void_p]
    lib.ts_launch_count.restype = ctypes.c_int64
    lib.ts_profile.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.ts_profile.restype = ctypes.c_int
    lib.ts_stage_times.argtypes = [ctypes.c_void_p, P(ctypes.c_float), ctypes.c_int]
    lib.ts_stage_times.restype = ctypes.c_int
    lib.ts_flagged_pixels.argtypes = [ctypes.c_void_p, P(ctypes.c_int64)]
    lib.ts_flagged_pixels.restype = ctypes.c_int
    _LIB = lib
    return lib


def check(rc: int, what: str = ""):
    if rc != TS_OK:
        msg = load().ts_error_string(rc).decode()
        raise RuntimeError(f"trisplat_b200 {what} failed: {msg} ({rc})")
