"""Adaptive density control on device-resident triangles:
drop-ins for the reference's ``ViewStats``, ``prune``, ``sample_candidates``
and ``densify_step`` (trisplat/density.py:27-263) over a ``DeviceSoup``.

The array work runs in ts_density.cu through the C ABI: statistics folded per
view, prune flags + in-order compaction of the survivors, sampling weights +
exponential keys + a stable radix sort, per-pick source / mean area /
degeneracy, the row gathers of the new soup and the children's vertices.  The
host keeps what is inherently sequential and cheap: the caller's numpy
Generator (rng.exponential per sampling round and the clones' uniform draws,
in the reference's order -- so a seeded run picks the same triangles) and the
pick loop of density.py:209-245, which is a prefix sum over the picks' costs
(3 for a split, 1 for a clone) until fewer than three additions remain.

Statistics come from the rasterizer's forward outputs (fp32 max weight and
area per triangle); aggregation and every threshold comparison is fp64 on
those values, in the order the views were first recorded.
"""
from __future__ import annotations

import ctypes
import enum
import math
from dataclasses import dataclass

import numpy as np


class SampleCriterion(enum.Enum):
    INVERSE_SIGMA = "inverse_sigma"
    OPACITY = "opacity"


@dataclass
class DensifyConfig:
    """Same fields and defaults as the reference's DensifyConfig (config.py:12-30)."""
    tau_prune: float = 0.022
    min_views: int = 2
    min_pixels: int = 2
    opacity_dead: float = 0.014
    growth_rate: float = 0.30
    tau_small: float = 24.0
    max_noise_factor: float = 1.5
    interval: int = 500
    start_iter: int = 500
    stop_iter: int = 25000

    def __post_init__(self):
        if not 0.0 <= self.growth_rate:
            raise ValueError("growth_rate must be >= 0")
        if self.interval <= 0:
            raise ValueError("interval must be positive")


def _vp(t):
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)


def _ctx(rasterizer):
    from .rasterizer import default_rasterizer
    r = rasterizer or default_rasterizer()
    return r, r.lib, r._ctx


def _stream(stream):
    import torch
    return ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)


def _dtype_code(soup):
    import torch
    if soup.vertices.dtype == torch.float64:
        return 1
    if soup.vertices.dtype == torch.float32:
        return 0
    raise TypeError("DeviceSoup parameters must be float32 or float64")


def reduce_across_ranks(max_weight, views, area, n_views: int, group=None):
    """View-parallel statistics: each rank aggregates the views it
    rendered; MAX of the peak weights, SUM of the covering-view counts, area
    sums and view counts over the ranks (in place; returns the global view
    count).  With replicated soups and identically seeded Generators every rank
    then takes the same densify_step."""
    import torch
    import torch.distributed as dist
    dist.all_reduce(max_weight, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(views, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(area, op=dist.ReduceOp.SUM, group=group)
    nv = torch.tensor([int(n_views)], dtype=torch.int64, device=max_weight.device)
    dist.all_reduce(nv, op=dist.ReduceOp.SUM, group=group)
    return int(nv.item())


class DeviceViewStats:
    """ViewStats (density.py:27-71) with the per-view arrays on the device.
    Re-recording a view replaces its arrays and keeps its position.  With
    ``group`` set (torch.distributed), the aggregates and the view count are
    reduced over the ranks, each holding the views it rendered."""

    def __init__(self, n_triangles: int, group=None):
        self.n_triangles = int(n_triangles)
        self.per_view: dict = {}  # view id -> (max weight f32, pixel count i32, area f32, min_pixels)
        self.group = group
        self._views_total = None

    @classmethod
    def empty(cls, n_triangles: int, group=None) -> "DeviceViewStats":
        return cls(n_triangles, group)

    def update(self, view_id, output, min_pixels: int = 2):
        """output: a ForwardResult (device tensors) or a RenderOutput (numpy)."""
        import torch
        if hasattr(output, "max_weight"):
            mw, pc, ar = output.max_weight, output.pixel_count, output.area
        else:
            mw, pc, ar = output.per_triangle_max_weight, output.per_triangle_pixel_count, output.per_triangle_area
        if len(mw) != self.n_triangles:
            raise ValueError("render output population does not match stats")
        dev = lambda a, dt: torch.as_tensor(a).to(device="cuda", dtype=dt).contiguous().clone()  # noqa: E731
        self.per_view[view_id] = (dev(mw, torch.float32), dev(pc, torch.int32), dev(ar, torch.float32),
                                  int(min_pixels))

    @property
    def n_views(self) -> int:
        """Views recorded (over all ranks once aggregated with a group)."""
        return len(self.per_view) if self.group is None or self._views_total is None else self._views_total

    def aggregate(self, rasterizer=None, stream=None):
        """(max weight f64, covering views i32, area sum f64) device tensors."""
        import torch
        from . import _lib
        _, lib, ctx = _ctx(rasterizer)
        n = self.n_triangles
        mw = torch.zeros(n, dtype=torch.float64, device="cuda")
        views = torch.zeros(n, dtype=torch.int32, device="cuda")
        area = torch.zeros(n, dtype=torch.float64, device="cuda")
        st = _stream(stream)
        for k, (w, pc, ar, mp) in enumerate(self.per_view.values()):
            _lib.check(lib.ts_view_stats_accumulate(ctx, n, _vp(w), _vp(pc), _vp(ar), mp, int(k == 0), _vp(mw),
                                                    _vp(views), _vp(area), st), "view_stats_accumulate")
        if self.group is not None:
            self._views_total = reduce_across_ranks(mw, views, area, len(self.per_view), self.group)
        return mw, views, area

    def max_weight(self, **kw):
        return self.aggregate(**kw)[0]

    def covering_views(self, **kw):
        return self.aggregate(**kw)[1].to(dtype=__import__("torch").int64)

    def mean_area(self, **kw):
        a = self.aggregate(**kw)[2]  # (sets the global view count with a group)
        # a tensor divisor: a true division (torch turns a scalar divisor into a reciprocal product)
        return a / a.new_full(a.shape, float(max(self.n_views, 1)))


def _prune_dev(soup, stats, cfg, rasterizer, stream):
    import torch
    from . import _lib
    if stats.n_triangles != len(soup):
        raise ValueError("stats population does not match soup")
    _, lib, ctx = _ctx(rasterizer)
    n = len(soup)
    acc = stats.aggregate(rasterizer, stream)
    flags = torch.empty(n, dtype=torch.uint8, device="cuda")
    kept = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    n_kept = torch.zeros(1, dtype=torch.int64, device="cuda")
    _lib.check(lib.ts_prune_mark(ctx, n, _vp(acc[0]), _vp(acc[1]), _vp(soup.opacity), _dtype_code(soup),
                                 float(cfg.tau_prune), int(cfg.min_views), float(cfg.opacity_dead), _vp(flags),
                                 _vp(kept), _vp(n_kept), _stream(stream)), "prune_mark")
    f = flags.cpu().numpy()
    alive = int(n_kept.item())
    report = {
        "low_weight": np.nonzero(f & 1)[0].tolist(),
        "few_views": np.nonzero(f & 2)[0].tolist(),
        "dead_opacity": np.nonzero(f & 4)[0].tolist(),
        "n_removed": int(n - alive),
        "kept_index": kept[:alive].cpu().numpy(),
    }
    return acc, kept[:alive], report


def _gather_soup(soup, origin_dev, n_out, rasterizer, stream):
    import torch
    from . import _lib
    from .rasterizer import DeviceSoup
    _, lib, ctx = _ctx(rasterizer)
    dt = soup.vertices.dtype
    es = 8 if dt == torch.float64 else 4
    new = DeviceSoup(torch.empty((n_out, 3, 3), dtype=dt, device="cuda"), torch.empty(n_out, dtype=dt, device="cuda"),
                     torch.empty(n_out, dtype=dt, device="cuda"), torch.empty((n_out, 16, 3), dtype=dt, device="cuda"),
                     soup.solid)
    st = _stream(stream)
    for src, dst, w in ((soup.vertices, new.vertices, 9), (soup.opacity, new.opacity, 1),
                        (soup.sigma, new.sigma, 1), (soup.sh, new.sh, 48)):
        _lib.check(lib.ts_gather_rows(ctx, n_out, _vp(origin_dev), _vp(src), _vp(dst), w, es, st), "gather_rows")
    return new


def prune(soup, stats: DeviceViewStats, cfg, rasterizer=None, stream=None):
    """density.py:74-94 on the device: returns (survivors DeviceSoup, report)."""
    _, kept, report = _prune_dev(soup, stats, cfg, rasterizer, stream)
    return _gather_soup(soup, kept, int(kept.numel()), rasterizer, stream), report


def _sample_dev(soup, n_pool, pool_dev, kept_dev, count, criterion, rng, rasterizer, stream):
    import torch
    from . import _lib
    _, lib, ctx = _ctx(rasterizer)
    expo = torch.as_tensor(rng.exponential(size=n_pool), dtype=torch.float64).to("cuda")
    picked = torch.empty(max(count, 1), dtype=torch.int64, device="cuda")
    inverse = criterion is SampleCriterion.INVERSE_SIGMA
    param = soup.sigma if inverse else soup.opacity
    _lib.check(lib.ts_sample_candidates(ctx, n_pool, _vp(pool_dev), _vp(kept_dev), _vp(param), _dtype_code(soup),
                                        0 if inverse else 1, _vp(expo), count, _vp(picked), _stream(stream)),
               "sample_candidates")
    return picked[:count]


def sample_candidates(soup, count: int, criterion: SampleCriterion, rng: np.random.Generator, rasterizer=None,
                      stream=None) -> np.ndarray:
    """density.py:103-120: weighted sampling without replacement (exponential
    keys, stable sort) of ``count`` triangles of a DeviceSoup."""
    n = len(soup)
    count = min(count, n)
    if count <= 0:
        return np.zeros(0, dtype=np.int64)
    return _sample_dev(soup, n, None, None, count, criterion, rng, rasterizer, stream).cpu().numpy()


def step_criterion(iteration: int, cfg) -> SampleCriterion:
    step = (iteration - cfg.start_iter) // cfg.interval
    return SampleCriterion.INVERSE_SIGMA if step % 2 == 0 else SampleCriterion.OPACITY


def _decide(elig: np.ndarray, remaining: int):
    """The pick loop of density.py:221-245 as a prefix sum: returns (processed
    mask, split mask, remaining after).  While at least three additions remain a
    pick splits iff it is eligible (mean area >= tau_small, not degenerate);
    after that every processed pick is a clone of cost 1."""
    k = len(elig)
    cost = np.where(elig, 3, 1)
    before = remaining - np.concatenate([[0], np.cumsum(cost)[:-1]]) if k else np.zeros(0, np.int64)
    low = np.nonzero(before < 3)[0]
    split = elig.copy()
    proc = np.ones(k, dtype=bool)
    if len(low) == 0:
        return proc, split, int(remaining - cost.sum())
    kk = int(low[0])
    rem = int(before[kk])
    for j in range(kk, k):
        if rem <= 0:
            proc[j:] = False
            break
        split[j] = False
        rem -= 1
    split &= proc
    return proc, split, rem


def densify_step(soup, stats: DeviceViewStats, iteration: int, cfg, rng: np.random.Generator, rasterizer=None,
                 stream=None):
    """One prune-and-grow step (density.py:180-263) on a DeviceSoup.  Returns
    (new DeviceSoup, report) with the reference's report keys; ``origin`` maps
    each output triangle to its source index (numpy int64)."""
    import torch
    from . import _lib
    n0 = len(soup)
    identity = np.arange(n0, dtype=np.int64)
    scheduled = (cfg.start_iter <= iteration <= cfg.stop_iter
                 and (iteration - cfg.start_iter) % cfg.interval == 0)
    if not scheduled or n0 == 0:
        return soup, {"scheduled": False, "origin": identity, "n_before": n0, "n_after": n0}
    _, lib, ctx = _ctx(rasterizer)
    st = _stream(stream)
    acc, kept_dev, prune_report = _prune_dev(soup, stats, cfg, rasterizer, stream)
    kept = prune_report["kept_index"]
    alive = len(kept)
    if alive == 0:
        empty = torch.zeros(0, dtype=torch.int64, device="cuda")
        return _gather_soup(soup, empty, 0, rasterizer, stream), {
            "scheduled": True, "origin": np.zeros(0, np.int64), "prune": prune_report, "n_before": n0,
            "n_after": 0, "n_split": 0, "n_clone": 0}
    criterion = step_criterion(iteration, cfg)
    n_add = math.ceil(cfg.growth_rate * alive)
    removed = np.zeros(alive, dtype=bool)
    ch_parent, ch_code, uniforms = [], [], []
    n_split = n_clone = n_noise = 0
    remaining = n_add
    dcode = _dtype_code(soup)
    while remaining > 0:
        pool = np.nonzero(~removed)[0]
        if len(pool) == 0:
            break
        count = min(remaining, len(pool))
        pool_dev = None if len(pool) == alive else torch.as_tensor(pool, dtype=torch.int64).to("cuda")
        picked = _sample_dev(soup, len(pool), pool_dev, kept_dev, count, criterion, rng, rasterizer, stream)
        src = torch.empty(count, dtype=torch.int64, device="cuda")
        ma = torch.empty(count, dtype=torch.float64, device="cuda")
        degen = torch.empty(count, dtype=torch.uint8, device="cuda")
        _lib.check(lib.ts_pick_info(ctx, count, _vp(picked), _vp(pool_dev), _vp(kept_dev), _vp(acc[2]),
                                    stats.n_views, _vp(soup.vertices), dcode, _vp(src), _vp(ma), _vp(degen), st),
                   "pick_info")
        local = pool[picked.cpu().numpy()]
        src_h, ma_h, deg_h = src.cpu().numpy(), ma.cpu().numpy(), degen.cpu().numpy().astype(bool)
        proc, split, remaining = _decide((ma_h >= cfg.tau_small) & ~deg_h, remaining)
        removed[local[split]] = True
        clone = proc & ~split
        noisy = clone & ~deg_h
        nn = int(noisy.sum())
        if nn:
            uniforms.append(rng.random(6 * nn))
        # children in pick order: 4 corners per split, one row per clone
        per = np.where(split, 4, 1)[proc]
        par = np.repeat(src_h[proc], per)
        code = np.full(len(par), -1, dtype=np.int32)
        starts = np.concatenate([[0], np.cumsum(per)[:-1]]).astype(np.int64)
        sp = split[proc]
        for c in range(4):
            code[starts[sp] + c] = c
        nz = noisy[proc]
        code[starts[nz]] = 4 + n_noise + np.arange(nn, dtype=np.int32)
        n_noise += nn
        ch_parent.append(par)
        ch_code.append(code)
        n_split += int(split.sum())
        n_clone += int(clone.sum())
    base = kept[~removed]
    par = np.concatenate(ch_parent) if ch_parent else np.zeros(0, np.int64)
    origin = np.concatenate([base, par]).astype(np.int64)
    origin_dev = torch.as_tensor(origin).to("cuda")
    new = _gather_soup(soup, origin_dev, len(origin), rasterizer, stream)
    n_child = len(par)
    if n_child:
        code_dev = torch.as_tensor(np.concatenate(ch_code)).to("cuda")
        uni_dev = torch.as_tensor(np.concatenate(uniforms) if uniforms else np.zeros(1)).to("cuda")
        es = new.vertices.element_size()
        _lib.check(lib.ts_child_vertices(ctx, n_child, ctypes.c_void_p(origin_dev.data_ptr() + 8 * len(base)),
                                         _vp(code_dev), _vp(uni_dev), float(cfg.max_noise_factor),
                                         _vp(soup.vertices),
                                         ctypes.c_void_p(new.vertices.data_ptr() + es * 9 * len(base)), dcode, st),
                   "child_vertices")
    report = {
        "scheduled": True,
        "prune": prune_report,
        "criterion": criterion,
        "n_before": n0,
        "n_after": len(origin),
        "n_add": n_add,
        "n_split": n_split,
        "n_clone": n_clone,
        "origin": origin,
    }
    return new, report
