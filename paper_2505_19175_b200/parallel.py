"""View-parallel training step.

A batch of camera views is split into contiguous shards, one per rank; every
rank renders its views against replicated triangle parameters and
accumulates their gradients into ONE flat fp32 buffer
``[d_vertices | d_opacity | d_sigma | d_sh]`` (59 values per triangle), then a
single all-reduce (SUM) makes every rank hold the gradient of the whole batch.
A frame is never split.  The batch gradient is the sum of per-view
``render_backward`` results because the gradient is linear in ``d_image``
(test_backward.py:44-55 checks that linearity on the reference).

The gradient function is injected, so the same sharding / reduction logic runs
with the B200 rasterizer (NCCL) and, in the CPU tests, with the oracle (gloo).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import torch
import torch.distributed as dist


def shard(n: int, world: int, rank: int) -> range:
    """Contiguous shard of ``n`` items for ``rank`` of ``world`` (sizes differ by at most 1)."""
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return range(lo, lo + base + (1 if rank < rem else 0))


def flat_grad_size(n_triangles: int) -> int:
    return 59 * n_triangles


def chunk_bounds(n: int, k: int, align: int = 64) -> list:
    """k contiguous triangle ranges of [0, n): interior bounds rounded down to a
    multiple of ``align`` (ts_backward_chunked's requirement), non-decreasing
    (ranges may be empty for small n)."""
    k = max(1, int(k))
    b = [0]
    for i in range(1, k):
        b.append((i * n // k) // align * align)
    b.append(n)
    return b


def bucket_slices(flat: torch.Tensor, n: int, lo: int, hi: int) -> list:
    """Views of the flat [vertices 9n | opacity n | sigma n | sh 48n] gradient
    holding triangles [lo, hi) of every group."""
    return [flat[9 * lo:9 * hi], flat[9 * n + lo:9 * n + hi], flat[10 * n + lo:10 * n + hi],
            flat[11 * n + 48 * lo:11 * n + 48 * hi]]


class BucketedAllReduce:
    """SUM all-reduce of the flat gradient, one triangle-range bucket at a
    time: bucket k starts once ``event`` k fires (CUDA: on a side stream that
    waits on the event, so the collective overlaps the producer's next range;
    gloo / no event: at once).  ``wait()`` makes the current stream wait for
    every bucket."""

    def __init__(self, flat: torch.Tensor, n: int, bounds: list, comm_stream=None):
        self.flat, self.n, self.bounds = flat, n, bounds
        self.comm = comm_stream
        self.works = []

    def launch(self, k: int, event=None):
        lo, hi = self.bounds[k], self.bounds[k + 1]
        if hi <= lo:
            return
        if self.comm is not None:
            if event is not None:
                self.comm.wait_event(event)
            with torch.cuda.stream(self.comm):
                for sl in bucket_slices(self.flat, self.n, lo, hi):
                    self.works.append(dist.all_reduce(sl, op=dist.ReduceOp.SUM, async_op=True))
        else:
            for sl in bucket_slices(self.flat, self.n, lo, hi):
                self.works.append(dist.all_reduce(sl, op=dist.ReduceOp.SUM, async_op=True))

    def wait(self):
        for w in self.works:
            w.wait()
        self.works = []


def allreduce_(buf: torch.Tensor, bucket_bytes: int = 64 << 20):
    """In-place SUM all-reduce, bucketed so large buffers overlap in NCCL."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return buf
    step = max(1, bucket_bytes // buf.element_size())
    works = [dist.all_reduce(buf[i:i + step], op=dist.ReduceOp.SUM, async_op=True)
             for i in range(0, buf.numel(), step)]
    for w in works:
        w.wait()
    return buf


@dataclass
class StepResult:
    grads: torch.Tensor       # flat fp32 gradient of the whole batch (replicated)
    local_views: Sequence[int]


def train_step(grad_fn: Callable[[int, torch.Tensor, bool], None], n_views: int,
               grads: torch.Tensor, world: int | None = None, rank: int | None = None,
               last_grad_fn=None, n_triangles: int | None = None, n_buckets: int = 8,
               comm_stream=None) -> StepResult:
    """One view-parallel step.

    ``grad_fn(view, grads, accumulate)`` adds (or writes, when accumulate is
    False) the flat gradient of ``view`` into ``grads``.  Returns the reduced
    batch gradient (in place in ``grads``).

    With ``last_grad_fn(view, grads, accumulate, bounds) -> events`` (and
    ``n_triangles``) the rank's last view produces its gradient in
    ``n_buckets`` triangle ranges (``chunk_bounds``), returning one event per
    range (or None); each bucket's all-reduce is launched behind its event, so
    the collective overlaps the rest of that view's chain.
    """
    if world is None:
        world = dist.get_world_size() if dist.is_initialized() else 1
    if rank is None:
        rank = dist.get_rank() if dist.is_initialized() else 0
    views = shard(n_views, world, rank)
    overlap = last_grad_fn is not None and world > 1 and len(views) > 0 and n_triangles is not None
    if len(views) == 0:
        grads.zero_()
    last = len(views) - 1 if overlap else len(views)
    for k, v in enumerate(views):
        if k < last:
            grad_fn(v, grads, k > 0)
    if not overlap:
        allreduce_(grads)
        return StepResult(grads, list(views))
    bounds = chunk_bounds(n_triangles, n_buckets)
    events = last_grad_fn(views[last], grads, last > 0, bounds)
    red = BucketedAllReduce(grads, n_triangles, bounds, comm_stream)
    for k in range(len(bounds) - 1):
        red.launch(k, events[k] if events is not None else None)
    red.wait()
    return StepResult(grads, list(views))


class B200ViewTrainer:
    """Forward + backward of each local view on the B200 rasterizer, then one
    NCCL all-reduce.  ``poses`` / ``d_images`` index the batch.

    ``chain_views`` > 1 defers the chain to the parameter gradients: each
    view's blend backward fills a pending-view slot (ts_backward_screen) and
    every ``chain_views`` views -- and at the rank's last view -- one pass chains
    them all (ts_chain_views: one read of the parameters and one
    read-add-write of the gradient for the group instead of one per view)."""

    def __init__(self, soup, intr, poses, d_images, rasterizer=None, lrs=None, chain_views: int = 8,
                 **render_kw):
        from .rasterizer import DeviceGrads, Rasterizer
        self.rast = rasterizer or Rasterizer()
        self.soup = soup
        self.intr = intr
        self.poses = poses
        self.d_images = d_images
        self.kw = render_kw
        self.grads = DeviceGrads.zeros(len(soup), device=soup.vertices.device)
        self.comm = None          # side stream of the bucketed all-reduce (world > 1)
        self.n_buckets = 8
        self.chain_views = max(1, min(int(chain_views), Rasterizer.MAX_PENDING_VIEWS))
        # deferral needs the fast path with fp32 parameters
        if render_kw.get("precision", "fast") != "fast" or soup.vertices.dtype != torch.float32:
            self.chain_views = 1
        self._acc = False         # the gradient buffer already holds views of this step
        self._last_view = None
        # optional fused Adam after the all-reduce (training.py:165-168): every
        # rank applies the same update to its replica of the parameters
        self.lrs = lrs
        self.adam = None
        if lrs is not None:
            from .optim import DeviceAdamState
            self.adam = DeviceAdamState.zeros(len(soup))

    def _flush(self, chunks=None):
        self.rast.chain_views(self.grads, accumulate=self._acc, chunks=chunks)
        self._acc = True

    def _grad(self, v: int, flat: torch.Tensor, accumulate: bool):
        self.rast.forward(self.soup, self.intr, self.poses[v], keep_backward=True, **self.kw)
        if self.chain_views == 1:
            self.rast.backward(self.d_images[v], self.grads, accumulate=accumulate)
            return
        pending = self.rast.backward_screen(self.d_images[v])
        if pending >= self.chain_views or v == self._last_view:
            self._flush()

    def _grad_chunked(self, v: int, flat: torch.Tensor, accumulate: bool, bounds):
        """The rank's last view: the chain in triangle ranges, one event each."""
        self.rast.forward(self.soup, self.intr, self.poses[v], keep_backward=True, **self.kw)
        events = [torch.cuda.Event() for _ in range(len(bounds) - 1)]
        if self.chain_views == 1:
            self.rast.backward(self.d_images[v], self.grads, accumulate=accumulate, chunks=(bounds, events))
        else:
            self.rast.backward_screen(self.d_images[v])
            self._flush(chunks=(bounds, events))
        return events

    def step(self) -> StepResult:
        world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
        rank = dist.get_rank() if world > 1 else 0
        if self.comm is None and world > 1 and self.grads.flat.is_cuda:
            self.comm = torch.cuda.Stream()
        mine = shard(len(self.poses), world, rank)
        self._last_view = mine[-1] if len(mine) else None
        self._acc = False
        if self.chain_views > 1 and self.rast.pending_views():
            raise RuntimeError("pending views from an interrupted step: call rast.chain_views() first")
        res = train_step(self._grad, len(self.poses), self.grads.flat, world=world, rank=rank,
                         last_grad_fn=self._grad_chunked, n_triangles=len(self.soup), n_buckets=self.n_buckets,
                         comm_stream=self.comm)
        if self.adam is not None:
            from .optim import adam_step
            adam_step(self.soup, self.grads, self.adam, self.lrs, rasterizer=self.rast)
        return res
