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
               grads: torch.Tensor, world: int | None = None, rank: int | None = None) -> StepResult:
    """One view-parallel step.

    ``grad_fn(view, grads, accumulate)`` adds (or writes, when accumulate is
    False) the flat gradient of ``view`` into ``grads``.  Returns the reduced
    batch gradient (in place in ``grads``).
    """
    if world is None:
        world = dist.get_world_size() if dist.is_initialized() else 1
    if rank is None:
        rank = dist.get_rank() if dist.is_initialized() else 0
    views = shard(n_views, world, rank)
    if len(views) == 0:
        grads.zero_()
    for k, v in enumerate(views):
        grad_fn(v, grads, k > 0)
    allreduce_(grads)
    return StepResult(grads, list(views))


class B200ViewTrainer:
    """Forward + backward of each local view on the B200 rasterizer, then one
    NCCL all-reduce.  ``poses`` / ``d_images`` index the batch."""

    def __init__(self, soup, intr, poses, d_images, rasterizer=None, lrs=None, **render_kw):
        from .rasterizer import DeviceGrads, Rasterizer
        self.rast = rasterizer or Rasterizer()
        self.soup = soup
        self.intr = intr
        self.poses = poses
        self.d_images = d_images
        self.kw = render_kw
        self.grads = DeviceGrads.zeros(len(soup))
        # optional fused Adam after the all-reduce (training.py:165-168): every
        # rank applies the same update to its replica of the parameters
        self.lrs = lrs
        self.adam = None
        if lrs is not None:
            from .optim import DeviceAdamState
            self.adam = DeviceAdamState.zeros(len(soup))

    def _grad(self, v: int, flat: torch.Tensor, accumulate: bool):
        self.rast.forward(self.soup, self.intr, self.poses[v], keep_backward=True, **self.kw)
        self.rast.backward(self.d_images[v], self.grads, accumulate=accumulate)

    def step(self) -> StepResult:
        res = train_step(self._grad, len(self.poses), self.grads.flat)
        if self.adam is not None:
            from .optim import adam_step
            adam_step(self.soup, self.grads, self.adam, self.lrs, rasterizer=self.rast)
        return res
