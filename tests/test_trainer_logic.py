"""The view-parallel trainer's control flow on CPU (gloo, world_size 2), with a
stand-in rasterizer that records the calls: deferred chains in groups of
``chain_views``, the first chain of a step overwriting and later ones
accumulating, the rank's last view chained in bucket ranges (its events feed
the bucketed all-reduce), and the reduced gradient the sum over every view of
the batch."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_19175_b200 import parallel
from paper_2505_19175_b200.rasterizer import DeviceSoup

N_VIEWS, N_TRI, K = 7, 64, 3


class FakeRasterizer:
    """forward(pose = view id); backward_screen queues the view; chain_views adds
    (view + 1) per pending view to every gradient entry."""
    MAX_PENDING_VIEWS = 8

    def __init__(self):
        self.cur, self.pending, self.log = None, [], []

    def forward(self, soup, intr, pose, keep_backward=True, **kw):
        self.cur = pose

    def backward_screen(self, d_image):
        self.pending.append(self.cur)
        return len(self.pending)

    def pending_views(self):
        return len(self.pending)

    def chain_views(self, grads, accumulate=False, chunks=None):
        val = float(sum(v + 1 for v in self.pending))
        if accumulate:
            grads.flat += val
        else:
            grads.flat.fill_(val)
        self.log.append((tuple(self.pending), accumulate, chunks is not None))
        self.pending = []
        return grads

    def backward(self, d_image, grads, accumulate=False, chunks=None):
        self.pending = [self.cur]
        return self.chain_views(grads, accumulate, chunks)


def _worker(rank, world, port, chain_views, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    soup = DeviceSoup(torch.zeros((N_TRI, 3, 3)), torch.zeros(N_TRI), torch.ones(N_TRI), torch.zeros((N_TRI, 16, 3)))
    fake = FakeRasterizer()
    tr = parallel.B200ViewTrainer(soup, None, list(range(N_VIEWS)), [None] * N_VIEWS, rasterizer=fake,
                                  chain_views=chain_views)
    for _ in range(2):  # (the second step starts from a fresh buffer)
        res = tr.step()
        g = res.grads.clone()
    q.put((rank, g.tolist()[:3] + g.tolist()[-3:], fake.log[-4:], list(res.local_views)))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("chain_views", [1, K])
def test_trainer_world2(chain_views):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, chain_views, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((r, (g, log, views)) for r, g, log, views in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = float(sum(v + 1 for v in range(N_VIEWS)))
    for r in (0, 1):
        g, log, views = out[r]
        assert all(x == want for x in g), (r, g)
    assert out[0][2] == [0, 1, 2, 3] and out[1][2] == [4, 5, 6]
    if chain_views == K:
        # rank 0: views 0-2 chained together (overwrite), view 3 last, in ranges (accumulate)
        assert out[0][1][-2:] == [((0, 1, 2), False, False), ((3,), True, True)]
        # rank 1: views 4, 5 pending, chained with the last view 6 in ranges (overwrite)
        assert out[1][1][-1:] == [((4, 5, 6), False, True)]
