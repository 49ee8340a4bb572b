"""Multi-process (gloo, world_size 2, CPU) test of the view-parallel step: the
all-reduced gradient of a sharded view batch equals the single-process sum
of per-view oracle gradients."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_19175_b200 import parallel, scenes


def test_shard_covers_batch():
    for n in (0, 1, 7, 64):
        for world in (1, 2, 3, 8):
            got = [i for r in range(world) for i in parallel.shard(n, world, r)]
            assert got == list(range(n))
            sizes = [len(parallel.shard(n, world, r)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def _scene():
    soup = scenes.make_soup(300, seed=21, size=0.25, sigma=(0.5, 3.0))
    intr, _ = scenes.frontal_camera(48, 40, 52.0)
    poses = scenes.orbit_cameras(5, seed=4)
    d_images = [np.random.default_rng(100 + v).normal(size=(40, 48, 3)) for v in range(5)]
    return soup, intr, poses, d_images


def _oracle_flat(soup, intr, pose, d_image):
    from oracle import oracle as O
    g = O.render_backward(soup, intr, pose, d_image=d_image)
    return np.concatenate([g.d_vertices.reshape(-1), g.d_opacity, g.d_sigma, g.d_sh.reshape(-1)])


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    soup, intr, poses, d_images = _scene()
    grads = torch.zeros(parallel.flat_grad_size(len(soup.vertices)), dtype=torch.float64)

    def grad_fn(v, flat, accumulate):
        g = torch.from_numpy(_oracle_flat(soup, intr, poses[v], d_images[v]))
        if accumulate:
            flat += g
        else:
            flat.copy_(g)

    res = parallel.train_step(grad_fn, len(poses), grads)
    if rank == 0:
        np.save(out_path, res.grads.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(300)
def test_gloo_world2_allreduce_matches_single_process(tmp_path):
    out = str(tmp_path / "g.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    soup, intr, poses, d_images = _scene()
    want = sum(_oracle_flat(soup, intr, poses[v], d_images[v]) for v in range(len(poses)))
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12)
    assert np.abs(want).max() > 0
