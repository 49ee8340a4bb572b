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


def _stats_worker(rank, world, port, out_path):
    # view-parallel density statistics: rank r holds views r, r + world, ...
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import density as OD
    from paper_2505_19175_b200.density import reduce_across_ranks
    mw_all, pix_all, area_all = _views()
    mine = list(range(rank, len(mw_all), world))
    if mine:
        mw, views, mean = OD.aggregate([(mw_all[v], pix_all[v] >= 2, area_all[v]) for v in mine])
        area = mean * len(mine)
    else:
        mw, views, area = np.zeros(50), np.zeros(50, np.int64), np.zeros(50)
    t = [torch.from_numpy(np.ascontiguousarray(a)) for a in (mw, views.astype(np.int32), area)]
    nv = reduce_across_ranks(t[0], t[1], t[2], len(mine))
    if rank == 0:
        np.savez(out_path, mw=t[0].numpy(), views=t[1].numpy(), area=t[2].numpy(), nv=nv)
    dist.barrier()
    dist.destroy_process_group()


def _views():
    rng = np.random.default_rng(8)
    return (np.float32(rng.uniform(0, 0.1, (5, 50))).astype(np.float64), rng.integers(0, 6, (5, 50)),
            np.float32(rng.uniform(0, 60, (5, 50))).astype(np.float64))


@pytest.mark.timeout(300)
def test_gloo_world2_density_stats_match_single_process(tmp_path):
    from oracle import density as OD
    out = str(tmp_path / "s.npz")
    mp.spawn(_stats_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    mw_all, pix_all, area_all = _views()
    mw, views, mean = OD.aggregate([(mw_all[v], pix_all[v] >= 2, area_all[v]) for v in range(5)])
    assert int(got["nv"]) == 5
    assert np.array_equal(got["mw"], mw) and np.array_equal(got["views"], views)
    assert np.allclose(got["area"] / 5, mean, rtol=1e-14)


def _overlap_worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    soup, intr, poses, d_images = _scene()
    n = len(soup.vertices)
    grads = torch.zeros(parallel.flat_grad_size(n), dtype=torch.float64)
    seen = []

    def grad_fn(v, flat, accumulate):
        g = torch.from_numpy(_oracle_flat(soup, intr, poses[v], d_images[v]))
        flat.add_(g) if accumulate else flat.copy_(g)

    def last_fn(v, flat, accumulate, bounds):
        seen.append(list(bounds))
        grad_fn(v, flat, accumulate)
        return None

    res = parallel.train_step(grad_fn, len(poses), grads, last_grad_fn=last_fn, n_triangles=n, n_buckets=3)
    assert len(seen) == 1 and seen[0][0] == 0 and seen[0][-1] == n
    if rank == 0:
        np.save(out_path, res.grads.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_bucketed_overlap_matches_single_process(tmp_path):
    """The overlapped step (last view's gradient in triangle-range buckets, one
    all-reduce per bucket) reduces to the same batch gradient."""
    out = str(tmp_path / "o.npy")
    mp.spawn(_overlap_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    soup, intr, poses, d_images = _scene()
    want = sum(_oracle_flat(soup, intr, poses[v], d_images[v]) for v in range(len(poses)))
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12)


def test_chunk_bounds_and_bucket_slices_cover_the_buffer():
    for n in (0, 1, 63, 64, 300, 1000, 2_000_000):
        for k in (1, 3, 8):
            b = parallel.chunk_bounds(n, k)
            assert b[0] == 0 and b[-1] == n and len(b) == k + 1
            assert all(b[i] <= b[i + 1] for i in range(k))
            assert all(x % 64 == 0 for x in b[:-1])
    n = 300
    flat = torch.arange(59 * n)
    b = parallel.chunk_bounds(n, 3)
    cover = torch.cat([s for i in range(3) for s in parallel.bucket_slices(flat, n, b[i], b[i + 1])])
    assert torch.equal(cover.sort().values, flat)
