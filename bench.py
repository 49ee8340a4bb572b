"""Benchmark: forward render FPS of the B200 rasterizer (north-star workload).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one render() of one 1280x720 view of the 2M-triangle synthetic
scene (SURVEY.md section 8d "north-star"): projection + depth sort + tile
binning + blend, parameters resident in HBM (472 MB of fp32 parameters, larger
than the 126 MB L2, so no explicit L2 flush is needed between steps).  With
N GPUs (torchrun, one rank per GPU) every rank renders its own frames of the
same scene -- view-parallel weak scaling with no data-path collective; the
whole-job value is frames/s summed over ranks, timed as the max over ranks.

Extra keys: ``e2e`` (same metric through the public API with host-pinned
inputs uploaded and the image read back every step), ``roofline`` (blend
kernel, algorithmic bytes per launch / CUDA-event duration vs the measured
HBM peak), ``cpu_baseline`` (the CPU oracle port on this host's cores,
bounded sample), ``stages`` (per-stage device ms), ``train`` (forward +
backward step of the same view, iters/s).

``--impl reference`` times the CPU implementation of the same path (the oracle
restatement of the reference, all host threads) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "render FPS @1280×720 and train iters/s (fwd+bwd) vs #triangles, 1/2/4/8 B200"
UNIT = "frames/s"
WORKLOAD = "ns"  # 2M triangles, 1280x720, sigma=1, SH degree 3, forward render


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=WORKLOAD)
    ap.add_argument("--precision", default="fast", choices=["fast", "exact"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-train", action="store_true")
    ap.add_argument("--train-views", type=int, default=64)
    ap.add_argument("--train-steps", type=int, default=2)
    return ap.parse_args()


def peaks():
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_for(kernel: str):
    """dram bytes per launch of ``kernel`` from the committed ncu summary."""
    p = os.path.join(HERE, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def rows_so_far(self) -> int:
        try:
            with open(self.path) as f:
                return sum(1 for _ in f)
        except Exception:
            return 0

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) == 6 and parts[0].isdigit():
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = sorted(int(r[0]) for r in rows)
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": int(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def blend_bytes(e, p, v):
    """Algorithmic bytes of one blend launch: per entry a 64 B
    record + 4 B index, per pixel 24 B of outputs, per visible triangle 8 B of
    statistics."""
    return 68 * e + 24 * p + 8 * v


def run_reference(args):
    """CPU implementation of the same path: the oracle restatement of the
    reference, all host threads, same workload; rank 0 only."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2505_19175_b200 import scenes
    cfg = scenes.CONFIGS[args.workload]
    soup, intr, pose = scenes.make_scene(cfg)
    threads = O.get_threads()
    # bounded sample: one warm-up frame, then up to --steps frames within ~60 s
    # (a CPU frame of the north-star takes ~1 s on the GPU box's 16 threads)
    for _ in range(min(args.warmup, 1)):
        O.render(soup, intr, pose)
    t0 = time.perf_counter()
    frames = 0
    while frames < args.steps and (frames == 0 or time.perf_counter() - t0 < 60.0):
        O.render(soup, intr, pose)
        frames += 1
    dt = time.perf_counter() - t0
    val = frames / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
        "steps": frames, "warmup": min(args.warmup, 1), "ms_per_step": dt * 1e3 / frames,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.n} triangles, {cfg.width}x{cfg.height}, "
                   f"sigma={cfg.sigma}, SH deg {cfg.sh_degree}, forward render",
                   "implementation": "oracle/trisplat_oracle.c (CPU restatement of the reference, "
                                     "OpenMP over tiles)"},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{frames} full frames of the workload (<= {args.steps}, ~60 s budget)"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, soup, intr, pose, budget_s=15.0, max_frames=8):
    from oracle import oracle as O
    O.render(soup, intr, pose)  # warm (page-in, thread pool)
    t0 = time.perf_counter()
    frames = 0
    while frames < max_frames and (time.perf_counter() - t0) < budget_s:
        O.render(soup, intr, pose)
        frames += 1
    dt = time.perf_counter() - t0
    return {"value": frames / dt, "unit": UNIT, "cores": O.get_threads(), "kind": "port",
            "sample": f"{frames} full frames of {cfg.name} ({cfg.n} tris, {cfg.width}x{cfg.height}) "
                      f"rendered by oracle/trisplat_oracle.c"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2505_19175_b200 import scenes
    from paper_2505_19175_b200.rasterizer import DeviceSoup, Rasterizer

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = scenes.CONFIGS[args.workload]
    soup, intr, pose = scenes.make_scene(cfg)
    ds = DeviceSoup.from_soup(soup, dtype=torch.float32)
    rast = Rasterizer(local)
    stream = torch.cuda.current_stream()
    P = cfg.width * cfg.height

    def step():
        return rast.forward(ds, intr, pose, precision=args.precision, keep_backward=False)

    for _ in range(max(args.warmup, 3)):
        fwd = step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    # keep the GPU busy while the sampler starts (an idle gap would let the
    # clocks drop before the timed frames): ~0.3 s of untimed frames
    rast.set_async(True)
    t_w = time.perf_counter()
    # (and until nvidia-smi has reported twice, so the timed frames are sampled)
    while time.perf_counter() - t_w < 0.3 or (clocks.proc is not None and clocks.rows_so_far() < 2
                                             and time.perf_counter() - t_w < 3.0):
        for _ in range(20):
            step()
        torch.cuda.synchronize()
    rast.status()
    rast.set_async(False)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = rast.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    # timed frames are enqueued back to back (asynchronous forwards: no host
    # round trip per frame); the last frame's status is checked afterwards
    rast.set_async(os.environ.get("TS_BENCH_SYNC") is None)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    status = rast.status()
    rast.set_async(False)
    launches = rast.launch_count() - l0
    flagged = status["n_flagged"] if args.precision == "fast" else 0
    # per-stage device times (CUDA events around each stage) from separate frames
    rast.profile(True)
    blend_ms = []
    stage_acc = {}
    n_prof = max(3, min(args.steps, 10))
    for _ in range(n_prof):
        fwd = step()
        st = rast.stage_times()
        blend_ms.append(st["blend"] + st["fixup"])
        for k, v in st.items():
            stage_acc[k] = stage_acc.get(k, 0.0) + v
    rast.profile(False)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed = ev0.elapsed_time(ev1) / 1e3
    t = torch.tensor([elapsed], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_max = float(t.item())
    value = world * args.steps / elapsed_max

    # ---- end to end through the public API: pinned host params -> device -> image back ----
    host = {k: torch.from_numpy(np.ascontiguousarray(getattr(soup, k), dtype=np.float32)).pin_memory()
            for k in ("vertices", "opacity", "sigma", "sh")}
    img_host = torch.empty((cfg.height, cfg.width, 3), dtype=torch.float32).pin_memory()
    alpha_host = torch.empty((cfg.height, cfg.width), dtype=torch.float32).pin_memory()
    h2d = sum(v.numel() * v.element_size() for v in host.values())
    d2h = img_host.numel() * 4 + alpha_host.numel() * 4

    def e2e_step():
        dsh = DeviceSoup(*(host[k].to("cuda", non_blocking=True) for k in
                           ("vertices", "opacity", "sigma", "sh")))
        f = rast.forward(dsh, intr, pose, precision=args.precision, keep_backward=False)
        img_host.copy_(f.image, non_blocking=True)
        alpha_host.copy_(f.alpha_map, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    e2e_steps = max(3, min(args.steps, 30))
    for _ in range(3):
        e2e_step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([e0.elapsed_time(e1) / 1e3], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_val = world * e2e_steps / float(te.item())

    # ---- C4 training step: 64 orbit views of the C3 scene, sharded across ranks,
    #      forward + backward per view, one NCCL all-reduce of the flat gradient ----
    train = None
    if not args.no_train:
        from paper_2505_19175_b200.parallel import B200ViewTrainer, shard
        c3 = scenes.CONFIGS["c3"]
        if (c3.n, c3.seed, c3.size, c3.sigma) != (cfg.n, cfg.seed, cfg.size, cfg.sigma):
            soup3 = scenes.make_soup(c3.n, c3.seed, c3.size, c3.sigma)
            ds3 = DeviceSoup.from_soup(soup3, dtype=torch.float32)
        else:
            ds3 = ds  # same soup (seed 3, size 0.02, sigma 1)
        intr3, _ = scenes.frontal_camera(c3.width, c3.height, c3.f)
        poses = scenes.orbit_cameras(args.train_views, seed=4)
        gen = torch.Generator("cuda").manual_seed(c3.seed + 100)
        mine = shard(len(poses), world, rank)
        d_images = [torch.randn((c3.height, c3.width, 3), device="cuda", generator=gen)
                    if v in mine else None for v in range(len(poses))]
        trainer = B200ViewTrainer(ds3, intr3, poses, d_images, rasterizer=rast,
                                  precision=args.precision)
        trainer.step()  # warm-up (synchronous forwards size the buffers)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0e = torch.cuda.Event(enable_timing=True)
        t1e = torch.cuda.Event(enable_timing=True)
        rast.set_async(os.environ.get("TS_BENCH_SYNC") is None)
        t0e.record(stream)
        for _ in range(args.train_steps):
            trainer.step()
        t1e.record(stream)
        torch.cuda.synchronize()
        rast.status()
        rast.set_async(False)
        tt = torch.tensor([t0e.elapsed_time(t1e) / 1e3], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        step_s = float(tt.item()) / args.train_steps
        # one fused Adam step (ts_adam_step, reference default rates config.py:54-58)
        # on a copy of the parameters with the batch gradient
        from paper_2505_19175_b200.optim import DeviceAdamState, adam_step
        from paper_2505_19175_b200.rasterizer import DeviceSoup as _DS
        ds_opt = _DS(ds3.vertices.clone(), ds3.opacity.clone(), ds3.sigma.clone(), ds3.sh.clone())
        ast = DeviceAdamState.zeros(len(ds_opt))
        lrs = {"vertices": 0.0018, "opacity": 0.014, "sigma": 0.0008, "sh": 0.0025}
        adam_step(ds_opt, trainer.grads, ast, lrs, rasterizer=rast)
        a0e = torch.cuda.Event(enable_timing=True)
        a1e = torch.cuda.Event(enable_timing=True)
        a0e.record(stream)
        for _ in range(5):
            adam_step(ds_opt, trainer.grads, ast, lrs, rasterizer=rast, check=False)
        a1e.record(stream)
        torch.cuda.synchronize()
        adam_ms = a0e.elapsed_time(a1e) / 5
        del ds_opt
        # one density-control step (prune + grow, density.py:180-263, default
        # DensifyConfig) from the statistics of 8 orbit views, plus the Adam
        # moment remap; host-side wall clock around the synchronized call
        # (it includes the numpy draws of the caller's Generator)
        import numpy as _np
        from paper_2505_19175_b200 import density as _dens
        dstats = _dens.DeviceViewStats.empty(len(ds3))
        for vi, pz in enumerate(poses[:8]):
            fo = rast.forward(ds3, intr3, pz, keep_backward=False, precision=args.precision)
            dstats.update(vi, fo, 2)
        torch.cuda.synchronize()
        dcfg = _dens.DensifyConfig()
        _dens.densify_step(ds3, dstats, 500, dcfg, _np.random.default_rng(0))  # warm-up
        torch.cuda.synchronize()
        tq = time.perf_counter()
        dsoup, drep = _dens.densify_step(ds3, dstats, 500, dcfg, _np.random.default_rng(1))
        ast2 = ast.remap(drep["origin"])
        torch.cuda.synchronize()
        densify_ms = (time.perf_counter() - tq) * 1e3
        dinfo = {"n_before": drep["n_before"], "n_after": drep["n_after"], "n_removed": drep["prune"]["n_removed"],
                 "n_split": drep["n_split"], "n_clone": drep["n_clone"], "views": dstats.n_views}
        del dsoup, ast2, ast, dstats
        rast.profile(True)
        trainer._grad(0 if len(mine) == 0 else mine[0], trainer.grads.flat, True)
        stt = rast.stage_times()
        rast.profile(False)
        train = {"metric": "train iters/s (C4: 64-view batch, fwd+bwd per view, NCCL all-reduce)",
                 "value": 1.0 / step_s, "unit": "steps/s (whole job)",
                 "view_iters_per_s": len(poses) / step_s, "ms_per_step": step_s * 1e3,
                 "views_per_step": len(poses), "views_per_rank": len(mine),
                 "grad_buffer_bytes": 4 * 59 * c3.n,
                 "optimizer": "none in the timed step (the metric is fwd+bwd); fused Adam timed "
                              "separately as adam_ms",
                 "adam_ms": adam_ms,
                 "densify_ms": densify_ms, "densify": dinfo,
                 "workload": f"{c3.n} triangles, {c3.width}x{c3.height}, orbit cameras r=6",
                 "last_view_backward_ms": stt["blend_bwd"] + stt["chain_bwd"],
                 "last_view_stages_ms": {k: round(v, 4) for k, v in stt.items()}}

    if rank != 0:
        dist.destroy_process_group() if world > 1 else None
        return
    peak, peak_src = peaks()
    bms = sorted(blend_ms)
    blend_avg = sum(bms) / len(bms)
    bbytes = blend_bytes(fwd.n_entries, P, fwd.n_visible)
    achieved = bbytes / (blend_avg / 1e3) / 1e9
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(cfg, soup, intr, pose)
        except Exception as ex:  # reported, not fatal
            cpu = {"error": str(ex)}
    stages = {k: v / n_prof for k, v in stage_acc.items() if v > 0}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_max * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.n} triangles, {cfg.width}x{cfg.height}, "
                               f"sigma={cfg.sigma}, SH degree {cfg.sh_degree}, forward render "
                               f"(SURVEY 8d north-star)",
                   "precision": args.precision,
                   "parallelism": f"view-parallel x{world} (each rank renders its own frames)",
                   "l2": "inputs (472 MB fp32 params) larger than the 126 MB L2; no flush",
                   "visible": fwd.n_visible, "entries": fwd.n_entries,
                   "guard_band_pixels": flagged},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "roofline": {"bound": "hbm", "kernel": "k_blend_dense (+ k_fixup_fwd)", "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic_for("k_blend_dense"),
                     "bytes_per_launch": bbytes, "avg_ms": blend_avg, "peak_source": peak_src},
        "cpu_baseline": cpu,
        "stages_ms": stages,
        "train": train,
        "gpu_launches": launches,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
