"""Benchmark: forward render FPS of the B200 rasterizer (north-star workload).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one render of one 1280x720 view of the 2M-triangle synthetic scene
(SURVEY.md section 8d "north-star"): projection + depth sort + tile binning +
blend, parameters resident in HBM (472 MB of fp32 parameters, larger than the
126 MB L2, so no explicit L2 flush is needed between steps).  With N GPUs (one
rank per GPU over NCCL) every rank renders its own frames of the same scene --
view-parallel weak scaling with no data-path collective; the whole-job value
is frames/s summed over ranks, timed as the max over ranks.  ``--gpus N``
without a torchrun environment re-launches itself under
``torch.distributed.run`` with N ranks (NCCL_DEBUG=INFO, logged to stderr).

Extra keys:
  ``e2e``            the same metric through the reference-facing drop-in
                     ``paper_2505_19175_b200.render(soup, intr, pose)``: the
                     reference's fp64 numpy soup uploaded and the full
                     RenderOutput (image, alpha, per-triangle max weight /
                     pixel count / area) returned to numpy, every step;
  ``e2e_device_api`` fp32 parameters from pinned host buffers through
                     ``Rasterizer.forward``, image + alpha read back;
  ``roofline``       blend kernel: algorithmic bytes per launch / CUDA-event
                     duration vs the measured HBM peak; ``traffic`` = ncu DRAM
                     bytes of the same kernel on the same workload;
  ``roofline_bwd``   training backward of one C3 view (SURVEY 8d B_bwd);
  ``cpu_baseline``   the CPU oracle port on this host's cores (bounded sample);
  ``stages_ms``      per-stage device ms;
  ``train``          C4: 64 orbit views of the C3 scene sharded over the ranks,
                     forward + backward per view and the NCCL all-reduce of the
                     flat gradient inside the timed step.

``--impl reference`` times the CPU implementation of the same path (the oracle
restatement of the reference, all host threads) on the same workload, rank 0
only.  ``--dry-run`` exercises the launcher and the collective on CPU (gloo,
synthetic gradients; no kernels) for tests.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--train-views", type=int, default=64)
    ap.add_argument("--train-steps", type=int, default=2)
    ap.add_argument("--dry-run", action="store_true", help="CPU/gloo launcher + collective check, no kernels")
    ap.add_argument("--tile-backward", action="store_true", help="training: tile backward instead of the streaming one")
    ap.add_argument("--chain-views", type=int, default=8,
                    help="training: views chained to parameter gradients per pass (1 = per view)")
    return ap.parse_args()


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_if_needed(args):
    """``--gpus N`` outside torchrun: run N ranks under torch.distributed.run.
    Returns the exit code of the launched job, or None to continue in-process."""
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is not None:
        if int(world_env) != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}")
        return None
    if args.gpus <= 1:
        return None
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # keep stdout to the one JSON line
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks():
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_for(workload: str, kernel: str):
    """ncu DRAM bytes (read + write) per launch of ``kernel`` on ``workload``
    (profiles/traffic.json, from the committed ncu captures), or None."""
    p = os.path.join(HERE, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f)[workload].get(kernel)
    except Exception:
        return None


def issue_roofline(workload: str, blend_ms, clk):
    """The blend's binding resource is instruction issue, not HBM: its warp-
    instructions per launch (ncu, profiles/traffic.json) over the event-timed blend
    against 4 issue slots per SM per clock (148 SMs at the sampled SM clock)."""
    inst = traffic_for(workload, "k_blend_dense_warp_instructions")
    if not inst or not blend_ms:
        return None
    mhz = (clk or {}).get("sm_mhz") or 1965
    slots = 148 * 4 * mhz * 1e6 * (blend_ms / 1e3)
    return {"bound": "issue", "warp_instructions": inst, "issue_slots": slots, "frac": inst / slots,
            "source": "smsp__inst_executed.sum of the committed ncu capture; blend stage time of this run"}


def bench_config(cfg, world: int) -> dict:
    """The ``config`` of both arms (identical dicts: same workload, same sharding)."""
    return {"workload": f"{cfg.name}: {cfg.n} triangles, {cfg.width}x{cfg.height}, sigma={cfg.sigma}, "
                        f"SH degree {cfg.sh_degree}, forward render (SURVEY 8d)",
            "parallelism": f"view-parallel x{world} (each rank renders its own frames)",
            "l2": "inputs (472 MB fp32 params at 2M triangles) larger than the 126 MB L2; no flush"}


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


def blend_bytes(e, p, v):
    """Algorithmic bytes of one blend launch: per entry a 64 B
    record + 4 B index, per pixel 24 B of outputs, per visible triangle 8 B of
    statistics."""
    return 68 * e + 24 * p + 8 * v


def backward_bytes(n, e, p, v):
    """Algorithmic bytes of one training backward (SURVEY.md 8d B_bwd): d_image
    + saved per-pixel state, the entries' records, per visible triangle the
    13-float screen-space gradient RMW + chain read, parameters read + 59
    gradients written (fp32)."""
    return 24 * p + 68 * e + 156 * v + 8 * 59 * n


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
    # warm-up frames (bounded: ~30 s), then the timed frames (bounded: ~60 s;
    # a CPU frame of the north-star takes ~1 s on the GPU box's 16 threads)
    tw = time.perf_counter()
    for i in range(args.warmup):
        if i > 0 and time.perf_counter() - tw > 30.0:
            break
        O.render(soup, intr, pose)
    t0 = time.perf_counter()
    frames = 0
    while frames < args.steps and (frames == 0 or time.perf_counter() - t0 < 60.0):
        O.render(soup, intr, pose)
        frames += 1
    dt = time.perf_counter() - t0
    val = frames / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
        "steps": frames, "warmup": args.warmup, "ms_per_step": dt * 1e3 / frames,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": bench_config(cfg, world),
        "implementation": "oracle/trisplat_oracle.c (CPU restatement of the reference, OpenMP over tiles, "
                          "bit-exact with the reference on tests/golden)",
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


def dry_run(args):
    """Launcher / collective check on CPU: gloo, one synthetic gradient per
    view, the same sharding and all-reduce as the training step."""
    import torch
    import torch.distributed as dist

    from paper_2505_19175_b200 import parallel
    world, rank, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    n, views = 1000, args.train_views
    grads = torch.zeros(parallel.flat_grad_size(n), dtype=torch.float64)

    def grad_fn(v, flat, accumulate):
        g = torch.full_like(flat, float(v + 1))
        flat.add_(g) if accumulate else flat.copy_(g)

    t0 = time.perf_counter()
    for _ in range(args.steps):
        res = parallel.train_step(grad_fn, views, grads)
    dt = time.perf_counter() - t0
    ok = bool(torch.all(res.grads == views * (views + 1) / 2))
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "allreduce_ok": ok, "views_per_rank": len(res.local_views),
                          "ms_per_step": dt * 1e3 / args.steps}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    rc = relaunch_if_needed(args)
    if rc is not None:
        sys.exit(rc)
    if args.dry_run:
        return dry_run(args)
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
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def max_over_ranks(x: float) -> float:
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

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
    rast.set_async(True)
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
    elapsed_max = max_over_ranks(ev0.elapsed_time(ev1) / 1e3)
    value = world * args.steps / elapsed_max

    conc = concurrent_frames(args, ds, intr, pose, world, max_over_ranks)
    e2e = e2e_dev = None
    if not args.no_e2e:
        e2e = e2e_render(args, soup, intr, pose, world, max_over_ranks)
        e2e_dev = e2e_device_api(args, rast, soup, intr, pose, cfg, world, stream, max_over_ranks)

    train = roof_bwd = None
    if not args.no_train:
        train, roof_bwd = train_step_bench(args, rast, ds, cfg, world, rank, stream, max_over_ranks)

    if rank != 0:
        dist.destroy_process_group() if world > 1 else None
        return
    peak, peak_src = peaks()
    blend_avg = sum(blend_ms) / len(blend_ms)
    bbytes = blend_bytes(fwd.n_entries, P, fwd.n_visible)
    achieved = bbytes / (blend_avg / 1e3) / 1e9
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(cfg, soup, intr, pose)
        except Exception as ex:  # reported, not fatal
            cpu = {"error": str(ex)}
    stages = {k: v / n_prof for k, v in stage_acc.items() if v > 0}
    if roof_bwd is not None:
        roof_bwd.update(peak=peak, frac=roof_bwd["achieved"] / peak)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_max * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": bench_config(cfg, world),
        "frame": {"precision": args.precision, "visible": fwd.n_visible, "entries": fwd.n_entries,
                  "guard_band_pixels": flagged},
        "e2e": e2e,
        "e2e_device_api": e2e_dev,
        "concurrent_frames": conc,
        "roofline": {"bound": "hbm", "kernel": "k_blend_dense (+ k_fixup_fwd)", "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic_for(cfg.name, "k_blend_dense"),
                     "bytes_per_launch": bbytes, "avg_ms": blend_avg, "peak_source": peak_src,
                     "issue": issue_roofline(cfg.name, stages.get("blend"), clk)},
        "roofline_bwd": roof_bwd,
        "cpu_baseline": cpu,
        "stages_ms": stages,
        "train": train,
        "gpu_launches": launches,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def concurrent_frames(args, ds, intr, pose, world, max_over_ranks, n_ctx=3):
    """Serving throughput with independent frames in flight: n_ctx rasterizer
    contexts (own buffers), each on its own stream, frames dealt round robin --
    one frame's latency-bound phases (preprocess, binning, fix-up tail) overlap
    another's blend.  Reported beside ``value`` (one context, one stream)."""
    import torch
    import torch.distributed as dist

    from paper_2505_19175_b200.rasterizer import Rasterizer
    rs = [Rasterizer(torch.cuda.current_device()) for _ in range(n_ctx)]
    sts = [torch.cuda.Stream() for _ in range(n_ctx)]
    for r, s in zip(rs, sts):
        with torch.cuda.stream(s):
            r.forward(ds, intr, pose, precision=args.precision, keep_backward=False)
            r.set_async(True)
            for _ in range(10):
                r.forward(ds, intr, pose, precision=args.precision, keep_backward=False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    cur = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = max(args.steps, 30)
    e0.record(cur)
    for s in sts:
        s.wait_stream(cur)
    for i in range(k):
        with torch.cuda.stream(sts[i % n_ctx]):
            rs[i % n_ctx].forward(ds, intr, pose, precision=args.precision, keep_backward=False)
    for s in sts:
        cur.wait_stream(s)
    e1.record(cur)
    torch.cuda.synchronize()
    for r, s in zip(rs, sts):
        r.status(stream=s)
    dt = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    return {"value": world * k / dt, "unit": UNIT, "contexts": n_ctx, "frames": k,
            "note": "independent frames of the workload, one context + stream each, round robin"}


def e2e_render(args, soup, intr, pose, world, max_over_ranks):
    """The metric through the drop-in a reference caller uses:
    ``render(soup, intr, pose)`` with the reference's fp64 numpy soup, the
    full RenderOutput back in numpy (render.py:364-432), every step."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2505_19175_b200 import rasterizer as tsb
    n = len(soup.vertices)
    host_bytes = sum(np.asarray(getattr(soup, k)).nbytes for k in ("vertices", "opacity", "sigma", "sh"))
    out = None
    for _ in range(2):
        out = tsb.render(soup, intr, pose)
    d2h = int(tsb.LAST_RENDER_D2H_BYTES)
    # bytes that crossed PCIe: the soup's fp32 values when they all are fp32 values
    # (ts_pack_f32 on the host, inside the timed call), else the fp64 arrays
    h2d = int(tsb.LAST_RENDER_TIMES.get("upload_bytes", host_bytes))
    steps = max(3, min(args.steps, 20))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        out = tsb.render(soup, intr, pose)
    dt = max_over_ranks(time.perf_counter() - t0)
    assert out.per_triangle_area.shape == (n,)
    return {"value": world * steps / dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": d2h, "steps": steps, "host_soup_bytes": int(host_bytes),
            "last_call_ms": {k: round(v, 3) for k, v in tsb.LAST_RENDER_TIMES.items() if k.endswith("_ms")},
            "upload": tsb.LAST_RENDER_TIMES.get("upload"),
            "api": "paper_2505_19175_b200.render(TriangleSoup fp64, intr, pose) -> RenderOutput (numpy), "
                   "wall clock per call"}


def e2e_device_api(args, rast, soup, intr, pose, cfg, world, stream, max_over_ranks):
    """fp32 parameters from pinned host buffers through Rasterizer.forward,
    image + alpha read back, every step."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2505_19175_b200.rasterizer import DeviceSoup
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

    steps = max(3, min(args.steps, 30))
    for _ in range(3):
        e2e_step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    dt = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    return {"value": world * steps / dt, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "steps": steps, "api": "Rasterizer.forward(DeviceSoup from pinned fp32 host tensors)"}


def train_step_bench(args, rast, ds, cfg, world, rank, stream, max_over_ranks):
    """C4 training step: 64 orbit views of the C3 scene, sharded across ranks,
    forward + backward per view, one NCCL all-reduce of the flat gradient."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2505_19175_b200 import density as dens
    from paper_2505_19175_b200 import scenes
    from paper_2505_19175_b200.optim import DeviceAdamState, adam_step
    from paper_2505_19175_b200.parallel import B200ViewTrainer, shard
    from paper_2505_19175_b200.rasterizer import DeviceSoup
    c3 = scenes.CONFIGS["c3"]
    if (c3.n, c3.seed, c3.size, c3.sigma) != (cfg.n, cfg.seed, cfg.size, cfg.sigma):
        ds3 = DeviceSoup.from_soup(scenes.make_soup(c3.n, c3.seed, c3.size, c3.sigma), dtype=torch.float32)
    else:
        ds3 = ds  # same soup (seed 3, size 0.02, sigma 1)
    intr3, _ = scenes.frontal_camera(c3.width, c3.height, c3.f)
    poses = scenes.orbit_cameras(args.train_views, seed=4)
    gen = torch.Generator("cuda").manual_seed(c3.seed + 100)
    mine = shard(len(poses), world, rank)
    d_images = [torch.randn((c3.height, c3.width, 3), device="cuda", generator=gen)
                if v in mine else None for v in range(len(poses))]
    if args.tile_backward:
        from paper_2505_19175_b200 import _lib
        rast.set_option(_lib.TS_OPT_TILE_BACKWARD, 1)
    trainer = B200ViewTrainer(ds3, intr3, poses, d_images, rasterizer=rast, precision=args.precision,
                              chain_views=args.chain_views)
    trainer.step()  # warm-up (synchronous forwards size the buffers)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0e = torch.cuda.Event(enable_timing=True)
    t1e = torch.cuda.Event(enable_timing=True)
    l0 = rast.launch_count()
    rast.set_async(True)
    t0e.record(stream)
    for _ in range(args.train_steps):
        trainer.step()
    t1e.record(stream)
    torch.cuda.synchronize()
    rast.status()
    rast.set_async(False)
    launches = rast.launch_count() - l0
    step_s = max_over_ranks(t0e.elapsed_time(t1e) / 1e3) / args.train_steps
    # one fused Adam step (ts_adam_step, reference default rates config.py:54-58)
    # on a copy of the parameters with the batch gradient
    ds_opt = DeviceSoup(ds3.vertices.clone(), ds3.opacity.clone(), ds3.sigma.clone(), ds3.sh.clone())
    ast = DeviceAdamState.zeros(len(ds_opt))
    lrs = {"vertices": 0.0018, "opacity": 0.014, "sigma": 0.0008, "sh": 0.0025}
    adam_step(ds_opt, trainer.grads, ast, lrs, rasterizer=rast)
    a0e = torch.cuda.Event(enable_timing=True)
    a1e = torch.cuda.Event(enable_timing=True)
    a0e.record(stream)
    for _ in range(5):
        adam_step(ds_opt, trainer.grads, ast, lrs, rasterizer=rast)
    a1e.record(stream)
    torch.cuda.synchronize()
    adam_ms = a0e.elapsed_time(a1e) / 5
    del ds_opt
    # one density-control step (prune + grow, density.py:180-263, default
    # DensifyConfig) from the statistics of 8 orbit views, plus the Adam moment
    # remap; host-side wall clock around the synchronized call (it includes the
    # numpy draws of the caller's Generator)
    dstats = dens.DeviceViewStats.empty(len(ds3))
    for vi, pz in enumerate(poses[:8]):
        fo = rast.forward(ds3, intr3, pz, keep_backward=False, precision=args.precision)
        dstats.update(vi, fo, 2)
    torch.cuda.synchronize()
    dcfg = dens.DensifyConfig()
    dens.densify_step(ds3, dstats, 500, dcfg, np.random.default_rng(0))  # warm-up
    torch.cuda.synchronize()
    tq = time.perf_counter()
    dsoup, drep = dens.densify_step(ds3, dstats, 500, dcfg, np.random.default_rng(1))
    ast2 = ast.remap(drep["origin"])
    torch.cuda.synchronize()
    densify_ms = (time.perf_counter() - tq) * 1e3
    dinfo = {"n_before": drep["n_before"], "n_after": drep["n_after"], "n_removed": drep["prune"]["n_removed"],
             "n_split": drep["n_split"], "n_clone": drep["n_clone"], "views": dstats.n_views}
    del dsoup, ast2, ast, dstats
    # the reference's default training iteration (training.py:121-160: beta_distortion,
    # beta_normal > 0, so fragments every iteration) on one C3 view: training forward,
    # fragments(), photometric + distortion + depth + normal losses, the backward with
    # fragment gradients (streaming, weights from fragments())
    from paper_2505_19175_b200 import losses as L
    tgt = torch.rand((c3.height, c3.width, 3), device="cuda", generator=gen)
    v1 = mine[0] if len(mine) else 0

    def default_iteration(ev=None):
        mark = (lambda k: ev[k].record(stream)) if ev else (lambda k: None)
        mark(0)
        fo = rast.forward(ds3, intr3, poses[v1], keep_backward=True, precision=args.precision)
        mark(1)
        fr = rast.fragments()
        mark(2)
        _, d_img = L.photometric_loss(fo.image, tgt, 0.2, rasterizer=rast)
        _, d_w, d_z = L.distortion_loss(fr, rasterizer=rast)
        dep = L.depth_from_fragments(fr, c3.height, c3.width, rasterizer=rast)
        _, _, d_w2 = L.normal_loss(ds3, fr, dep, intr3, poses[v1], rasterizer=rast)
        mark(3)
        # the caller's loss weights, combined in place on the fresh loss gradients
        rast.backward_fragments(d_img, fr.offsets, d_w.mul_(100.0).add_(d_w2, alpha=1e-4), d_z.mul_(100.0),
                                trainer.grads, accumulate=True, weight=fr.weight)
        mark(4)

    default_iteration()
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    default_iteration(evs)
    torch.cuda.synchronize()
    parts = ["forward", "fragments", "losses", "backward_fragments"]
    default_it = {p: round(evs[i].elapsed_time(evs[i + 1]), 3) for i, p in enumerate(parts)}
    default_it["total_ms"] = round(evs[0].elapsed_time(evs[4]), 3)
    # per-stage times of one view as in the step (synchronous forward: its entry /
    # visible counts; the backward accumulating into the batch gradient)
    v0 = mine[0] if len(mine) else 0
    d_img = d_images[v0] if d_images[v0] is not None else torch.zeros((c3.height, c3.width, 3), device="cuda")
    rast.profile(True)
    bw = []
    for _ in range(3):
        fo = rast.forward(ds3, intr3, poses[v0], keep_backward=True, precision=args.precision)
        rast.backward(d_img, trainer.grads, accumulate=True)
        stt = rast.stage_times()
        bw.append(stt["blend_bwd"] + stt["chain_bwd"])
    # the deferred chain of the step (chain_views views per pass): ms per view
    kdef = trainer.chain_views
    chain_def = None
    if kdef > 1:
        for v in range(kdef):
            rast.forward(ds3, intr3, poses[v0], keep_backward=True, precision=args.precision)
            rast.backward_screen(d_img)
        rast.chain_views(trainer.grads, accumulate=True)
        chain_def = round(rast.stage_times()["chain_bwd"] / kdef, 4)
    rast.profile(False)
    bwd_ms = sorted(bw)[len(bw) // 2]
    bbytes = backward_bytes(c3.n, fo.n_entries, c3.width * c3.height, fo.n_visible)
    roof_bwd = {"bound": "hbm", "kernel": "k_bwd_stream + k_chain_bwd32 (one C3 training view)",
                "achieved": bbytes / (bwd_ms / 1e3) / 1e9, "unit": "GB/s", "bytes_per_launch": bbytes,
                "avg_ms": bwd_ms, "traffic": traffic_for("c3", "backward"),
                "view": {"visible": fo.n_visible, "entries": fo.n_entries}}
    train = {"metric": "train iters/s (C4: 64-view batch, fwd+bwd per view, NCCL all-reduce)",
             "value": 1.0 / step_s, "unit": "steps/s (whole job)", "n_gpus": world,
             "view_iters_per_s": len(poses) / step_s, "ms_per_step": step_s * 1e3,
             "views_per_step": len(poses), "views_per_rank": len(mine),
             "grad_buffer_bytes": 4 * 59 * c3.n,
             "allreduce": "NCCL SUM of the flat fp32 gradient inside the timed step" if world > 1 else "none (N=1)",
             "optimizer": "none in the timed step (the metric is fwd+bwd); fused Adam timed separately as adam_ms",
             "gpu_launches_per_step": launches / args.train_steps,
             "chain_views": kdef,
             "deferred_chain_ms_per_view": chain_def,
             "adam_ms": adam_ms,
             "default_iteration_ms": default_it,
             "densify_ms": densify_ms, "densify": dinfo,
             "workload": f"{c3.n} triangles, {c3.width}x{c3.height}, orbit cameras r=6",
             "last_view_stages_ms": {k: round(v, 4) for k, v in stt.items()}}
    return train, roof_bwd


if __name__ == "__main__":
    main()
