"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py launches <launches.csv>          # per-kernel share of the step
    python tools/ncu_summary.py full <report.ncu-rep> [kernel]   # key counters of one capture
"""
import collections
import csv
import io
import subprocess
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
        "s": 1e6, "second": 1e6}


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("ts::", "")
        v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    out = ["| kernel | launches | total us | avg us | share |", "|---|---:|---:|---:|---:|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {n} | {t:.1f} | {t / n:.2f} | {100 * t / tot:.1f}% |")
    return "\n".join(out)


KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_requests_op_red.sum",
    "lts__t_requests_op_atom.sum",
    "smsp__average_warp_latency_issue_stalled_barrier.ratio",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def full(path, kernel=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        if kernel and kernel not in name:
            continue
        out.append(f"### `{name.split('(')[0]}`\n")
        out.append("| metric | value | unit |\n|---|---:|---|")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                out.append(f"| {k} | {r[i]} | {units[i]} |")
        out.append("")
    return "\n".join(out)


def metrics(path):
    """--metrics --csv capture (one row per launch and metric) -> per-kernel
    medians of every metric."""
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, ui, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    per = collections.OrderedDict()
    units = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("ts::", "")
        per.setdefault(name, collections.defaultdict(list))[r[mi]].append(float(r[vi].replace(",", "")))
        units[r[mi]] = r[ui]
    out = []
    for name, m in per.items():
        n = len(next(iter(m.values())))
        out.append(f"### `{name}` (median of {n} launches)\n")
        out.append("| metric | value | unit |\n|---|---:|---|")
        for k, vals in m.items():
            v = sorted(vals)[len(vals) // 2]
            out.append(f"| {k} | {v:,.6g} | {units[k]} |")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]))
    elif sys.argv[1] == "metrics":
        print(metrics(sys.argv[2]))
    else:
        print(full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None))
