"""Per-CUDA-source-line hot spots of one kernel in an ncu report (needs -lineinfo).

    python tools/ncu_lines.py <report.ncu-rep> [top] [kernel-regex]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 3:
    cmd += ["-k", "regex:" + sys.argv[3]]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
c_s = h.index("Warp Stall Sampling (All Samples)")
c_i = h.index("Instructions Executed")
c_t = h.index("Thread Instructions Executed")
stall_cols = [(i, n) for i, n in enumerate(h) if n.startswith("stall_") or "Stall" in n and "(" not in n]
data = []
for r in rows[hi + 1:]:
    if len(r) < len(h) or not r[0]:
        continue
    try:
        s, ie, te = float(r[c_s] or 0), float(r[c_i] or 0), float(r[c_t] or 0)
    except ValueError:
        continue
    data.append((s, ie, te, r[0], r[1].strip()[:100]))
tot_s = sum(d[0] for d in data) or 1
tot_i = sum(d[1] for d in data) or 1
print(f"total samples {tot_s:.0f}, warp instructions {tot_i:.3e}")
for s, ie, te, ln, src in sorted(data, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% smp {100*ie/tot_i:5.1f}% inst {te/max(ie,1):4.1f} thr  L{ln:>4} {src}")
