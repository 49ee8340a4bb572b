"""Share of stall samples / warp instructions per source region of one file.

    python tools/ncu_regions.py <report> <file.cu> name:lo-hi [name:lo-hi ...]
"""
import csv
import io
import subprocess
import sys


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rep, fname = sys.argv[1], sys.argv[2]
reg = {}
for a in sys.argv[3:]:
    n, r = a.split(":")
    lo, hi = r.split("-")
    reg[n] = (int(lo), int(hi))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(r for r in rows if r and r[0] == "Line No")
cs, ci = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
acc = {k: [0.0, 0.0] for k in reg}
other = {}
f = None
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) < len(h) or not r[0].isdigit():
        continue
    ln, s, i = int(r[0]), num(r[cs]), num(r[ci])
    tgt = None
    if f == fname:
        tgt = next((acc[k] for k, (a, b) in reg.items() if a <= ln <= b), None)
    if tgt is None:
        tgt = other.setdefault(f"{f} (other)", [0.0, 0.0])
    tgt[0] += s
    tgt[1] += i
allv = list(acc.items()) + list(other.items())
ts = sum(v[0] for _, v in allv) or 1
ti = sum(v[1] for _, v in allv) or 1
for k, v in allv:
    print(f"{k:28s} {100*v[0]/ts:5.1f}% samples {100*v[1]/ti:5.1f}% warp-inst")
