"""Debug: screen-space gradients of the streaming backward vs the oracle on a golden scene."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch

from conftest import GoldenScene, golden_paths
from oracle import oracle as O
from paper_2505_19175_b200.rasterizer import DeviceSoup, Rasterizer

g = GoldenScene(golden_paths()[0])
r = Rasterizer()
ds = DeviceSoup.from_soup(g.soup, dtype=torch.float64)
f = r.forward(ds, g.intr, g.pose, mode=g.mode, background=g.background, debug=True)
gr = r.backward(torch.as_tensor(g.d_image, dtype=torch.float32, device="cuda"))
n = len(g.soup.vertices)
sg = r.dump_sgrad(n)
osg = O.render_backward(g.soup, g.intr, g.pose, mode=g.mode, background=g.background, d_image=g.d_image,
                        return_screen=True)
names = ["gq0x", "gq0y", "gq1x", "gq1y", "gq2x", "gq2y", "go", "gsig", "gr", "gg", "gb", "gphis", "gz"]
for j, nm in enumerate(names):
    a, b = sg[:, j], osg[:, j]
    d = np.abs(a - b)
    i = int(np.argmax(d))
    print(f"{nm:6s} maxabs={np.abs(b).max():.3e} maxdiff={d.max():.3e} at {i}: gpu={a[i]:.6e} ora={b[i]:.6e}")
print("n_frag total", int(f.n_frag.sum()), "flagged", f.n_flagged)
# records of triangle 4 vs a replay of the oracle's per-pixel fragment lists
tc, ids = r.dump_fragment_records(200000)
ref = O.render(g.soup, g.intr, g.pose, mode=g.mode, background=g.background, collect_fragments=True)
fo = ref.fragments
W = g.intr.width
print("records", len(ids), "holes", int((ids[:, 0] == 0xffffffff).sum()), "oracle frags", len(fo.triangle))
live = ids[:, 0] != 0xffffffff
cnt = np.bincount(ids[live, 1], minlength=n)
ocnt = np.bincount(fo.triangle, minlength=n)
print("per-triangle record counts", cnt.tolist())
print("per-triangle oracle counts", ocnt.tolist())
pix = ids[live, 0]
dup = len(pix) - len(set(zip(pix.tolist(), ids[live, 1].tolist())))
print("duplicate (pixel, tri) records:", dup)
# T / C of each record against the oracle's fragment list of its pixel
off = fo.offsets
proj_rgb = O.render(g.soup, g.intr, g.pose, mode=g.mode, background=g.background).proj.rgb if hasattr(O.render(g.soup, g.intr, g.pose, mode=g.mode, background=g.background).proj, "rgb") else None
bad = 0
for q in np.nonzero(live)[0]:
    p, src, ordk = int(ids[q, 0]), int(ids[q, 1]), int(ids[q, 2])
    lst = fo.triangle[off[p]:off[p + 1]]
    wl = fo.weight[off[p]:off[p + 1]]
    if ordk >= len(lst) or lst[ordk] != src:
        bad += 1
        if bad < 5: print("order mismatch", p, src, ordk, lst.tolist())
        continue
    T_ref = 1.0 - wl[:ordk].sum()
    if abs(tc[q, 0] - T_ref) > 1e-9:
        bad += 1
        if bad < 5: print("T mismatch", p, src, ordk, tc[q, 0], T_ref)
print("record mismatches:", bad)
# gr of triangle 4 from the records (w from the oracle weights) vs gpu / oracle
d = g.d_image
acc = 0.0
for q in np.nonzero(live)[0]:
    p, src, ordk = int(ids[q, 0]), int(ids[q, 1]), int(ids[q, 2])
    if src != 4: continue
    wk = fo.weight[off[p] + ordk]
    acc += wk * d[p // W, p % W, 0]
print("gr(4) from records:", acc, "gpu", sg[4, 8], "oracle", osg[4, 8])
t4 = [q for q in np.nonzero(live)[0] if ids[q, 1] == 4]
print("record index range of tri 4:", min(t4), max(t4), "count", len(t4))
runs = np.split(np.array(t4), np.nonzero(np.diff(t4) != 1)[0] + 1)
print("runs:", [(int(r[0]), len(r)) for r in runs])
# recompute alpha of triangle 4's records with the oracle's projection
proj = O.render(g.soup, g.intr, g.pose, mode=g.mode, background=g.background).proj
m4 = int(np.nonzero(proj.sorted_idx == 4)[0][0])
print("tri 4: sig", proj.sig[m4], "opa", proj.opa[m4], "phis", proj.phis[m4], "area", proj.area[m4])
errs = []
for q in t4:
    p, ordk = int(ids[q, 0]), int(ids[q, 2])
    px, py = p % W, p // W
    phi = max(proj.nrm[m4, e, 0] * (px + .5) + proj.nrm[m4, e, 1] * (py + .5) + proj.doff[m4, e] for e in range(3))
    r = min(phi / proj.phis[m4], 1.0)
    a = min(proj.opa[m4] * r ** proj.sig[m4], 0.99)
    wk = fo.weight[off[p] + ordk]
    errs.append(abs(tc[q, 0] * a - wk))
print("max |T a - w| over tri-4 records:", max(errs), "r>=1 count", sum(1 for q in t4 if False))
import ctypes
from paper_2505_19175_b200 import _lib
lib = _lib.load()
if os.environ.get("TS_STREAM_DEBUG"):
    buf = np.zeros((len(ids), 4))
    lib.ts_debug_stream_copy(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_longlong(len(ids)))
    bad = 0
    for q in t4:
        p, ordk = int(ids[q, 0]), int(ids[q, 2])
        wk = fo.weight[off[p] + ordk]
        if abs(buf[q, 0] - wk) > 1e-12 or abs(buf[q, 3] - d[p // W, p % W, 0]) > 1e-6:
            bad += 1
            if bad < 6: print("rec", q, "pix", p, "w gpu", buf[q, 0], "w ref", wk, "a", buf[q, 1], "r", buf[q, 2], "d0", buf[q, 3], d[p // W, p % W, 0])
    print("tri-4 records with a wrong w / d:", bad)
if os.environ.get("TS_STREAM_DEBUG"):
    contrib = {}
    for q in t4:
        step = (q // 32) * 32
        contrib[step] = contrib.get(step, 0.0) + buf[q, 0] * buf[q, 3]
    deficit = sum(contrib.values()) - sg[4, 8]
    print("deficit", deficit)
    for st_, v in sorted(contrib.items()):
        lanes = [q - st_ for q in t4 if (q // 32) * 32 == st_]
        print(f"step {st_}: lanes {min(lanes)}..{max(lanes)} n={len(lanes)} contrib={v:.6f}")
