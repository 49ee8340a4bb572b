"""GPU vs oracle at the BASELINE scales (C3 fwd+bwd, C5 fwd): discrete outputs,
RGB, and the gradient error under several criteria (for choosing precision).

    python tools/scale_probe.py [c3] [c5]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from conftest import rel_err  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2505_19175_b200 import scenes  # noqa: E402
from paper_2505_19175_b200.rasterizer import DeviceSoup, Rasterizer  # noqa: E402


def fwd_check(r, f, ref, intr, label):
    m = f.n_visible
    ok = {}
    ok["sorted"] = np.array_equal(r.dump_sorted_idx(m), ref.proj.sorted_idx)
    ntiles = ((intr.width + 15) // 16) * ((intr.height + 15) // 16)
    ok["tile_start"] = np.array_equal(r.dump_tile_start(ntiles), ref.tile_start)
    ok["entries"] = np.array_equal(r.dump_entry_rank(f.n_entries), ref.entry_tri)
    ok["last"] = int((f.last_src.cpu().numpy() != ref.last_src).sum())
    ok["nfrag"] = int((f.n_frag.cpu().numpy() != ref.nfrag).sum())
    ok["pixcount"] = int((f.pixel_count.cpu().numpy() != ref.per_triangle_pixel_count).sum())
    ok["rgb"] = float(np.abs(f.image.double().cpu().numpy() - ref.image).max())
    ok["maxw"] = float(np.abs(f.max_weight.double().cpu().numpy() - ref.per_triangle_max_weight).max())
    print(label, ok, "M", m, "E", f.n_entries, "flagged", f.n_flagged, flush=True)


def grad_report(g, gr, label):
    for k in ("d_vertices", "d_opacity", "d_sigma", "d_sh"):
        got = getattr(g, k).double().cpu().numpy().reshape(len(gr.d_opacity), -1)
        want = getattr(gr, k).reshape(len(gr.d_opacity), -1)
        d = np.abs(got - want)
        scale = np.abs(want).max()
        # reference test_backward.py:171 style: |d| <= rel*|want| + abs
        need_abs = float(np.max(d - 1e-4 * np.abs(want)))
        viol = int((d > 1e-4 * np.abs(want) + 1e-7).sum())
        i = np.unravel_index(np.argmax(d / (np.abs(want) + 1e-7)), d.shape)
        print(f"{label} {k}: scale {scale:.3e} rel(1e-3 floor) {rel_err(got, want):.2e} "
              f"abs needed at rtol 1e-4: {need_abs:.2e}  #viol(abs=1e-7) {viol} "
              f"worst tri {i[0]} got {got[i]:.6e} want {want[i]:.6e}", flush=True)


def c3():
    soup, intr, pose = scenes.make_scene("c3")
    ds = DeviceSoup.from_soup(soup, dtype=torch.float32)
    r = Rasterizer()
    d_image = scenes.make_d_image(3, intr.height, intr.width)
    if os.environ.get("ROUND_D"):
        d_image = d_image.astype(np.float32).astype(np.float64)
    t0 = time.time()
    ref = O.render(soup, intr, pose)
    gr = O.render_backward(soup, intr, pose, d_image=d_image)
    print("oracle c3 fwd+bwd s", time.time() - t0, flush=True)
    for prec in os.environ.get("PRECS", "fast,exact").split(","):
        f = r.forward(ds, intr, pose, precision=prec, debug=True)
        f = r.forward(ds, intr, pose, precision=prec, debug=True)  # (record buffer sized by the first)
        fwd_check(r, f, ref, intr, f"c3-{prec}")
        g = r.backward(torch.as_tensor(d_image, dtype=torch.float32, device="cuda"))
        grad_report(g, gr, f"c3-{prec}")


def c5():
    soup, intr, pose = scenes.make_scene("c5")
    ds = DeviceSoup.from_soup(soup, dtype=torch.float32)
    r = Rasterizer()
    t0 = time.time()
    ref = O.render(soup, intr, pose)
    print("oracle c5 fwd s", time.time() - t0, flush=True)
    for prec, kb in (("fast", False), ("fast", True), ("exact", True)):
        f = r.forward(ds, intr, pose, precision=prec, debug=True, keep_backward=kb)
        fwd_check(r, f, ref, intr, f"c5-{prec}-kb{int(kb)}")


if __name__ == "__main__":
    which = sys.argv[1:] or ["c3", "c5"]
    for w in which:
        globals()[w]()
