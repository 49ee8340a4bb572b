"""C4-style views on 1 or 2 rasterizer contexts (one stream each, views dealt
alternately), deferred chains serialised on the shared gradient: view-iters/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_19175_b200 import DeviceGrads, DeviceSoup, Rasterizer, scenes  # noqa: E402

c3 = scenes.CONFIGS["c3"]
ds = DeviceSoup.from_soup(scenes.make_soup(c3.n, c3.seed, c3.size, c3.sigma), dtype=torch.float32)
intr, _ = scenes.frontal_camera(c3.width, c3.height, c3.f)
poses = scenes.orbit_cameras(32, seed=4)
gen = torch.Generator("cuda").manual_seed(103)
d_imgs = [torch.randn((c3.height, c3.width, 3), device="cuda", generator=gen) for _ in poses]
grads = DeviceGrads.zeros(len(ds))
K = 8


def run(nctx, rs, sts):
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(cur)
    for s in sts:
        s.wait_stream(cur)
    acc = False
    for i, p in enumerate(poses):
        c = i % nctx
        with torch.cuda.stream(sts[c]):
            rs[c].forward(ds, intr, p, keep_backward=True)
            n = rs[c].backward_screen(d_imgs[i])
            last = i >= len(poses) - nctx
            if n >= K // nctx or last:
                sts[c].wait_event(ev)
                rs[c].chain_views(grads, accumulate=acc)
                acc = True
                ev = torch.cuda.Event()
                ev.record(sts[c])
    for s in sts:
        cur.wait_stream(s)


for nctx in (1, 2, 1, 2):
    rs = [Rasterizer() for _ in range(nctx)]
    sts = [torch.cuda.Stream() for _ in range(nctx)]
    for r, s in zip(rs, sts):
        with torch.cuda.stream(s):
            r.forward(ds, intr, poses[0], keep_backward=True)
            r.backward_screen(d_imgs[0])
            r.chain_views(grads)
        r.set_async(True)
    torch.cuda.synchronize()
    run(nctx, rs, sts)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        run(nctx, rs, sts)
    e1.record()
    torch.cuda.synchronize()
    for r, s in zip(rs, sts):
        r.status(stream=s)
    ms = e0.elapsed_time(e1) / 3
    print(f"{nctx} context(s): {len(poses) / ms * 1e3:.1f} view-iters/s ({ms / len(poses):.3f} ms/view)")
    del rs
