import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_19175_b200 import scenes
from paper_2505_19175_b200.rasterizer import DeviceSoup, Rasterizer
soup, intr, pose = scenes.make_scene("ns")
ds = DeviceSoup.from_soup(soup, dtype=torch.float32)
r = Rasterizer()
for _ in range(5): r.forward(ds, intr, pose, keep_backward=False)
torch.cuda.synchronize()
r.set_async(True)
for steps in (50, 200):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps): r.forward(ds, intr, pose, keep_backward=False)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(steps, "host enqueue ms/frame %.3f" % ((t1 - t0) * 1e3 / steps), "gpu ms/frame %.4f" % (e0.elapsed_time(e1) / steps), "wall %.4f" % ((t2 - t0) * 1e3 / steps))
r.status()
