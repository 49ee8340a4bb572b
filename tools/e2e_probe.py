"""Where the drop-in render()'s wall clock goes (north-star scene, fp64 soup)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_19175_b200 import rasterizer as R, scenes  # noqa: E402

soup, intr, pose = scenes.make_scene("ns")
rast = R.default_rasterizer()


def t(f, k=10):
    f()
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        r = f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e3, r


ms, ds = t(lambda: R.DeviceSoup.from_soup(soup, dtype=torch.float64))
print(f"upload fp64 soup (staged): {ms:.2f} ms")
ms, f = t(lambda: rast.forward(ds, intr, pose))
print(f"forward on the fp64 soup: {ms:.2f} ms")
ms, ds32 = t(lambda: R.DeviceSoup.from_soup_f32_exact(soup))
print(f"upload fp64 soup as exact fp32 (ts_pack_f32 + staged DMA): {ms:.2f} ms")
ms, _ = t(lambda: rast.forward(ds32, intr, pose))
print(f"forward on the fp32 soup: {ms:.2f} ms")
def outputs():
    packed = torch.cat([f.image.reshape(-1).double(), f.alpha_map.reshape(-1).double(), f.max_weight.double(),
                        f.area.double()])
    h = torch.empty(packed.numel(), dtype=torch.float64, pin_memory=True)
    h.copy_(packed, non_blocking=True)
    hp = torch.empty(f.pixel_count.numel(), dtype=torch.int64, pin_memory=True)
    hp.copy_(f.pixel_count.long(), non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return h.numpy(), hp.numpy()


ms, _ = t(outputs)
print(f"outputs to host (pinned): {ms:.2f} ms")
ms, _ = t(lambda: R.render(soup, intr, pose))
print(f"render() total: {ms:.2f} ms ({1e3 / ms:.1f} FPS)", {k: (round(v, 2) if isinstance(v, float) else v)
                                                           for k, v in R.LAST_RENDER_TIMES.items()})

from paper_2505_19175_b200.types import ImageBuffer  # noqa: E402
img = np.random.default_rng(0).random((720, 1280, 3))
ms, _ = t(lambda: ImageBuffer(img))
print(f"ImageBuffer(image) check: {ms:.2f} ms")
ms, _ = t(lambda: R.as_soup(soup))
print(f"as_soup: {ms:.2f} ms")
