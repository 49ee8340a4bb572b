"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family of the path on a ~3k-triangle scene -- render forward
(fp32 + guard band + fix-up), training forward + streaming backward, the tile
backward, exact mode, fragment collection + fragment-gradient backward, the
tile sort's long-tile paths (a dense 5k-triangle view), the losses, Adam,
project_scene / build_tile_lists dumps.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_19175_b200 import _lib, rasterizer as R, scenes  # noqa: E402
from paper_2505_19175_b200.rasterizer import DeviceSoup, Rasterizer  # noqa: E402

rast = Rasterizer(0)
soup = scenes.make_soup(3000, seed=11, size=0.15, sigma=(0.5, 4.0))
intr, pose = scenes.frontal_camera(96, 80, 110.0)
ds = DeviceSoup.from_soup(soup, dtype=torch.float32)
d_image = torch.as_tensor(scenes.make_d_image(11, intr.height, intr.width), dtype=torch.float32, device="cuda")
for mode in (0, 1):
    rast.forward(ds, intr, pose, mode=mode, keep_backward=False, debug=True)       # render path
    rast.forward(ds, intr, pose, mode=mode, debug=True)                            # training forward
    g = rast.backward(d_image)                                                      # streaming backward
    rast.set_option(_lib.TS_OPT_TILE_BACKWARD, 1)
    rast.forward(ds, intr, pose, mode=mode)
    rast.backward(d_image, g, accumulate=True)                                      # tile backward
    rast.set_option(_lib.TS_OPT_TILE_BACKWARD, 0)
    rast.forward(ds, intr, pose, mode=mode, precision="exact", debug=True)         # exact fp64 path
    rast.backward(d_image)
    rast.forward(ds, intr, pose, mode=mode)
    fr = rast.fragments()                                                           # collect_fragments
    rast.backward_fragments(d_image, fr.offsets, torch.ones_like(fr.weight), torch.ones_like(fr.depth))
# a dense view: long tiles (the tile sort's big / fallback paths)
dense = scenes.make_soup(6000, seed=12, size=0.3, sigma=1.0)
intr2, pose2 = scenes.frontal_camera(64, 48, 60.0)
ds2 = DeviceSoup.from_soup(dense, dtype=torch.float32)
rast.forward(ds2, intr2, pose2, keep_backward=False, debug=True)
rast.forward(ds2, intr2, pose2)
rast.backward(torch.ones((48, 64, 3), device="cuda"))
rast.set_option(_lib.TS_OPT_LEGACY_BINNING, 1)
rast.forward(ds2, intr2, pose2, keep_backward=False)
rast.set_option(_lib.TS_OPT_LEGACY_BINNING, 0)
# parity dumps
proj = R.project_scene(soup, intr, pose)
R.build_tile_lists(proj, intr, 7)
# losses + Adam
from paper_2505_19175_b200 import losses, optim  # noqa: E402
f = rast.forward(ds, intr, pose)
target = torch.rand_like(f.image)
losses.photometric_loss(f.image, target, 0.2, rasterizer=rast)
grads = rast.backward(d_image)
st = optim.DeviceAdamState.zeros(len(ds))
optim.adam_step(ds, grads, st, {"vertices": 1e-3, "opacity": 1e-2, "sigma": 1e-3, "sh": 1e-3}, rasterizer=rast)
torch.cuda.synchronize()
print("sanitize workload done, launches:", rast.launch_count())
