"""At-scale golden digests from the LIVE reference package (run in the build
container, where /root/reference exists; the GPU box only reads the .npz).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_scale.py [c2 ns c3 c5]

The BASELINE configs are too large to commit verbatim (C5 alone is 5M
triangles and 2M pixels), so each ``scale_<cfg>.npz`` keeps:

* an input digest of the scene (regenerated from its seed by
  ``paper_2505_19175_b200.scenes``; both sides see the same fp32-rounded values),
* sha256 digests of every discrete output: ``sorted_idx`` (render.py:275-277),
  ``tile_start`` / ``entry_tri`` (render.py:349-361), per-pixel last contributor
  and fragment count (from ``FragmentData``, render.py:68-81,420-425) and
  ``per_triangle_pixel_count`` (render.py:412-418),
* float outputs as per-channel sums plus a seeded sample of pixels / triangles
  (image, alpha, max weight, area), and for C3 the ``render_backward`` gradients
  (backward.py:93-211) of a seeded, fp32-representable ``d_image`` as
  per-group sums plus the full 59-value rows of a seeded sample of triangles.
"""
from __future__ import annotations

import hashlib
import importlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

R = importlib.import_module("trisplat.render")
B = importlib.import_module("trisplat.backward")
G = importlib.import_module("trisplat.geometry")
S = importlib.import_module("trisplat.soup")

from paper_2505_19175_b200 import scenes  # noqa: E402

N_PIX_SAMPLE = 4096
N_TRI_SAMPLE = 4096
BACKWARD = {"c3"}


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def samples(seed, n_pix, n_tri):
    rng = np.random.default_rng(seed)
    return (np.sort(rng.choice(n_pix, size=min(N_PIX_SAMPLE, n_pix), replace=False)),
            np.sort(rng.choice(n_tri, size=min(N_TRI_SAMPLE, n_tri), replace=False)))


def make(name):
    cfg = scenes.CONFIGS[name]
    t0 = time.time()
    soup, intr, pose = scenes.make_scene(cfg)
    rsoup = S.TriangleSoup(soup.vertices, soup.opacity, soup.sigma, soup.sh)
    rintr = G.CameraIntrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height)
    rpose = G.CameraPose(pose.rotation, pose.translation)
    out = R.render(rsoup, rintr, rpose, collect_fragments=True)
    proj = R.project_scene(rsoup, rintr, rpose, G.WindowMode.NORMALIZED)
    _, _, tile_start, entry_tri = R.build_tile_lists(proj, rintr)
    fr = out.fragments
    hw = intr.height * intr.width
    cnt = np.diff(fr.offsets)
    last = np.full(hw, -1, np.int64)
    nz = cnt > 0
    last[nz] = fr.triangle[fr.offsets[1:][nz] - 1]
    pix_s, tri_s = samples(cfg.seed + 1000, hw, cfg.n)
    img = out.image.rgb.reshape(hw, 3)
    res = dict(
        input_digest=np.array(digest(soup.vertices, soup.opacity, soup.sigma, soup.sh)),
        n_visible=np.array(len(proj.sorted_idx)), n_entries=np.array(len(entry_tri)),
        n_fragments=np.array(int(fr.offsets[-1])),
        sorted_idx_digest=np.array(digest(proj.sorted_idx.astype(np.int64))),
        tile_start_digest=np.array(digest(np.asarray(tile_start, np.int64))),
        entry_tri_digest=np.array(digest(np.asarray(entry_tri, np.int64))),
        last_src_digest=np.array(digest(last.astype(np.int32))),
        nfrag_digest=np.array(digest(cnt.astype(np.int32))),
        pixcount_digest=np.array(digest(out.per_triangle_pixel_count.astype(np.int64))),
        image_sum=img.sum(0), alpha_sum=np.array(out.alpha_map.sum()),
        maxw_sum=np.array(out.per_triangle_max_weight.sum()),
        area_sum=np.array(out.per_triangle_area.sum()),
        pix_sample=pix_s, tri_sample=tri_s,
        image_sample=img[pix_s], alpha_sample=out.alpha_map.reshape(hw)[pix_s],
        last_src_sample=last[pix_s].astype(np.int32), nfrag_sample=cnt[pix_s].astype(np.int32),
        maxw_sample=out.per_triangle_max_weight[tri_s],
        pixcount_sample=out.per_triangle_pixel_count[tri_s].astype(np.int64),
        area_sample=out.per_triangle_area[tri_s])
    t1 = time.time()
    if name in BACKWARD:
        d_image = scenes.make_d_image(cfg.seed, cfg.height, cfg.width, fp32=True)
        g = B.render_backward(rsoup, rintr, rpose, d_image=d_image)
        rows = np.concatenate([g.d_vertices.reshape(cfg.n, 9), g.d_opacity[:, None], g.d_sigma[:, None],
                               g.d_sh.reshape(cfg.n, 48)], axis=1)
        res.update(d_image_digest=np.array(digest(d_image)),
                   grad_sum=np.array([g.d_vertices.sum(), g.d_opacity.sum(), g.d_sigma.sum(), g.d_sh.sum()]),
                   grad_abs_sum=np.array([np.abs(g.d_vertices).sum(), np.abs(g.d_opacity).sum(),
                                          np.abs(g.d_sigma).sum(), np.abs(g.d_sh).sum()]),
                   grad_sample=rows[tri_s])
    np.savez_compressed(os.path.join(HERE, f"scale_{name}.npz"), **res)
    print(f"{name}: M={len(proj.sorted_idx)} E={len(entry_tri)} F={int(fr.offsets[-1])} "
          f"forward {t1 - t0:.1f}s backward {time.time() - t1:.1f}s", flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["c2", "ns", "c3", "c5"]:
        make(nm)
