"""Generate golden fixtures from the LIVE reference package (run in the build
container, where /root/reference exists; the GPU box only reads the .npz).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Scenes:
  rs_*.npz   small random scenes from the reference's own conftest.random_scene
             (fp64 inputs stored), normalized + sigmoid, with background and
             collect_fragments, plus render_backward gradients for a seeded d_image
  c1.npz     configs[0] (10k triangles, 128x128) regenerated from its seed by
             paper_2505_19175_b200.scenes; inputs are checked by a digest
  kat.npz    the reference's closed-form/known-answer cases (test_render.py:83-118,
             212-222; test_backward.py:32-42)
"""
from __future__ import annotations

import hashlib
import importlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, REPO)

R = importlib.import_module("trisplat.render")
B = importlib.import_module("trisplat.backward")
G = importlib.import_module("trisplat.geometry")
S = importlib.import_module("trisplat.soup")
from conftest import random_scene  # noqa: E402  (reference test helper)

from paper_2505_19175_b200 import scenes  # noqa: E402


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def run_reference(soup, intr, pose, mode, bg, seed_d):
    out = R.render(soup, intr, pose, mode=mode, background=bg, collect_fragments=True)
    proj = R.project_scene(soup, intr, pose, mode)
    _, _, tile_start, entry_tri = R.build_tile_lists(proj, intr)
    fr = out.fragments
    hw = intr.height * intr.width
    cnt = np.diff(fr.offsets)
    last = np.full(hw, -1, np.int64)
    nz = cnt > 0
    last[nz] = fr.triangle[fr.offsets[1:][nz] - 1]
    d_image = np.random.default_rng(seed_d).normal(size=(intr.height, intr.width, 3))
    g = B.render_backward(soup, intr, pose, mode=mode, background=bg, d_image=d_image)
    return dict(
        image=out.image.rgb, alpha_map=out.alpha_map,
        maxw=out.per_triangle_max_weight, pixcount=out.per_triangle_pixel_count,
        area=out.per_triangle_area, frag_offsets=fr.offsets, frag_triangle=fr.triangle,
        frag_weight=fr.weight, frag_depth=fr.depth, last_src=last.reshape(intr.height, intr.width),
        nfrag=cnt.reshape(intr.height, intr.width), sorted_idx=proj.sorted_idx, z=proj.z,
        bbox=proj.bbox, tile_start=tile_start, entry_tri=entry_tri, d_image_seed=seed_d,
        d_vertices=g.d_vertices, d_opacity=g.d_opacity, d_sigma=g.d_sigma, d_sh=g.d_sh)


def cam_arrays(intr, pose):
    return dict(cam=np.array([intr.fx, intr.fy, intr.cx, intr.cy, intr.z_near]),
                size=np.array([intr.width, intr.height]), rotation=pose.rotation,
                translation=pose.translation)


def small_scenes():
    rng = np.random.default_rng(20261018)
    k = 0
    for i in range(10):
        mode = G.WindowMode.SIGMOID if i % 4 == 3 else G.WindowMode.NORMALIZED
        n_tri = int(rng.integers(1, 30))
        soup, intr, pose = random_scene(rng, n_tri=n_tri, width=int(rng.choice([32, 48, 64])),
                                        height=int(rng.choice([24, 40, 64])))
        bg = tuple(float(x) for x in rng.uniform(0, 1, 3)) if i % 2 else (0.0, 0.0, 0.0)
        res = run_reference(soup, intr, pose, mode, bg, 1000 + i)
        np.savez_compressed(os.path.join(HERE, f"rs_{k:02d}.npz"), vertices=soup.vertices,
                            opacity=soup.opacity, sigma=soup.sigma, sh=soup.sh,
                            mode=np.array(0 if mode is G.WindowMode.NORMALIZED else 1),
                            background=np.array(bg), **cam_arrays(intr, pose), **res)
        k += 1
    print("small scenes:", k)


def c1():
    cfg = scenes.CONFIGS["c1"]
    soup, intr, pose = scenes.make_scene(cfg)
    rsoup = S.TriangleSoup(soup.vertices, soup.opacity, soup.sigma, soup.sh)
    rintr = G.CameraIntrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height)
    rpose = G.CameraPose(pose.rotation, pose.translation)
    res = run_reference(rsoup, rintr, rpose, G.WindowMode.NORMALIZED, (0.0, 0.0, 0.0),
                        cfg.seed + 100)
    keep = 500  # gradients of the first triangles verbatim, checksums for all
    out = dict(input_digest=np.array(digest(soup.vertices, soup.opacity, soup.sigma, soup.sh)),
               image=res["image"], alpha_map=res["alpha_map"], maxw=res["maxw"],
               pixcount=res["pixcount"].astype(np.int32), area=res["area"],
               last_src=res["last_src"].astype(np.int32), nfrag=res["nfrag"].astype(np.int32),
               sorted_idx=res["sorted_idx"].astype(np.int32),
               tile_start=res["tile_start"].astype(np.int32),
               entry_tri=res["entry_tri"].astype(np.int32),
               frag_digest=np.array(digest(res["frag_offsets"], res["frag_triangle"])),
               d_vertices=res["d_vertices"][:keep], d_opacity=res["d_opacity"][:keep],
               d_sigma=res["d_sigma"][:keep], d_sh=res["d_sh"][:keep],
               grad_abs_sum=np.array([np.abs(res[k]).sum() for k in
                                      ("d_vertices", "d_opacity", "d_sigma", "d_sh")]),
               grad_sum=np.array([res[k].sum() for k in
                                  ("d_vertices", "d_opacity", "d_sigma", "d_sh")]))
    np.savez_compressed(os.path.join(HERE, "c1.npz"), **out)
    print("c1: M=%d E=%d" % (len(res["sorted_idx"]), len(res["entry_tri"])))


def kat():
    """Known answers from the reference tests, evaluated by the reference."""
    ident = G.CameraPose(rotation=np.eye(3), translation=np.zeros(3))
    out = {}
    # single opaque triangle (test_render.py:235-245)
    intr = G.CameraIntrinsics(fx=20, fy=20, cx=8, cy=8, width=16, height=16)
    sh = np.zeros((16, 3)); sh[0, 0] = 1.0
    tri = G.Triangle3D(vertices=np.array([[-0.4, -0.4, 1], [0.4, -0.4, 1], [0, 0.4, 1]], float),
                       opacity=0.99, sigma=1e-3, sh=sh)
    r = R.render([tri], intr, ident)
    out["opaque_image"] = r.image.rgb
    # two-layer compositing (test_render.py:247-262)
    intr2 = G.CameraIntrinsics(fx=4, fy=4, cx=8, cy=8, width=16, height=16)
    sh1 = np.zeros((16, 3)); sh2 = np.zeros((16, 3))
    sh1[0] = (np.array([0.9, 0.1, 0.1]) - 0.5) / 0.28209479177387814
    sh2[0] = (np.array([0.1, 0.9, 0.1]) - 0.5) / 0.28209479177387814
    big = np.array([[-8, -8, 0], [8, -8, 0], [0, 12, 0]], float)
    front = G.Triangle3D(vertices=big + [0, 0, 1], opacity=0.5, sigma=1e-5, sh=sh1)
    back = G.Triangle3D(vertices=big * 2 + [0, 0, 2], opacity=0.5, sigma=1e-5, sh=sh2)
    r2 = R.render([front, back], intr2, ident, background=(0.0, 0.0, 1.0))
    out["two_layer_image"] = r2.image.rgb
    np.savez_compressed(os.path.join(HERE, "kat.npz"), **out)
    print("kat done")


if __name__ == "__main__":
    small_scenes()
    c1()
    kat()
