"""Model I/O for device-resident soups: drop-ins for the
reference's ``export_mesh`` / ``import_ply`` / ``save_model`` / ``load_model``
(trisplat/scene_io.py:365-527).

* PLY (binary little endian): the body is packed / unpacked on the device
  (ts_io.cu, ``ts_ply_pack`` / ``ts_ply_unpack``) and crosses PCIe as two
  contiguous byte buffers; the ASCII header is written / parsed here with the
  reference's checks and messages.  Output files are byte-identical to the
  reference's for the same parameters.
* OBJ (text, ``%.17g`` per coordinate plus a per-face material sidecar) is
  formatted on the host from one download of the vertices / colours.
* ``.npz`` models keep the reference's keys and fp64 arrays, so models move
  between the two implementations and the reference CLI unchanged; cameras
  (``scene``) are passed through as in the reference.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

SH_C0 = 0.28209479177387814
_VDT = np.dtype([("x", "<f4"), ("y", "<f4"), ("z", "<f4"), ("red", "u1"), ("green", "u1"), ("blue", "u1")])
_FDT = np.dtype([("count", "<i4"), ("i0", "<i4"), ("i1", "<i4"), ("i2", "<i4")])


def _device_soup(triangles):
    import torch
    from .rasterizer import DeviceSoup
    if isinstance(getattr(triangles, "vertices", None), torch.Tensor):
        return triangles
    from .types import as_soup
    return DeviceSoup.from_soup(as_soup(triangles), dtype=torch.float64)


def _ctx(rasterizer):
    from .rasterizer import default_rasterizer
    r = rasterizer or default_rasterizer()
    return r.lib, r._ctx


def _ply_header(n: int) -> bytes:
    return ("ply\n"
            "format binary_little_endian 1.0\n"
            f"element vertex {3 * n}\n"
            "property float x\n"
            "property float y\n"
            "property float z\n"
            "property uchar red\n"
            "property uchar green\n"
            "property uchar blue\n"
            f"element face {n}\n"
            "property list int int vertex_indices\n"
            "end_header\n").encode("ascii")


def ply_body(triangles, rasterizer=None, stream=None):
    """(vertex bytes, face bytes) CUDA uint8 tensors of the PLY body."""
    import torch
    from . import _lib
    soup = _device_soup(triangles)
    lib, ctx = _ctx(rasterizer)
    n = len(soup)
    vb = torch.empty(45 * n + 16, dtype=torch.uint8, device="cuda")
    fb = torch.empty(16 * n + 16, dtype=torch.uint8, device="cuda")
    dt = 1 if soup.vertices.dtype == torch.float64 else 0
    st = ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)
    _lib.check(lib.ts_ply_pack(ctx, ctypes.c_void_p(soup.vertices.data_ptr()), ctypes.c_void_p(soup.sh.data_ptr()),
                               dt, n, ctypes.c_void_p(vb.data_ptr()), ctypes.c_void_p(fb.data_ptr()), st),
               "ply_pack")
    return vb[:45 * n], fb[:16 * n]


def _export_ply(soup, path: Path, rasterizer=None) -> Path:
    import torch
    n = len(soup)
    head = _ply_header(n)
    vb, fb = ply_body(soup, rasterizer)
    host = torch.empty(len(head) + 61 * n, dtype=torch.uint8, pin_memory=True)
    host[len(head):len(head) + 45 * n].copy_(vb, non_blocking=True)
    host[len(head) + 45 * n:].copy_(fb, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    buf = host.numpy()
    buf[:len(head)] = np.frombuffer(head, dtype=np.uint8)
    with open(path, "wb") as f:
        f.write(memoryview(buf))
    return path


def soup_colors(triangles) -> np.ndarray:
    """Degree-0 RGB per triangle (scene_io.py:360-363), host fp64."""
    soup = _device_soup(triangles)
    sh0 = soup.sh[:, 0, :].double().cpu().numpy()
    return np.clip(SH_C0 * sh0 + 0.5, 0.0, 1.0)


def _fmt(x) -> str:
    return f"{float(x):.17g}"


def _export_obj(soup, path: Path) -> Path:
    n = len(soup)
    mtl_path = path.with_suffix(".mtl")
    colors = soup_colors(soup)
    with open(mtl_path, "w", encoding="utf-8") as f:
        f.write("".join(f"newmtl tri{i}\nKd {c[0]:.6f} {c[1]:.6f} {c[2]:.6f}\n" for i, c in enumerate(colors)))
    v = soup.vertices.double().cpu().numpy().reshape(3 * n, 3)
    with open(path, "w", encoding="utf-8") as f:
        f.write(f"mtllib {mtl_path.name}\n")
        f.write("".join(f"v {_fmt(a)} {_fmt(b)} {_fmt(c)}\n" for a, b, c in v))
        f.write("".join(f"usemtl tri{i}\nf {3 * i + 1} {3 * i + 2} {3 * i + 3}\n" for i in range(n)))
    return path


def export_mesh(triangles, path, format: str = "ply", rasterizer=None) -> Path:
    """scene_io.py:365-379: 3N unshared vertices, N faces; PLY body built on the device."""
    path = Path(path)
    fmt = format.lower()
    if fmt not in ("ply", "obj"):
        raise ValueError(f"unsupported mesh format '{format}' (ply or obj)")
    soup = _device_soup(triangles)
    return _export_ply(soup, path, rasterizer) if fmt == "ply" else _export_obj(soup, path)


def import_ply(path, sigma: float = 0.05, dtype=None, rasterizer=None):
    """scene_io.py:417-455: a soup PLY back into a solid DeviceSoup (opacity 1,
    the given sigma, SH DC from the first vertex's colour)."""
    import torch
    from . import _lib
    from .rasterizer import DeviceSoup
    dtype = dtype or torch.float32
    path = Path(path)
    with open(path, "rb") as f:
        if f.readline().strip() != b"ply":
            raise ValueError(f"{path}: not a PLY file")
        n_vertex = n_face = None
        while True:
            line = f.readline()
            if not line:
                raise ValueError(f"{path}: unterminated PLY header")
            parts = line.decode("ascii", "replace").split()
            if parts[:2] == ["element", "vertex"]:
                n_vertex = int(parts[2])
            elif parts[:2] == ["element", "face"]:
                n_face = int(parts[2])
            elif parts == ["end_header"]:
                break
        if n_vertex is None or n_face is None or n_vertex != 3 * n_face:
            raise ValueError(f"{path}: not an unshared triangle-soup PLY")
        vraw = f.read(n_vertex * _VDT.itemsize)
        fraw = f.read(n_face * _FDT.itemsize)
    if len(vraw) != n_vertex * _VDT.itemsize or len(fraw) != n_face * _FDT.itemsize:
        raise ValueError(f"{path}: truncated PLY body")
    lib, ctx = _ctx(rasterizer)
    vb = torch.frombuffer(bytearray(vraw), dtype=torch.uint8).to("cuda") if n_vertex else \
        torch.zeros(16, dtype=torch.uint8, device="cuda")
    fb = torch.frombuffer(bytearray(fraw), dtype=torch.uint8).to("cuda") if n_face else \
        torch.zeros(16, dtype=torch.uint8, device="cuda")
    soup = DeviceSoup(torch.empty((n_face, 3, 3), dtype=dtype, device="cuda"),
                      torch.empty(n_face, dtype=dtype, device="cuda"),
                      torch.empty(n_face, dtype=dtype, device="cuda"),
                      torch.empty((n_face, 16, 3), dtype=dtype, device="cuda"), True)
    bad = torch.empty(1, dtype=torch.int64, device="cuda")
    p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(lib.ts_ply_unpack(ctx, p(vb), n_vertex, p(fb), n_face, float(sigma),
                                 1 if dtype == torch.float64 else 0, p(soup.vertices), p(soup.opacity),
                                 p(soup.sigma), p(soup.sh), p(bad), st), "ply_unpack")
    code = int(bad.item()) & 0xFFFFFFFFFFFFFFFF
    if code != 0xFFFFFFFFFFFFFFFF:
        if code >> 62 == 1:
            raise ValueError(f"{path}: non-triangle face found")
        raise IndexError(f"{path}: face {code & ((1 << 62) - 1)} indexes past the {n_vertex} vertices")
    return soup


def save_model(path, soup, scene=None):
    """scene_io.py:486-504: .npz with the reference's keys (fp64 arrays)."""
    s = _device_soup(soup)
    data = {"vertices": s.vertices.double().cpu().numpy(), "opacity": s.opacity.double().cpu().numpy(),
            "sigma": s.sigma.double().cpu().numpy(), "sh": s.sh.double().cpu().numpy(),
            "solid": np.array(bool(s.solid))}
    if scene is not None:
        cam_ids = sorted(scene.cameras)
        data["camera_ids"] = np.array(cam_ids)
        data["camera_params"] = np.array([[scene.cameras[i].fx, scene.cameras[i].fy, scene.cameras[i].cx,
                                           scene.cameras[i].cy, scene.cameras[i].width, scene.cameras[i].height]
                                          for i in cam_ids])
        data["view_names"] = np.array([v.name for v in scene.views])
        data["view_camera"] = np.array([v.camera_id for v in scene.views])
        data["view_split"] = np.array([v.split for v in scene.views])
        data["view_rotation"] = np.stack([v.pose.rotation for v in scene.views])
        data["view_translation"] = np.stack([v.pose.translation for v in scene.views])
    np.savez(path, **data)


def load_model(path, dtype=None):
    """scene_io.py:507-527: (DeviceSoup, views or None); views are
    (name, CameraIntrinsics, CameraPose, split)."""
    import torch
    from .rasterizer import DeviceSoup
    from .types import CameraIntrinsics, CameraPose, TriangleSoup
    dtype = dtype or torch.float32
    with np.load(path, allow_pickle=False) as data:
        soup = DeviceSoup.from_soup(TriangleSoup(vertices=data["vertices"], opacity=data["opacity"],
                                                 sigma=data["sigma"], sh=data["sh"]), dtype=dtype)
        soup.solid = bool(data["solid"])
        if "view_names" not in data:
            return soup, None
        cams = {int(c): CameraIntrinsics(fx=p[0], fy=p[1], cx=p[2], cy=p[3], width=int(p[4]), height=int(p[5]))
                for c, p in zip(data["camera_ids"], data["camera_params"])}
        views = [(str(name), cams[int(data["view_camera"][i])],
                  CameraPose(rotation=data["view_rotation"][i], translation=data["view_translation"][i]),
                  str(data["view_split"][i])) for i, name in enumerate(data["view_names"])]
        return soup, views
