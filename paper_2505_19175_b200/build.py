"""Build the sm_100a C-ABI library ``libtrisplat_b200.so`` in-tree with nvcc.

    python -m paper_2505_19175_b200.build          # incremental
    python -m paper_2505_19175_b200.build --force
    python -m paper_2505_19175_b200.build --checked  # + libtrisplat_b200_checked.so

The checked build compiles the TS_ASSERT bounds / invariant checks into the
kernels (device asserts); tests run against it with
TRISPLAT_B200_LIB=paper_2505_19175_b200/libtrisplat_b200_checked.so.

Translation units that restate fp64 reference arithmetic are compiled with
``-fmad=false`` (no FMA contraction, as numba without fastmath); the fast
fp32 kernels keep FMA.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libtrisplat_b200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
          "--expt-relaxed-constexpr", "-I", INCLUDE, "-I", CSRC]
# per-TU extra flags
EXTRA = {
    "ts_exact.cu": ["-fmad=false"],
}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def host_cxx_flags():
    cuda_inc = os.path.join(os.path.dirname(os.path.dirname(os.path.realpath(nvcc()))), "include")
    return ["-O3", "-std=c++17", "-fPIC", "-pthread", "-I", INCLUDE, "-I", CSRC, "-I", cuda_inc]


def headers_mtime() -> float:
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(INCLUDE, "trisplat_b200.h"))
    return max(os.path.getmtime(h) for h in hs if os.path.exists(h))


def build(force: bool = False, verbose: bool = False, checked: bool = False, defines=(), out=None) -> str:
    """defines: extra -D flags for a measurement variant, built into its own
    directory and library ``out`` (product builds take none)."""
    tag = ("_checked" if checked else "") + "".join("_" + d.replace("=", "") for d in defines)
    build_dir = BUILD + tag
    lib = out or (LIB.replace(".so", tag + ".so") if tag else LIB)
    extra_all = (["-DTS_CHECKED"] if checked else []) + ["-D" + d for d in defines]
    os.makedirs(build_dir, exist_ok=True)
    hm = headers_mtime()
    objs = []
    changed = force or not os.path.exists(lib)
    for src in sources():
        sp = os.path.join(CSRC, src)
        obj = os.path.join(build_dir, os.path.splitext(src)[0] + ".o")
        objs.append(obj)
        if (not force and os.path.exists(obj) and os.path.getmtime(obj) >= os.path.getmtime(sp)
                and os.path.getmtime(obj) >= hm):
            continue
        if src.endswith(".cpp"):  # host-only code: the host compiler directly
            cmd = [os.environ.get("CXX", "g++")] + host_cxx_flags() + extra_all + ["-c", sp, "-o", obj]
        else:
            cmd = [nvcc()] + ARCH + COMMON + extra_all + EXTRA.get(src, []) + ["-c", sp, "-o", obj]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        changed = True
    if changed or any(os.path.getmtime(o) > os.path.getmtime(lib) for o in objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", lib] + objs + ["-lcudart", "-Xcompiler", "-pthread"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv, defines=defs,
          out=outs[0] if outs else None)
