"""Build liblidarsplat_cuda.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

Bit-exact translation units (projection, cull, grid, filter) are compiled with
-fmad=false in addition to their explicit round-to-nearest intrinsics; the
U-Net tensor-core units keep FMA contraction.  The CUDA runtime is linked
statically so the library loads on a GPU-less host (symbol checks in the CPU
test suite); the driver entry point needed for TMA descriptors is resolved at
run time through cudaGetDriverEntryPoint.

    python -m paper_2502_11618_b200.build [--force]
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "liblidarsplat_cuda.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
          "-I", os.path.join(ROOT, "include"), "-I", CSRC]
EXACT = ["-fmad=false"]

# (source, extra flags)
SOURCES = [
    ("project.cu", EXACT),
    ("filter.cu", EXACT),
    ("cull.cu", EXACT),
    ("grid.cu", EXACT),
    ("unet.cu", []),
]
HEADERS = ["ls_common.cuh", "umma.cuh"]


def _mtime(path: str) -> float:
    return os.path.getmtime(path) if os.path.exists(path) else 0.0


def _deps_mtime() -> float:
    paths = [os.path.join(CSRC, h) for h in HEADERS]
    paths.append(os.path.join(ROOT, "include", "lidarsplat_cuda.h"))
    paths.append(os.path.join(ROOT, "include", "lidarsplat_unet.h"))
    return max(_mtime(p) for p in paths)


def build(force: bool = False, verbose: bool = True) -> str:
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    dep_t = _deps_mtime()
    procs = []
    for src, flags in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _mtime(o) < max(_mtime(s), dep_t, _mtime(__file__)):
            cmd = [NVCC, *ARCH, *COMMON, *flags, "-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd), flush=True)
            procs.append((src, subprocess.Popen(cmd)))
    for src, p in procs:
        if p.wait() != 0:
            raise RuntimeError(f"nvcc failed on {src}")
    if procs or not os.path.exists(LIB) or _mtime(LIB) < max(_mtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
