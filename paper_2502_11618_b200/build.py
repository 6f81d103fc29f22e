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


# Checked build (LS_DEBUG_BOUNDS=1): the index-arithmetic kernels with their
# LS_ASSERT bounds checks compiled in, linked with the product U-Net object
# (whose global traffic goes through bounds-checked TMA), into a separate
# library that `_lib` loads when LS_DEBUG_BOUNDS=1 is set at run time.
BUILD_DEBUG = os.path.join(PKG, "_build_debug")
LIB_DEBUG = os.path.join(PKG, "liblidarsplat_cuda_debug.so")
CHECKED = {"project.cu", "filter.cu", "cull.cu", "grid.cu"}


def build(force: bool = False, verbose: bool = True, debug: bool = False) -> str:
    if debug:
        build(force, verbose)  # the product objects (unet.o is shared)
    bdir, lib = (BUILD_DEBUG, LIB_DEBUG) if debug else (BUILD, LIB)
    os.makedirs(bdir, exist_ok=True)
    objs = []
    dep_t = _deps_mtime()
    procs = []
    for src, flags in SOURCES:
        s = os.path.join(CSRC, src)
        if debug and src not in CHECKED:
            objs.append(os.path.join(BUILD, src.replace(".cu", ".o")))
            continue
        o = os.path.join(bdir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _mtime(o) < max(_mtime(s), dep_t, _mtime(__file__)):
            extra = ["-DLS_DEBUG_BOUNDS"] if debug else []
            cmd = [NVCC, *ARCH, *COMMON, *flags, *extra, "-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd), flush=True)
            procs.append((src, subprocess.Popen(cmd)))
    for src, p in procs:
        if p.wait() != 0:
            raise RuntimeError(f"nvcc failed on {src}")
    if procs or not os.path.exists(lib) or _mtime(lib) < max(_mtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", lib, *objs]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv,
          debug="--debug" in sys.argv or os.environ.get("LS_DEBUG_BOUNDS") == "1")
