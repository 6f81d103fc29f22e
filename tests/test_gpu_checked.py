"""The checked build (LS_DEBUG_BOUNDS=1 -> liblidarsplat_cuda_debug.so).

compute-sanitizer is not available on the GPU pool, so out-of-bounds scatter
targets and work-list overruns are caught by the kernels' own LS_ASSERT checks
(csrc/ls_common.cuh), compiled into a separate library.  CPU: the checked
library carries the device asserts and the product library does not.  GPU:
the projection / multi-view / filter / engine parity suites pass on the
checked library (a failed check aborts the kernel with cudaErrorAssert).
"""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2502_11618_b200")
PRODUCT = os.path.join(PKG, "liblidarsplat_cuda.so")
CHECKED = os.path.join(PKG, "liblidarsplat_cuda_debug.so")


def _assert_refs(lib):
    out = subprocess.run(["cuobjdump", "-elf", lib], capture_output=True, text=True,
                         check=True).stdout
    return out.count("__assertfail")


def test_checked_library_has_asserts_product_has_none():
    assert os.path.exists(CHECKED), "build it with `python -m paper_2502_11618_b200.build --debug`"
    assert _assert_refs(CHECKED) > 0
    assert _assert_refs(PRODUCT) == 0


def _exports(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True,
                         check=True).stdout
    return {l.split()[-1] for l in out.splitlines() if l.split()[-1].startswith("ls_")}


def test_checked_library_exports_the_same_abi():
    exp = _exports(PRODUCT)
    assert len(exp) > 20 and _exports(CHECKED) == exp


@pytest.mark.gpu
def test_parity_suites_on_checked_library():
    env = dict(os.environ, LS_DEBUG_BOUNDS="1")
    probe = subprocess.run([sys.executable, "-c",
                            "from paper_2502_11618_b200 import _lib; print(_lib.LIB_PATH)"],
                           cwd=ROOT, env=env, capture_output=True, text=True, check=True)
    assert probe.stdout.strip() == CHECKED
    suites = ["tests/test_gpu_projection.py", "tests/test_gpu_views.py",
              "tests/test_gpu_filter.py", "tests/test_gpu_kernels.py",
              "tests/test_gpu_engine.py"]
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        "-p", "no:cacheprovider", *suites], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-2000:]
    assert " passed" in p.stdout
