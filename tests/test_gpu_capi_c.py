"""The C ABI from C: tests/capi_smoke.c is compiled with gcc against
include/lidarsplat_cuda.h and the in-tree liblidarsplat_cuda.so, and renders a
tiny scene with no Python on the path (what INTEGRATION.md's cgo / JNI /
C++ callers do)."""

import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_program_renders_expected_pixels(cuda_ready, tmp_path):
    pkg = os.path.join(ROOT, "paper_2502_11618_b200")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    exe = tmp_path / "capi_smoke"
    subprocess.run(["gcc", "-O1", os.path.join(ROOT, "tests", "capi_smoke.c"),
                    "-I", os.path.join(ROOT, "include"), "-I", os.path.join(cuda, "include"),
                    "-L", pkg, "-llidarsplat_cuda", "-L", os.path.join(cuda, "lib64"),
                    "-lcudart", f"-Wl,-rpath,{pkg}", f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}",
                    "-lm", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr + out.stdout
    assert "capi_smoke OK" in out.stdout
