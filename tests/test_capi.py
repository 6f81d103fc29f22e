"""The C-ABI library loads on a GPU-less host and exports every entry point
declared in include/*.h; the ctypes table covers all of them.  CPU only."""

import ctypes
import glob
import os
import re

from conftest import ROOT

from paper_2502_11618_b200 import _lib


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"\b(ls_[a-z0-9_]+)\s*\(", text))
    return names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 25
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_table_matches_headers():
    assert declared_symbols() == set(_lib.SIGNATURES)


def test_version_and_status_strings():
    lib = _lib.load()
    assert lib.ls_version() >= 1
    assert lib.ls_status_string(0) == b"ok"
    assert lib.ls_status_string(_lib.LS_EINVAL) == b"invalid argument"


def test_workspace_queries_need_no_gpu():
    lib = _lib.load()
    assert lib.ls_ranges_workspace(4) == 40
    assert lib.ls_pyramid_floats(1080, 1920, 4) == 2 * sum(
        ((1080 + 2**k - 1) // 2**k) * ((1920 + 2**k - 1) // 2**k) for k in range(1, 5))
    assert lib.ls_pyramid_floats(16, 16, 0) == -1
    assert lib.ls_compact_workspace(1000) > 0
    assert lib.ls_counting_sort_workspace(1000, 64) > 0


def test_invalid_arguments_rejected_before_launch():
    lib = _lib.load()
    assert lib.ls_min_pool_2x2(None, 0, 5, None, None) == _lib.LS_EINVAL
    assert lib.ls_frame_pass1(None, None, None, None, None, None, None, None) == _lib.LS_EINVAL
    f = _lib.LsFilterParams()
    f.levels_n, f.filter_strength, f.edge_threshold = 5, 0.1, 0.25
    # 16x16 is too small for 5 levels (filtering.py:75-78)
    assert lib.ls_filter_depth_image(1, 16, 16, f, 1, 1, None) == _lib.LS_EINVAL
