"""ctypes binding of liblidarsplat_cuda.so (include/lidarsplat_cuda.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is visible, every operator raises ``CudaUnavailableError`` instead of
silently computing on the host.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import LidarSplatError

_HERE = os.path.dirname(os.path.abspath(__file__))
# LS_DEBUG_BOUNDS=1 selects the checked build (build.py --debug): same kernels
# with their bounds asserts compiled in.
LIB_PATH = os.path.join(_HERE, "liblidarsplat_cuda_debug.so"
                        if os.environ.get("LS_DEBUG_BOUNDS") == "1" else "liblidarsplat_cuda.so")
# experiment builds (scripts/exp/*.sh) point LS_LIB_PATH at their own library
LIB_PATH = os.environ.get("LS_LIB_PATH") or LIB_PATH

LS_EINVAL = -22
LS_TILE_POINTS = 128
LS_PACKED_COUNT_LIMIT = 65793
LS_MAX_VIEWS = 8
INF_BITS = 0x7FF0000000000000


class CudaUnavailableError(LidarSplatError, RuntimeError):
    """The CUDA extension or device needed by the product path is missing."""


class LsCamera(ctypes.Structure):
    _fields_ = [("rot", ctypes.c_double * 9), ("t", ctypes.c_double * 3),
                ("fx", ctypes.c_double), ("fy", ctypes.c_double),
                ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("width", ctypes.c_int64), ("height", ctypes.c_int64),
                ("z_near", ctypes.c_double), ("z_far", ctypes.c_double)]


class LsScene(ctypes.Structure):
    _fields_ = [("d_positions", ctypes.c_void_p), ("d_colors", ctypes.c_void_p),
                ("n_points", ctypes.c_int64),
                ("d_occ_cells", ctypes.c_void_p), ("d_occ_offsets", ctypes.c_void_p),
                ("n_occ", ctypes.c_int64),
                ("d_tile_c0", ctypes.c_void_p), ("d_tile_c1", ctypes.c_void_p),
                ("n_tiles", ctypes.c_int64),
                ("origin", ctypes.c_double * 3), ("cell_size", ctypes.c_double),
                ("dims", ctypes.c_int64 * 3)]


class LsFilterParams(ctypes.Structure):
    _fields_ = [("levels_n", ctypes.c_int32), ("filter_strength", ctypes.c_double),
                ("edge_threshold", ctypes.c_double)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double
_F = ctypes.c_float
_SZ = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/lidarsplat_cuda.h + lidarsplat_unet.h
SIGNATURES = {
    "ls_version": (ctypes.c_int, []),
    "ls_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "ls_assign_cells": (ctypes.c_int, [_P, _I64, _P, _D, _P, _P, _P]),
    "ls_counting_sort_workspace": (_SZ, [_I64, _I64]),
    "ls_counting_sort": (ctypes.c_int, [_P, _I64, _I64, _P, _P, _P, _SZ, _P]),
    "ls_ranges_workspace": (_SZ, [_I64]),
    "ls_project_min_depth": (ctypes.c_int, [_P, _P, _P, _I64, ctypes.POINTER(LsCamera),
                                            _P, _P, _P, _P, _SZ, _P]),
    "ls_project_accumulate": (ctypes.c_int, [_P, _P, _P, _I64, _P, _P, _D, _P, _P, _P, _SZ,
                                             _P]),
    "ls_min_pool_2x2": (ctypes.c_int, [_P, _I64, _I64, _P, _P]),
    "ls_laplacian_edges": (ctypes.c_int, [_P, _I64, _I64, _D, _P, _P]),
    "ls_filter_keep": (ctypes.c_int, [_P, _I64, _I64, _P, _P, _I64, _I64, _D, _P, _P]),
    "ls_bilinear_fill": (ctypes.c_int, [_P, _I64, _I64, _P, _I64, _I64, _P, _P]),
    "ls_assemble": (ctypes.c_int, [_P, _P, _I64, _P, _P, _P, _P]),
    "ls_morton_order_workspace": (_SZ, [_I64, _I64]),
    "ls_morton_order": (ctypes.c_int, [_P, _I64, _P, _D, _P, _P, _P, _SZ, _P]),
    "ls_gather_points": (ctypes.c_int, [_P, _P, _P, _I64, _P, _P, _P]),
    "ls_occupied_workspace": (_SZ, [_I64]),
    "ls_occupied_cells": (ctypes.c_int, [_P, _I64, _P, _P, _P, _P, _SZ, _P]),
    "ls_scene_tile_index": (ctypes.c_int, [_P, _I64, _I64, _P, _P, _P]),
    "ls_cull": (ctypes.c_int, [ctypes.POINTER(LsScene), _P, _D, _P, _P]),
    "ls_compact_workspace": (_SZ, [_I64]),
    "ls_cull_compact": (ctypes.c_int, [_P, _P, _I64, _P, _P, _P, _SZ, _P]),
    "ls_tile_worklist": (ctypes.c_int, [ctypes.POINTER(LsScene), _P, _P, _P, _P]),
    "ls_frame_project": (ctypes.c_int, [ctypes.POINTER(LsScene), _P, _P, _P,
                                        ctypes.POINTER(LsCamera), _D, _P, _P, _P, _P]),
    "ls_frame_cache_bytes": (_SZ, [ctypes.POINTER(LsScene)]),
    "ls_frame_pass1": (ctypes.c_int, [ctypes.POINTER(LsScene), _P, _P, _P,
                                      ctypes.POINTER(LsCamera), _P, _P, _P]),
    "ls_frame_pass2": (ctypes.c_int, [ctypes.POINTER(LsScene), _P, _P, _P,
                                      ctypes.POINTER(LsCamera), _D, _P, _P, _P, _P]),
    "ls_tile_worklist_views": (ctypes.c_int, [ctypes.POINTER(LsScene), _P, _I64, _I32, _P, _P,
                                              _P, _P]),
    "ls_frame_project_views": (ctypes.c_int, [ctypes.POINTER(LsScene), _P, _I64, _P, _P, _P,
                                              _P, _I32, _D, _P, _P, _P, _P]),
    "ls_frame_views_cache_bytes": (_SZ, [ctypes.POINTER(LsScene), _I32]),
    "ls_pyramid_floats": (_I64, [_I64, _I64, _I32]),
    "ls_frame_finish": (ctypes.c_int, [_P, _P, _I64, _I64, ctypes.POINTER(LsFilterParams),
                                       _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I32, _D, _P, _P,
                                       _P]),
    "ls_unet_pack_rgbda": (ctypes.c_int, [_P, _I64, _I64, _I32, _D, _P, _P]),
    "ls_filter_depth_image": (ctypes.c_int, [_P, _I64, _I64, ctypes.POINTER(LsFilterParams),
                                             _P, _P, _P]),
    "ls_depth_filter_frame": (ctypes.c_int, [_P, _P, _P, _I64, _I64,
                                             ctypes.POINTER(LsFilterParams), _P, _P, _P, _P, _P,
                                             _P]),
    "ls_frame_graph_set_camera": (ctypes.c_int, [_P, _P, ctypes.POINTER(LsCamera), _P]),
    "ls_filter_sweep_floats": (_I64, [_I64, _I64, _I32, _I32]),
    "ls_depth_filter_sweep": (ctypes.c_int, [_P, _P, _P, _I64, _I64, _I32, _D, _P, _I32, _P,
                                             _P, _P, _P, _P, _P]),
    # lidarsplat_unet.h
    "ls_conv_plan_create": (ctypes.c_void_p, [_P, _I32, _P, _I32, _I32, _I32, _I32, _P, _I32,
                                              _I32, _I32, _P, _P, _I32, _F, _P, _P, _P, _P, _P,
                                              _I32, _P, ctypes.POINTER(ctypes.c_int32)]),
    "ls_conv_plan_launch": (ctypes.c_int, [_P, _P]),
    "ls_conv_plan_destroy": (None, [_P]),
    "ls_conv_plan_set_rows": (ctypes.c_int, [_P, _I32, _I32]),
    "ls_conv_plan_set_reverse": (ctypes.c_int, [_P, _I32]),
    "ls_conv_plan_create_upfused": (_P, [_P, _P, _P, _P, _I32, _I32, _I32, _P, _P, _P, _I32,
                                         ctypes.c_float, _P, _P]),
    "ls_conv_plan_tile_rows": (_I32, [_P]),
    "ls_conv2d": (ctypes.c_int, [_P, _I32, _P, _I32, _I32, _I32, _I32, _P, _I32, _I32, _P, _P,
                                 _I32, _F, _P, _P, _P, _P, _P, _I32, _P, _P]),
    "ls_conv_transpose2x2": (ctypes.c_int, [_P, _I32, _I32, _I32, _I32, _P, _I32, _P, _P, _P,
                                            _P]),
}

_lock = threading.Lock()
_lib = None


def load(required: bool = True):
    """Load (once) and return the ctypes library."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            if not required:
                return None
            raise CudaUnavailableError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2502_11618_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(status: int, what: str) -> None:
    if status != 0:
        msg = load().ls_status_string(status).decode()
        if status == LS_EINVAL:
            raise ValueError(f"{what}: {msg}")
        raise RuntimeError(f"{what} failed: CUDA error {status} ({msg})")


def device():
    """The CUDA device the product path runs on; raises if none."""
    import torch

    if not torch.cuda.is_available():
        raise CudaUnavailableError("no CUDA device visible: the B200 path has no CPU fallback")
    load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    import torch

    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def make_camera(camera) -> LsCamera:
    pose = camera.world_to_camera
    rot = np.ascontiguousarray(pose.rotation, np.float64).ravel()
    tr = np.ascontiguousarray(pose.translation, np.float64).ravel()
    c = LsCamera()
    c.rot[:] = rot.tolist()
    c.t[:] = tr.tolist()
    c.fx, c.fy, c.cx, c.cy = (float(camera.fx), float(camera.fy), float(camera.cx),
                              float(camera.cy))
    c.width, c.height = int(camera.width), int(camera.height)
    c.z_near, c.z_far = float(camera.z_near), float(camera.z_far)
    return c


def make_filter(params) -> LsFilterParams:
    f = LsFilterParams()
    f.levels_n = int(params.levels_n)
    f.filter_strength = float(params.filter_strength)
    f.edge_threshold = float(params.edge_threshold)
    return f
