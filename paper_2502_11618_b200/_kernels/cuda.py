"""The ``cuda`` kernel backend: the reference's 8-function `_kernels` protocol
(_native.pyx:19-297) served by the sm_100a library through its C ABI.

Each function takes and returns host numpy arrays with the reference's
signatures, dtypes and in/out conventions (typed-memoryview checks raise
ValueError on dtype/shape/contiguity mismatch, like Cython's).  Internally the
inputs are staged to the GPU, the device twin runs on the current stream and
the results are copied back.  The per-frame pipeline does not use this module
(it keeps everything device-resident, see ..device); it exists so code written
against the reference backend protocol -- and the parity suite -- run unchanged.
"""

from __future__ import annotations

import numpy as np

from .. import _lib

name = "cuda"


def _need(arr, dtype, ndim, what, writable=False):
    if not isinstance(arr, np.ndarray):
        raise TypeError(f"{what}: expected a numpy array, got {type(arr).__name__}")
    if arr.dtype != np.dtype(dtype):
        raise ValueError(f"{what}: buffer dtype mismatch, expected {np.dtype(dtype)} "
                         f"but got {arr.dtype}")
    if arr.ndim != ndim:
        raise ValueError(f"{what}: buffer has wrong number of dimensions "
                         f"(expected {ndim}, got {arr.ndim})")
    if not arr.flags.c_contiguous:
        raise ValueError(f"{what}: ndarray is not C-contiguous")
    if writable and not arr.flags.writeable:
        raise ValueError(f"{what}: buffer source array is read-only")
    return arr


class _Stage:
    """Host->device staging that keeps every uploaded tensor alive until the
    call's results are read back (a bare ``tensor.data_ptr()`` would let the
    caching allocator recycle the block while the kernel is still queued)."""

    def __init__(self):
        self.keep = []

    def __call__(self, arr) -> int:
        import torch

        t = torch.from_numpy(np.array(arr, copy=True)).to(_lib.device())
        self.keep.append(t)
        return t.data_ptr()


def _dev(arr):
    import torch

    return torch.from_numpy(np.array(arr, copy=True)).to(_lib.device())


def _empty(shape, dtype):
    import torch

    return torch.empty(shape, dtype=dtype, device=_lib.device())


def _host(t) -> np.ndarray:
    return t.cpu().numpy()


def _cam(rot, t, fx, fy, cx, cy, width, height, z_near, z_far):
    c = _lib.LsCamera()
    c.rot[:] = np.ascontiguousarray(rot, np.float64).ravel().tolist()
    c.t[:] = np.ascontiguousarray(t, np.float64).ravel().tolist()
    c.fx, c.fy, c.cx, c.cy = float(fx), float(fy), float(cx), float(cy)
    c.width, c.height = int(width), int(height)
    c.z_near, c.z_far = float(z_near), float(z_far)
    return c


def assign_cells(positions, origin, cell_size, dims):
    up = _Stage()
    _need(positions, np.float32, 2, "positions")
    origin = np.ascontiguousarray(_need(origin, np.float64, 1, "origin"))
    dims = np.ascontiguousarray(_need(dims, np.int64, 1, "dims"))
    n = positions.shape[0]
    ids = _empty((n,), __import__("torch").int64)
    lib = _lib.load()
    _lib.check(lib.ls_assign_cells(up(positions), n,
                                   origin.ctypes.data, float(cell_size), dims.ctypes.data,
                                   ids.data_ptr(), _lib.stream_ptr()), "assign_cells")
    return _host(ids)


def counting_sort(ids, n_cells):
    up = _Stage()
    import torch

    _need(ids, np.int64, 1, "ids")
    n, n_cells = ids.shape[0], int(n_cells)
    offsets = np.zeros(n_cells + 1, np.int64)
    if n == 0:
        return offsets, np.empty(0, np.int64)
    lib = _lib.load()
    ws_bytes = lib.ls_counting_sort_workspace(n, n_cells)
    if ws_bytes == 0:
        raise ValueError("counting_sort: sizes out of range")
    ws = _empty((ws_bytes,), torch.uint8)
    d_off = _empty((n_cells + 1,), torch.int64)
    d_order = _empty((n,), torch.int64)
    _lib.check(lib.ls_counting_sort(up(ids), n, n_cells, d_off.data_ptr(),
                                    d_order.data_ptr(), ws.data_ptr(), ws_bytes,
                                    _lib.stream_ptr()), "counting_sort")
    return _host(d_off), _host(d_order)


def project_min_depth(positions, starts, ends, rot, t, fx, fy, cx, cy, width, height,
                      z_near, z_far, minz, pix_cache, z_cache):
    up = _Stage()
    import torch

    _need(positions, np.float32, 2, "positions")
    _need(starts, np.int64, 1, "starts")
    _need(ends, np.int64, 1, "ends")
    _need(minz, np.float64, 1, "minz", writable=True)
    _need(pix_cache, np.int64, 1, "pix_cache", writable=True)
    _need(z_cache, np.float64, 1, "z_cache", writable=True)
    nr = starts.shape[0]
    if nr == 0:
        return None
    lib = _lib.load()
    cam = _cam(rot, t, fx, fy, cx, cy, width, height, z_near, z_far)
    d_minz = _dev(minz)
    d_pix = _empty(pix_cache.shape, torch.int64)
    d_z = _empty(z_cache.shape, torch.float64)
    ws_bytes = lib.ls_ranges_workspace(nr)
    ws = _empty((ws_bytes,), torch.uint8)
    _lib.check(lib.ls_project_min_depth(up(positions), up(starts),
                                        up(ends), nr, cam, d_minz.data_ptr(),
                                        d_pix.data_ptr(), d_z.data_ptr(), ws.data_ptr(),
                                        ws_bytes, _lib.stream_ptr()), "project_min_depth")
    minz[:] = _host(d_minz)
    pix_cache[:] = _host(d_pix)
    z_cache[:] = _host(d_z)
    return None


def project_accumulate(colors, starts, ends, pix_cache, z_cache, eps_rel, minz, accum):
    up = _Stage()
    import torch

    _need(colors, np.uint8, 2, "colors")
    _need(starts, np.int64, 1, "starts")
    _need(ends, np.int64, 1, "ends")
    _need(pix_cache, np.int64, 1, "pix_cache")
    _need(z_cache, np.float64, 1, "z_cache")
    _need(minz, np.float64, 1, "minz")
    _need(accum, np.uint64, 2, "accum", writable=True)
    nr = starts.shape[0]
    if nr == 0:
        return None
    lib = _lib.load()
    d_acc = _dev(accum.view(np.int64))
    ws_bytes = lib.ls_ranges_workspace(nr)
    ws = _empty((ws_bytes,), torch.uint8)
    _lib.check(lib.ls_project_accumulate(up(colors), up(starts),
                                         up(ends), nr, up(pix_cache),
                                         up(z_cache), float(eps_rel),
                                         up(minz), d_acc.data_ptr(), ws.data_ptr(),
                                         ws_bytes, _lib.stream_ptr()), "project_accumulate")
    accum[:] = _host(d_acc).view(np.uint64)
    return None


def min_pool_2x2(img):
    up = _Stage()
    import torch

    _need(img, np.float32, 2, "img")
    h, w = img.shape
    out = _empty(((h + 1) // 2, (w + 1) // 2), torch.float32)
    _lib.check(_lib.load().ls_min_pool_2x2(up(img), h, w, out.data_ptr(),
                                           _lib.stream_ptr()), "min_pool_2x2")
    return _host(out)


def laplacian_edges(img, threshold):
    up = _Stage()
    import torch

    _need(img, np.float32, 2, "img")
    h, w = img.shape
    out = _empty((h, w), torch.uint8)
    _lib.check(_lib.load().ls_laplacian_edges(up(img), h, w, float(threshold),
                                              out.data_ptr(), _lib.stream_ptr()),
               "laplacian_edges")
    return _host(out)


def filter_keep(coarse, edges, fine, filter_strength):
    up = _Stage()
    import torch

    _need(coarse, np.float32, 2, "coarse")
    _need(edges, np.uint8, 2, "edges")
    _need(fine, np.float32, 2, "fine")
    ch, cw = coarse.shape
    fh, fw = fine.shape
    out = _empty((fh, fw), torch.float32)
    _lib.check(_lib.load().ls_filter_keep(up(coarse), ch, cw,
                                          up(edges), up(fine), fh, fw,
                                          float(filter_strength), out.data_ptr(),
                                          _lib.stream_ptr()), "filter_keep")
    return _host(out)


def bilinear_fill(coarse, fine):
    up = _Stage()
    import torch

    _need(coarse, np.float32, 2, "coarse")
    _need(fine, np.float32, 2, "fine")
    ch, cw = coarse.shape
    fh, fw = fine.shape
    out = _empty((fh, fw), torch.float32)
    _lib.check(_lib.load().ls_bilinear_fill(up(coarse), ch, cw,
                                            up(fine), fh, fw, out.data_ptr(),
                                            _lib.stream_ptr()), "bilinear_fill")
    return _host(out)
