"""Deterministic point projection into an RGBDA frame (reference render.py).

Two passes over the candidate points, on the GPU:
  pass 1: per-pixel minimum camera depth (64-bit atomicMin on the f64 bits)
  pass 2: integer colour sums of every point with zc <= minz*(1+eps)
then the integer-mean assembly.  Min and integer add are order-free, so the
frame is bit-identical to the reference for any point order and schedule.

``project_points`` on a grid runs the device fast path: culling bits + warp
tile passes over the resident cell-major scan + the fused assembly kernel.
``project_candidates`` keeps the reference's range/cache interface (the
backend-protocol twins).  Both return frames identical to the reference's.
"""

from __future__ import annotations

import os
import threading
import types
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._kernels import get_backend
from .cloud import PointCloud
from .frame import FrameRGBDA, RenderParams
from .geometry import CameraModel, extract_frustum
from .grid import DeviceScene, UniformGrid, cull_cells


def worker_count(n_points: int) -> int:
    """Kept for API compatibility: one GPU stream does the whole pass."""
    return 1


@dataclass
class Candidates:
    """Points surviving cell culling: ranges into position/colour arrays."""

    positions: np.ndarray
    colors: np.ndarray
    starts: np.ndarray
    ends: np.ndarray

    @property
    def count(self) -> int:
        return int((self.ends - self.starts).sum())


def candidates(cloud: PointCloud, grid: UniformGrid | None, camera: CameraModel) -> Candidates:
    """Candidate set for a view: the whole cloud when ``grid`` is None, else the
    merged ranges of the frustum-culled cells (culled on the GPU)."""
    if grid is None:
        return Candidates(cloud.positions, cloud.colors, np.zeros(1, np.int64),
                          np.array([cloud.count], np.int64))
    starts, ends = grid.cell_ranges(cull_cells(grid, extract_frustum(camera)))
    return Candidates(grid.sorted_positions, grid.sorted_colors, starts, ends)


def project_candidates(cands: Candidates, camera: CameraModel, params: RenderParams,
                       backend=None, workers: int | None = None) -> FrameRGBDA:
    """Rasterise candidate ranges with the reference's two-pass interface."""
    import torch

    kern = get_backend() if backend is None else backend
    w, h = int(camera.width), int(camera.height)
    rot = camera.world_to_camera.rotation
    t = camera.world_to_camera.translation
    n = cands.count
    minz = np.full(h * w, np.inf)
    pix = np.empty(n, np.int64)
    z = np.empty(n, np.float64)
    starts = np.ascontiguousarray(cands.starts, np.int64)
    ends = np.ascontiguousarray(cands.ends, np.int64)
    kern.project_min_depth(cands.positions, starts, ends, rot, t, float(camera.fx),
                           float(camera.fy), float(camera.cx), float(camera.cy), w, h,
                           float(camera.z_near), float(camera.z_far), minz, pix, z)
    accum = np.zeros((h * w, 4), np.uint64)
    kern.project_accumulate(cands.colors, starts, ends, pix, z,
                            float(params.zbuffer_epsilon_rel), minz, accum)
    return assemble_frame(minz, accum, w, h)


def assemble_frame(minz: np.ndarray, accum: np.ndarray, width: int, height: int) -> FrameRGBDA:
    """Fold pass buffers (f64 minz, u64 x4 accum) into a frame on the GPU."""
    import torch

    dev = _lib.device()
    npix = width * height
    d_minz = torch.from_numpy(np.ascontiguousarray(minz, np.float64)).to(dev)
    d_acc = torch.from_numpy(np.ascontiguousarray(accum).view(np.int64)).to(dev)
    rgb = torch.empty((height, width, 3), dtype=torch.float32, device=dev)
    depth = torch.empty((height, width), dtype=torch.float32, device=dev)
    alpha = torch.empty((height, width), dtype=torch.uint8, device=dev)
    _lib.check(_lib.load().ls_assemble(d_minz.data_ptr(), d_acc.data_ptr(), npix,
                                       rgb.data_ptr(), depth.data_ptr(), alpha.data_ptr(),
                                       _lib.stream_ptr()), "assemble")
    return FrameRGBDA(rgb.cpu().numpy(), depth.cpu().numpy(), alpha.cpu().numpy())


class FrameBuffers:
    """Per-resolution device buffers of the fused frame path."""

    def __init__(self, width: int, height: int, device):
        import torch

        self.width, self.height = int(width), int(height)
        npix = self.width * self.height
        self.minz = torch.full((npix,), _lib.INF_BITS, dtype=torch.int64, device=device)
        # {sum r, sum g, sum b, count} as f32 (exact integers below 2^24)
        self.accum = torch.zeros((npix, 4), dtype=torch.float32, device=device)
        self.rgb = torch.empty((self.height, self.width, 3), dtype=torch.float32, device=device)
        self.depth = torch.empty((self.height, self.width), dtype=torch.float32, device=device)
        self.alpha = torch.empty((self.height, self.width), dtype=torch.uint8, device=device)
        self.flags = torch.zeros(1, dtype=torch.int32, device=device)


# Pass-1 -> pass-2 cache (ls_frame_cache_bytes): pass 2 decides from each
# candidate's cached pixel + f16 rounded-down depth instead of re-projecting.  Frames are
# identical either way; LS_FRAME_CACHE=0 selects re-projection.
USE_FRAME_CACHE = os.environ.get("LS_FRAME_CACHE", "1") != "0"


def frame_cache(scene, camera: CameraModel, scratch=None):
    """The scratch's pass-1 -> pass-2 cache (allocated once per FrameScratch;
    default: the scene's own), or None when disabled or the frame is too large
    for u32 pixel slots."""
    if not USE_FRAME_CACHE or camera.width * camera.height >= 0xFFFFFFFF:
        return None
    sc = scratch or scene.scratch
    if sc.frame_cache is None:
        import torch

        nbytes = int(_lib.load().ls_frame_cache_bytes(scene.struct))
        sc.frame_cache = torch.empty(max(nbytes // 4, 4), dtype=torch.int32,
                                     device=_lib.device())
    return sc.frame_cache


def project_scene(scene: DeviceScene, camera: CameraModel, eps_rel: float, bufs: FrameBuffers,
                  cull: bool = True, filter_params=None, filtered=None, keep=None,
                  unet_in=None, unet_znear: float = 0.1, pyramid=None,
                  stage_events=None, raw: bool = True, scratch=None, flags=None) -> None:
    """Enqueue one fused frame on the current stream (no host sync):
    cull -> pass 1 -> pass 2 -> assemble (+ filter / U-Net input).
    ``stage_events``: optional CUDA events recorded after cull, pass 1,
    pass 2 and assemble/filter.  ``raw=False`` (U-Net-only frames: a filter,
    ``unet_in`` and no filtered outputs) skips the raw f32 rgb / alpha frame:
    the assembly writes the U-Net input directly (bufs.rgb / bufs.alpha are
    then not updated).  ``scratch``: the FrameScratch of this frame stream
    (default: the scene's shared one -- hold ``scene.lock`` until the frame
    has completed).  ``flags``: int32 word the assembly ORs 1 into when a
    pixel's f32 accumulator reached 2^24 (default ``bufs.flags``)."""
    lib = _lib.load()
    st = _lib.stream_ptr()
    cam = _lib.make_camera(camera)
    ev = stage_events or [None] * 4
    bits = lst = cnt = None
    if cull:
        bits = scene.cull_bits(extract_frustum(camera).planes, scratch=scratch).data_ptr()
        tl, tc = scene.worklist(scratch)
        lst, cnt = tl.data_ptr(), tc.data_ptr()
    if ev[0] is not None:
        ev[0].record()
    cache = _lib.ptr(frame_cache(scene, camera, scratch))
    _lib.check(lib.ls_frame_pass1(scene.struct, bits, lst, cnt, cam, bufs.minz.data_ptr(), cache,
                                  st), "frame_pass1")
    if ev[1] is not None:
        ev[1].record()
    _lib.check(lib.ls_frame_pass2(scene.struct, bits, lst, cnt, cam, float(eps_rel),
                                  bufs.minz.data_ptr(), cache, bufs.accum.data_ptr(), st),
               "frame_pass2")
    if ev[2] is not None:
        ev[2].record()
    fp = None if filter_params is None else _lib.make_filter(filter_params)
    frgb = fdepth = falpha = None
    if filtered is not None:
        frgb, fdepth, falpha = (_lib.ptr(filtered[0]), _lib.ptr(filtered[1]),
                                _lib.ptr(filtered[2]))
    unet_h, unet_c = (0, 0) if unet_in is None else (int(unet_in.shape[-3]),
                                                      int(unet_in.shape[-1]))
    raw_rgb, raw_alpha = (bufs.rgb.data_ptr(), bufs.alpha.data_ptr()) if raw else (None, None)
    _lib.check(lib.ls_frame_finish(bufs.minz.data_ptr(), bufs.accum.data_ptr(), bufs.width,
                                   bufs.height, fp, raw_rgb, bufs.depth.data_ptr(),
                                   raw_alpha, frgb, fdepth, falpha, _lib.ptr(keep),
                                   _lib.ptr(unet_in), unet_h, unet_c, float(unet_znear),
                                   _lib.ptr(pyramid),
                                   (bufs.flags if flags is None else flags).data_ptr(), st),
               "frame_finish")
    if ev[3] is not None:
        ev[3].record()


class ViewBuffers:
    """Pass buffers of a batch of same-size views (ls_frame_project_views):
    view v's minz / accum are rows v of one block, its raw frame rows v of
    (n_views, H, W, ...) tensors."""

    def __init__(self, width: int, height: int, n_views: int, device):
        import torch

        if not 1 <= n_views <= _lib.LS_MAX_VIEWS:
            raise ValueError(f"n_views must be in [1, {_lib.LS_MAX_VIEWS}]")
        self.width, self.height, self.n_views = int(width), int(height), int(n_views)
        npix = self.width * self.height
        k, h, w = self.n_views, self.height, self.width
        self.minz = torch.full((k, npix), _lib.INF_BITS, dtype=torch.int64, device=device)
        self.accum = torch.zeros((k, npix, 4), dtype=torch.float32, device=device)
        self.rgb = torch.empty((k, h, w, 3), dtype=torch.float32, device=device)
        self.depth = torch.empty((k, h, w), dtype=torch.float32, device=device)
        self.alpha = torch.empty((k, h, w), dtype=torch.uint8, device=device)
        self.flags = torch.zeros(k, dtype=torch.int32, device=device)


def views_cache(scene, camera: CameraModel, n_views: int, scratch=None):
    """The scratch's multi-view pass-1 -> pass-2 cache (n_views KB per warp
    tile, grown on demand), or None when disabled / the frame is too large."""
    if not USE_FRAME_CACHE or camera.width * camera.height >= 0xFFFFFFFF:
        return None
    sc = scratch or scene.scratch
    nbytes = int(_lib.load().ls_frame_views_cache_bytes(scene.struct, n_views))
    if sc.views_cache is None or sc.views_cache.numel() * 4 < nbytes:
        import torch

        sc.views_cache = torch.empty(max(nbytes // 4, 4), dtype=torch.int32,
                                     device=_lib.device())
    return sc.views_cache


def project_scene_views(scene: DeviceScene, cameras, eps_rel: float, vb: ViewBuffers,
                        cull: bool = True, filter_params=None, filtered=None, keep=None,
                        unet_in=None, unet_znear: float = 0.1, pyramid=None,
                        raw: bool = True, scratch=None) -> None:
    """Enqueue a batch of views on the current stream (no host sync): per-view
    culls, ONE multi-view pass pair over the scan (each tile read once for all
    views), then one assemble/filter per view.  ``filtered`` / ``keep`` /
    ``unet_in``: optional per-view outputs indexed by view (row v).  Each view's
    frame is bit-identical to ``project_scene`` of that view alone."""
    cameras = list(cameras)
    k = len(cameras)
    if k != vb.n_views:
        raise ValueError(f"{k} cameras for a batch of {vb.n_views} views")
    if any(c.width != vb.width or c.height != vb.height for c in cameras):
        raise ValueError("every view of a batch must have the batch's width and height")
    lib = _lib.load()
    st = _lib.stream_ptr()
    cams = (_lib.LsCamera * k)(*[_lib.make_camera(c) for c in cameras])
    bits = lst = status = cnt = None
    stride = 0
    if cull:
        vbits, lst_t, status_t, cnt_t = scene.view_buffers(scratch)
        for v, cam in enumerate(cameras):
            scene.cull_bits(extract_frustum(cam).planes, out=vbits[v])
        bits, stride = vbits.data_ptr(), int(vbits.shape[1])
        lst, status, cnt = lst_t.data_ptr(), status_t.data_ptr(), cnt_t.data_ptr()
    cache = _lib.ptr(views_cache(scene, cameras[0], k, scratch))
    _lib.check(lib.ls_frame_project_views(scene.struct, bits, stride, lst, status, cnt, cams, k,
                                          float(eps_rel), vb.minz.data_ptr(), cache,
                                          vb.accum.data_ptr(), st), "frame_project_views")
    fp = None if filter_params is None else _lib.make_filter(filter_params)
    for v in range(k):
        frgb = fdepth = falpha = None
        if filtered is not None:
            frgb, fdepth, falpha = (None if t is None else t[v] for t in filtered)
        uin = None if unet_in is None else unet_in[v]
        unet_h, unet_c = (0, 0) if uin is None else (int(uin.shape[-3]), int(uin.shape[-1]))
        _lib.check(lib.ls_frame_finish(vb.minz[v].data_ptr(), vb.accum[v].data_ptr(), vb.width,
                                       vb.height, fp, vb.rgb[v].data_ptr() if raw else None,
                                       vb.depth[v].data_ptr(),
                                       vb.alpha[v].data_ptr() if raw else None,
                                       _lib.ptr(frgb), _lib.ptr(fdepth), _lib.ptr(falpha),
                                       _lib.ptr(None if keep is None else keep[v]),
                                       _lib.ptr(uin), unet_h, unet_c, float(unet_znear),
                                       _lib.ptr(pyramid), vb.flags[v:].data_ptr(), st),
                   "frame_finish")


def project_points_views(cloud: PointCloud, grid: UniformGrid | None, cameras,
                         params: RenderParams | None = None) -> list[FrameRGBDA]:
    """``project_points`` for a batch of same-size cameras in one multi-view
    pass pair (at most LS_MAX_VIEWS per batch; longer lists run in batches).
    Returns one frame per camera, each identical to ``project_points``."""
    params = params or RenderParams()
    cameras = list(cameras)
    if not cameras:
        return []
    dev = _lib.device()
    if grid is None:
        pos, col = cloud.device_arrays()
        scene = _brute_scene(cloud, pos, col)
        cull = False
    else:
        scene = grid.scene()
        cull = True
    out = []
    for b0 in range(0, len(cameras), _lib.LS_MAX_VIEWS):
        batch = cameras[b0:b0 + _lib.LS_MAX_VIEWS]
        if not scene.n_points:
            out += [FrameRGBDA.empty(c.width, c.height) for c in batch]
            continue
        vb = ViewBuffers(batch[0].width, batch[0].height, len(batch), dev)
        with scene.lock:  # the scene's shared scratch, until the batch completed
            project_scene_views(scene, batch, params.zbuffer_epsilon_rel, vb, cull=cull)
            flags = vb.flags.cpu().numpy()
        rgb, depth, alpha = vb.rgb.cpu().numpy(), vb.depth.cpu().numpy(), vb.alpha.cpu().numpy()
        for v, cam in enumerate(batch):
            if flags[v] & 1:
                out.append(_exact_frame(cloud, grid, cam, params))
            else:
                out.append(FrameRGBDA(rgb[v], depth[v], alpha[v]))
    return out


def _exact_frame(cloud, grid, camera, params):
    """Exact (u64 x 4) path, used if a pixel may exceed the f32 accumulator bound."""
    cands = candidates(cloud, grid, camera)
    return project_candidates(cands, camera, params)


def project_points(cloud: PointCloud, grid: UniformGrid | None, camera: CameraModel,
                   params: RenderParams | None = None, backend=None,
                   workers: int | None = None) -> FrameRGBDA:
    """Render ``cloud`` through ``camera``.  With a grid the candidates come
    from frustum-culled cells; with ``grid=None`` every point is considered.
    Both yield bit-identical frames (reference render.py:164-178)."""
    params = params or RenderParams()
    if backend is not None and getattr(backend, "name", "cuda") != "cuda":
        raise ValueError(f"unknown backend {backend!r}")
    dev = _lib.device()
    if grid is None:
        pos, col = cloud.device_arrays()
        scene = _brute_scene(cloud, pos, col)
        cull = False
    else:
        scene = grid.scene()
        cull = True
    bufs = FrameBuffers(camera.width, camera.height, dev)
    if not scene.n_points:
        return FrameRGBDA.empty(camera.width, camera.height)
    with scene.lock:  # the scene's shared scratch, until the frame completed
        project_scene(scene, camera, params.zbuffer_epsilon_rel, bufs, cull=cull)
        flagged = int(bufs.flags.item()) & 1
    if flagged:
        return _exact_frame(cloud, grid, camera, params)
    return FrameRGBDA(bufs.rgb.cpu().numpy(), bufs.depth.cpu().numpy(),
                      bufs.alpha.cpu().numpy())


class _BruteScene:
    """The whole cloud, input order, no culling (grid=None reference path)."""

    def __init__(self, pos, col):
        self.n_points = int(pos.shape[0])
        s = _lib.LsScene()
        s.d_positions, s.d_colors, s.n_points = pos.data_ptr(), col.data_ptr(), self.n_points
        s.n_tiles = (self.n_points + _lib.LS_TILE_POINTS - 1) // _lib.LS_TILE_POINTS
        s.cell_size = 1.0
        self.struct = s
        self._keep = (pos, col)
        self.lock = threading.RLock()
        # no cull bits / work list: only the pass-1 -> pass-2 caches
        self.scratch = types.SimpleNamespace(frame_cache=None, views_cache=None)


def _brute_scene(cloud, pos, col):
    key = "brute:" + str(pos.device)
    sc = cloud._device.get(key)
    if sc is None:
        sc = _BruteScene(pos, col)
        cloud._device[key] = sc
    return sc
