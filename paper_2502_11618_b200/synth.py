"""Training-pair synthesis on the device (R:synth.py:77-115).

Both recipes of the reference are one fused frame (cull -> project ->
assemble -> depth filter, the same kernels as the render path) plus a
per-pixel selection against the ground-truth photo, all in HBM; the pair
comes back to the host in one copy:

  filtered : input = filtered depth/alpha, rgb = gt where the filtered
             alpha is set, else 0                       (R:synth.py:77-93)
  leaky    : input = raw depth/alpha, rgb = gt on filter-kept pixels, the
             projected colour on filled-but-dropped pixels, else 0
                                                         (R:synth.py:96-115)

The frame parts are bit-exact (the projection/filter parity bar), the
selection copies values, so pairs equal the reference's bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .cloud import PointCloud
from .errors import DatasetError
from .filtering import FilterParams, depth_filter
from .frame import FrameRGBDA, RenderParams
from .geometry import CameraModel
from .grid import UniformGrid
from .render import FrameBuffers, project_points, project_scene


@dataclass
class TrainingPair:
    """input: synthetic RGBDA frame; target: the untouched ground-truth RGB."""

    input: FrameRGBDA
    target: np.ndarray
    id: str


def _check_gt(gt_image: np.ndarray, camera: CameraModel) -> np.ndarray:
    gt = np.ascontiguousarray(gt_image, dtype=np.float32)
    if gt.shape != (camera.height, camera.width, 3):
        raise DatasetError(f"ground truth {gt.shape} does not match camera "
                           f"{camera.height}x{camera.width}x3")
    return gt


def _device_frames(grid: UniformGrid, camera: CameraModel, fparams: FilterParams,
                   rparams: RenderParams):
    """Raw frame, filtered frame and keep mask of one view, on the device
    (None when a pixel exceeded the fast path's accumulator bound)."""
    import torch

    dev = _lib.device()
    h, w = camera.height, camera.width
    bufs = FrameBuffers(w, h, dev)
    filtered = (torch.empty((h, w, 3), dtype=torch.float32, device=dev),
                torch.empty((h, w), dtype=torch.float32, device=dev),
                torch.empty((h, w), dtype=torch.uint8, device=dev))
    keep = torch.empty((h, w), dtype=torch.uint8, device=dev)
    n = int(_lib.load().ls_pyramid_floats(h, w, fparams.levels_n))
    if n < 0:
        raise ValueError(f"image {w}x{h} too small for {fparams.levels_n} pyramid levels")
    pyramid = torch.empty(n, dtype=torch.float32, device=dev)
    project_scene(grid.scene(), camera, rparams.zbuffer_epsilon_rel, bufs, cull=True,
                  filter_params=fparams, filtered=filtered, keep=keep, pyramid=pyramid)
    if int(bufs.flags.item()) & 1:
        return None
    return (bufs.rgb, bufs.depth, bufs.alpha), filtered


def _pair(grid, gt_image, gt_camera, fparams, rparams, pair_id, leaky, cloud):
    import torch

    gt = _check_gt(gt_image, gt_camera)
    frames = _device_frames(grid, gt_camera, fparams, rparams)
    if frames is None:  # exact fallback: the reference-shaped calls
        raw = project_points(cloud, grid, gt_camera, rparams)
        filt = depth_filter(raw, fparams)
        raw_d = tuple(torch.from_numpy(np.ascontiguousarray(a)).to(_lib.device())
                      for a in (raw.rgb, raw.depth, raw.alpha))
        filt_d = tuple(torch.from_numpy(np.ascontiguousarray(a)).to(_lib.device())
                       for a in (filt.rgb, filt.depth, filt.alpha))
    else:
        raw_d, filt_d = frames
    gt_d = torch.from_numpy(gt).to(_lib.device())
    zero = torch.zeros((), dtype=torch.float32, device=gt_d.device)
    kept = filt_d[2].bool()[:, :, None]
    if leaky:
        background = (raw_d[2].bool() & ~filt_d[2].bool())[:, :, None]
        rgb = torch.where(kept, gt_d, torch.where(background, raw_d[0], zero))
        depth, alpha = raw_d[1], raw_d[2]
    else:
        rgb = torch.where(kept, gt_d, zero)
        depth, alpha = filt_d[1], filt_d[2]
    inp = FrameRGBDA(rgb=rgb.cpu().numpy(), depth=depth.cpu().numpy(), alpha=alpha.cpu().numpy())
    return TrainingPair(input=inp, target=gt, id=pair_id)


def make_filtered_pair(cloud: PointCloud, grid: UniformGrid, gt_image: np.ndarray,
                       gt_camera: CameraModel, fparams: FilterParams, rparams: RenderParams,
                       pair_id: str = "", backend=None) -> TrainingPair:
    """Filtered recipe (R:synth.py:77-93)."""
    return _pair(grid, gt_image, gt_camera, fparams, rparams, pair_id, False, cloud)


def make_leaky_pair(cloud: PointCloud, grid: UniformGrid, gt_image: np.ndarray,
                    gt_camera: CameraModel, fparams: FilterParams, rparams: RenderParams,
                    pair_id: str = "", backend=None) -> TrainingPair:
    """Leaky recipe (R:synth.py:96-115)."""
    return _pair(grid, gt_image, gt_camera, fparams, rparams, pair_id, True, cloud)
