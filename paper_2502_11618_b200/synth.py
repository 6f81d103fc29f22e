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


# ------------------------------------------------ augmentation + datasets ---
# Host-side, seeded and pure (R:synth.py:37-58, 118-253): the per-group colour
# jitter is a numpy Generator draw sequence, restated in the reference's order
# so a seed gives the reference's bytes.

_LATTICE_STEP = 32  # px between value-noise lattice nodes


@dataclass(frozen=True)
class AugmentParams:
    """Grouped brightness/contrast jitter; identity when the ranges collapse."""

    brightness_delta_range: tuple = (-0.15, 0.15)
    contrast_scale_range: tuple = (0.8, 1.25)
    group_count_range: tuple = (2, 4)
    seed: int = 0

    def __post_init__(self):
        for name in ("brightness_delta_range", "contrast_scale_range", "group_count_range"):
            lo, hi = getattr(self, name)
            if lo > hi:
                raise ValueError(f"{name} is not ordered: {(lo, hi)}")
        if self.group_count_range[0] < 1:
            raise ValueError("group count must be >= 1")
        if not 0 <= self.seed < 2**64:
            raise ValueError("seed must fit in 64 unsigned bits")


def _group_field(height: int, width: int, k: int, rng) -> np.ndarray:
    """Per-pixel group id in [0, k): a bilinear value-noise field quantised."""
    lat = rng.random((height // _LATTICE_STEP + 2, width // _LATTICE_STEP + 2))
    ys = np.arange(height) / _LATTICE_STEP
    xs = np.arange(width) / _LATTICE_STEP
    iy, ix = ys.astype(np.int64), xs.astype(np.int64)
    fy, fx = (ys - iy)[:, None], (xs - ix)[None, :]
    r0, r1 = iy[:, None], iy[:, None] + 1
    c0, c1 = ix[None, :], ix[None, :] + 1
    f = (lat[r0, c0] * (1 - fy) * (1 - fx) + lat[r0, c1] * (1 - fy) * fx
         + lat[r1, c0] * fy * (1 - fx) + lat[r1, c1] * fy * fx)
    lo, hi = f.min(), f.max()
    f = (f - lo) / (hi - lo) if hi > lo else np.zeros_like(f)
    return np.minimum((f * k).astype(np.int64), k - 1)


def augment_brightness_contrast(image: np.ndarray, alpha: np.ndarray, params: AugmentParams,
                                seed_sequence=None) -> np.ndarray:
    """out = clamp(c * (in - 0.5) + 0.5 + b, 0, 1) on filled pixels, with (c, b)
    drawn per spatial group; empty pixels are untouched.  Same seed, same bytes."""
    rng = np.random.default_rng(np.random.SeedSequence(params.seed)
                                if seed_sequence is None else seed_sequence)
    h, w = image.shape[:2]
    k = int(rng.integers(params.group_count_range[0], params.group_count_range[1] + 1))
    groups = _group_field(h, w, k, rng)
    contrast = rng.uniform(*params.contrast_scale_range, size=k)
    brightness = rng.uniform(*params.brightness_delta_range, size=k)
    shift = (0.5 - 0.5 * contrast) + brightness  # identity draw (1, 0) stays exact
    c = contrast[groups][:, :, None].astype(np.float32)
    s = shift[groups][:, :, None].astype(np.float32)
    out = np.clip(c * image + s, 0.0, 1.0)
    return np.where(alpha.astype(bool)[:, :, None], out, image).astype(np.float32)


def generate_dataset(cloud: PointCloud, scene_frames, out_dir, mode: str,
                     augment: AugmentParams, fparams: FilterParams, rparams: RenderParams,
                     backend=None, grid: UniformGrid | None = None, progress=None):
    """One training pair per (id, CameraModel, gt_image) plus a manifest
    (R:synth.py:184-253).  Pairs come from the device recipes above; the
    augmentation and file writing are host-side.  Deterministic."""
    from pathlib import Path

    from .grid import build_grid
    from .io.dataset import DatasetManifest, pair_paths, save_manifest
    from .io.frames import save_image_rgb, write_frame

    if mode not in ("filtered", "leaky"):
        raise DatasetError(f"unknown mode {mode!r}")
    frames = list(scene_frames)
    if not frames:
        raise DatasetError("scene has no frames")
    dims = {(cam.width, cam.height) for _, cam, _ in frames}
    if len(dims) != 1:
        raise DatasetError(f"frames disagree on dimensions: {sorted(dims)}")
    out = Path(out_dir)
    (out / "pairs").mkdir(parents=True, exist_ok=True)
    if grid is None:
        grid = build_grid(cloud, rparams.cell_size, backend)
    make = make_filtered_pair if mode == "filtered" else make_leaky_pair
    ids = []
    for i, (pid, cam, gt) in enumerate(frames):
        pair = make(cloud, grid, gt, cam, fparams, rparams, pair_id=str(pid), backend=backend)
        child = np.random.SeedSequence(entropy=augment.seed, spawn_key=(i,))
        rgb = augment_brightness_contrast(pair.input.rgb, pair.input.alpha, augment, child)
        paths = pair_paths(out, pair.id)
        write_frame(FrameRGBDA(rgb=rgb, depth=pair.input.depth, alpha=pair.input.alpha),
                    paths["input"])
        save_image_rgb(paths["target"], pair.target)
        ids.append(pair.id)
        if progress:
            progress(i + 1, len(frames), pair.id)
    manifest = DatasetManifest(
        mode=mode, ids=tuple(ids), seed=augment.seed,
        params={"filter": {"levels_n": fparams.levels_n,
                           "filter_strength": fparams.filter_strength,
                           "edge_threshold": fparams.edge_threshold},
                "render": {"zbuffer_epsilon_rel": rparams.zbuffer_epsilon_rel,
                           "cell_size": rparams.cell_size},
                "augment": {"brightness_delta_range": list(augment.brightness_delta_range),
                            "contrast_scale_range": list(augment.contrast_scale_range),
                            "group_count_range": list(augment.group_count_range)}})
    save_manifest(out, manifest)
    return manifest
