"""Bit-exact parity AT THE BENCHMARKED CONFIGURATIONS (BASELINE configs[1-3]).

tests/golden/configs.json holds sha256 digests of frames the REFERENCE itself
rendered (tests/golden/make_config_golden.py: lidarsplat native backend,
build_grid -> project_points -> depth_filter / filter_depth_image) on the
seeded multi-station hall scans.  Here the same scans (host-independent
generator; its digest is checked first) go through the product path the
bench times: FrameRenderer.enqueue, frames issued back to back on one stream
(programmatic-dependent-launch chained, no host sync between frames), raw
frame + filtered frame + keep mask + the U-Net input tensor of each frame
compared with the reference's digests (template:
/root/reference/pkg/tests/test_kernels_parity.py:121-139).

  c2  20M points, 1920x1080, 8 views     c3  100M points, 1920x1080, 8 views
  c4  400M points, 3840x2160, 1 view + the filter_strength sweep of SURVEY §8(d)
  c5  50M points, 1920x1080, 8 orbit views as one multi-view batch
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

with open(os.path.join(GOLDEN, "configs.json")) as _fh:
    CONFIGS = json.load(_fh)


@pytest.fixture(autouse=True)
def _gpu(cuda_ready):
    return cuda_ready


def digest(*tensors) -> str:
    h = hashlib.sha256()
    for t in tensors:
        a = t.cpu().numpy() if hasattr(t, "cpu") else t
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def cameras(cfg):
    from paper_2502_11618_b200 import CameraModel, RigidTransform

    fx, fy, cx, cy, zn, zf = cfg["intr"]
    return [CameraModel.unchecked(fx, fy, cx, cy, cfg["width"], cfg["height"],
                                  RigidTransform(np.array(fr["rot"], np.float64),
                                                 np.array(fr["t"], np.float64)), zn, zf)
            for fr in cfg["frames"]]


_GRIDS = {}


def config_grid(name):
    """Scan of config ``name`` (generated on the GPU, digest-checked) and its
    device grid; cached for the module."""
    import torch

    from paper_2502_11618_b200 import PointCloud, build_grid
    from paper_2502_11618_b200.scenes import multi_station_hall

    if name not in _GRIDS:
        _GRIDS.clear()
        torch.cuda.empty_cache()
        cfg = CONFIGS[name]
        pos, col, _ = multi_station_hall(cfg["points"], device="cuda")
        if digest(pos, col) != cfg["scene"]:
            # seen once over the round-2 full-suite runs and not reproduced since:
            # regenerate once -- a host-dependent generator fails both times
            torch.cuda.synchronize()
            pos, col, _ = multi_station_hall(cfg["points"], device="cuda")
        assert digest(pos, col) == cfg["scene"], "scan generator is not host-independent"
        cloud = PointCloud(pos, col)
        del pos, col
        _GRIDS[name] = build_grid(cloud, 1.0)
    return _GRIDS[name]


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_config_frames_match_reference(name):
    import torch

    from paper_2502_11618_b200.engine import FrameRenderer

    cfg = CONFIGS[name]
    grid = config_grid(name)
    cams = cameras(cfg)
    r = FrameRenderer(grid, cfg["width"], cfg["height"], keep_mask=True)
    outs = []
    for cam in cams:  # back to back on one stream; clones are stream-ordered
        r.enqueue(cam)
        outs.append([t.clone() for t in (r.bufs.rgb, r.bufs.depth, r.bufs.alpha, r.frgb,
                                         r.fdepth, r.falpha, r.keep)])
    torch.cuda.synchronize()
    r.check_flags()
    for i, (o, fr) in enumerate(zip(outs, cfg["frames"])):
        assert int(o[2].sum()) == fr["filled"], f"{name} frame {i}: filled pixels"
        assert digest(*o[:3]) == fr["raw"], f"{name} frame {i}: raw RGBDA differs"
        assert digest(*o[3:6]) == fr["filtered"], f"{name} frame {i}: filtered frame differs"
        assert digest(o[6]) == fr["keep"], f"{name} frame {i}: keep mask differs"


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_config_unet_input_matches_reference(name):
    """The bench's own configuration: U-Net attached, no f32 filtered frame
    (the assembly writes the bf16 U-Net input directly and the final filter
    step clears rejected pixels): the U-Net input of every frame equals the
    packing of the reference's filtered frame, and the U-Net runs on it."""
    import torch

    from paper_2502_11618_b200.engine import FrameRenderer
    from paper_2502_11618_b200.unet import UNet

    cfg = CONFIGS[name]
    grid = config_grid(name)
    unet = UNet.from_config("default", seed=7)
    r = FrameRenderer(grid, cfg["width"], cfg["height"], unet=unet, filtered_outputs=False)
    ins, outs = [], []
    for cam in cameras(cfg):
        r.enqueue(cam)
        ins.append(r.unet_in[0].view(torch.int16).clone())
        outs.append(r.rgb_out.clone())
    torch.cuda.synchronize()
    r.check_flags()
    for i, (x, fr) in enumerate(zip(ins, cfg["frames"])):
        assert digest(x) == fr["unet_in"], f"{name} frame {i}: U-Net input differs"
    for o in outs:
        assert bool(torch.isfinite(o).all()) and float(o.min()) >= 0 and float(o.max()) <= 1


def test_c4_sweep_matches_reference():
    """configs[3]: 400M points at 3840x2160 -- raw frame, default filter, and
    the keep mask / filtered frame of every filter_strength in the sweep."""
    import torch

    from paper_2502_11618_b200 import FilterParams
    from paper_2502_11618_b200.engine import FrameRenderer
    from paper_2502_11618_b200.filtering import depth_filter_sweep

    cfg = CONFIGS["c4"]
    grid = config_grid("c4")
    cam = cameras(cfg)[0]
    fr = cfg["frames"][0]
    r = FrameRenderer(grid, cfg["width"], cfg["height"], keep_mask=True)
    r.enqueue(cam)
    torch.cuda.synchronize()
    r.check_flags()
    assert digest(r.bufs.rgb, r.bufs.depth, r.bufs.alpha) == fr["raw"]
    assert digest(r.frgb, r.fdepth, r.falpha) == fr["filtered"]
    assert digest(r.keep) == fr["keep"]
    strengths = [s["fs"] for s in fr["sweep"]]
    res = depth_filter_sweep(r.bufs.rgb, r.bufs.depth, r.bufs.alpha, strengths,
                             FilterParams())
    for k, s in enumerate(fr["sweep"]):
        rgb, depth, alpha, keep = (t[k] for t in res)
        assert digest(keep) == s["keep"], f"fs={s['fs']}: keep mask differs"
        assert digest(rgb, depth, alpha) == s["filtered"], f"fs={s['fs']}: filtered differs"


def test_c2_default_unet_full_resolution_vs_f64_oracle():
    """The DEFAULT U-Net at the bench's own size (1920x1080 frame padded to
    1088 rows) on a real filtered hall frame (c2 view 0, whose filtered frame
    is digest-pinned above): the tcgen05 output vs the f64 restatement of
    FE:model/unet.ts (run on the GPU in float64), within the stated bound --
    max-abs <= 1.5e-2, PSNR >= 40 dB, and <= 2x the error of a plain PyTorch
    bf16 forward of the same weights (SURVEY §8(a) U-Net parity rule)."""
    import torch

    from oracle.unet_ref import forward, pack_input
    from paper_2502_11618_b200.engine import FrameRenderer
    from paper_2502_11618_b200.metrics import psnr
    from paper_2502_11618_b200.unet import UNet

    cfg = CONFIGS["c2"]
    grid = config_grid("c2")
    cam = cameras(cfg)[0]
    unet = UNet.from_config("default", seed=7)
    r = FrameRenderer(grid, cfg["width"], cfg["height"], unet=unet)
    got = r.render(cam)
    assert digest(r.frgb, r.fdepth, r.falpha) == cfg["frames"][0]["filtered"]
    x = pack_input(r.frgb.cpu().numpy(), r.fdepth.cpu().numpy(), r.falpha.cpu().numpy(), 0.1, 16)
    dev = torch.device("cuda")
    with torch.no_grad():
        ref = forward(unet.cfg, unet.params, x, device=dev)[0, :1080].cpu().numpy()
        floor = forward(unet.cfg, unet.params, torch.from_numpy(x), dtype=torch.bfloat16,
                        device=dev)[0, :1080].float().cpu().numpy()
    err = float(np.abs(got - ref).max())
    floor_err = float(np.abs(floor - ref).max())
    p = psnr(got, ref)
    print(f"DEFAULT U-Net 1920x1088 hall frame: max-abs {err:.3e} (bf16 torch floor "
          f"{floor_err:.3e}), PSNR {p:.1f} dB")
    assert got.shape == (1080, 1920, 3)
    assert err <= 1.5e-2 and p >= 40.0
    assert err <= 2 * max(floor_err, 1e-3)


def test_c5_multiview_batch_matches_reference():
    """configs[4]: 8 orbit views of the 50M-point scan as ONE multi-view batch
    (ViewBatchRenderer: one read of the culled scan for all 8 views, per-view
    assembly/filter): every view's raw and filtered frame and keep mask equal
    the reference's digests."""
    import torch

    from paper_2502_11618_b200.render import ViewBuffers, project_scene_views

    cfg = CONFIGS["c5"]
    grid = config_grid("c5")
    cams = cameras(cfg)
    w, h, k = cfg["width"], cfg["height"], len(cams)
    dev = torch.device("cuda")
    vb = ViewBuffers(w, h, k, dev)
    filt = (torch.empty((k, h, w, 3), dtype=torch.float32, device=dev),
            torch.empty((k, h, w), dtype=torch.float32, device=dev),
            torch.empty((k, h, w), dtype=torch.uint8, device=dev))
    keep = torch.empty((k, h, w), dtype=torch.uint8, device=dev)
    from paper_2502_11618_b200 import FilterParams, _lib

    fp = FilterParams()
    pyr = torch.empty(int(_lib.load().ls_pyramid_floats(h, w, fp.levels_n)),
                      dtype=torch.float32, device=dev)
    scene = grid.scene()
    with scene.lock:
        project_scene_views(scene, cams, 0.01, vb, cull=True, filter_params=fp, filtered=filt,
                            keep=keep, pyramid=pyr)
        torch.cuda.synchronize()
    assert int(vb.flags.max().item()) == 0
    for v, fr in enumerate(cfg["frames"]):
        assert digest(vb.rgb[v], vb.depth[v], vb.alpha[v]) == fr["raw"], f"view {v}: raw"
        assert digest(filt[0][v], filt[1][v], filt[2][v]) == fr["filtered"], f"view {v}: filtered"
        assert digest(keep[v]) == fr["keep"], f"view {v}: keep"
