#!/usr/bin/env python3
"""Golden digests of the BASELINE configurations, rendered BY THE REFERENCE.

Runs only in the build container (needs /root/reference): the reference
package itself (``lidarsplat_ref`` from make_golden.setup_reference, native
Cython backend, its own build_grid / project_points / depth_filter /
filter_depth_image) renders the seeded multi-station hall scans of
paper_2502_11618_b200.scenes, and tests/golden/configs.json records sha256
digests of every output array.  tests/test_gpu_configs.py renders the same
scans on the B200 and compares digests, so the bit-exactness claim covers the
configurations bench.py measures:

  c2  20M points, 1920x1080, the 8 hall_cameras      (BASELINE configs[1])
  c3  100M points, 1920x1080, the 8 hall_cameras     (configs[2], N=1 headline)
  c4  400M points, 3840x2160, f=2000, 1 view; keep mask + filtered depth for
      every filter_strength of SURVEY §8(d)'s sweep  (configs[3])
  c5  50M points, 1920x1080, 8 of the 64 orbit views (configs[4], multi-view)

Per frame: the raw RGBDA frame, the default-filtered frame, the keep mask and
the U-Net input tensor (bf16 NHWC [r,g,b,d',a,0,0,0], rows padded to 16) the
filter kernel writes -- the latter restated from FE:bridge.ts:31-53 /
weights.ts:90-95 (d' = zNear/max(d, zNear) in f64 -> f32 -> bf16).
The scan digest is recorded too: the generator is host-independent (no
transcendental functions), and the test checks it before comparing frames.

    python tests/golden/make_config_golden.py [c2 c3 c4]
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)

SWEEP = [0.0, 0.05, 0.1, 0.25, 0.5, 1.0, 1e30]
CONFIGS = {
    "c2": dict(points=20_000_000, width=1920, height=1080, f=1000.0, views=8, sweep=False),
    "c3": dict(points=100_000_000, width=1920, height=1080, f=1000.0, views=8, sweep=False),
    "c4": dict(points=400_000_000, width=3840, height=2160, f=2000.0, views=1, sweep=True),
    # configs[4]: the first 8 of the 64 orbit poses (one GPU's views)
    "c5": dict(points=50_000_000, width=1920, height=1080, f=1000.0, views=8, sweep=False,
               orbit=64),
}


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def unet_input_bytes(rgb, depth, alpha, z_near=0.1, pad=16, channels=8) -> np.ndarray:
    """bf16 NHWC U-Net input of a filtered frame, as raw u16 words."""
    import torch

    h, w = depth.shape
    dn = np.where(depth > 0, (z_near / np.maximum(depth.astype(np.float64), z_near))
                  .astype(np.float32), np.float32(0))
    x = np.zeros(((h + pad - 1) // pad * pad, w, channels), np.float32)
    x[:h, :, :3] = rgb
    x[:h, :, 3] = dn
    x[:h, :, 4] = alpha
    return torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy()


def ref_camera(R, cam):
    """The reference's CameraModel without its divisible-by-16 rule (1080 rows;
    the kernels take raw scalars)."""
    c = object.__new__(R.CameraModel)
    pose = R.RigidTransform(np.asarray(cam.world_to_camera.rotation, np.float64),
                            np.asarray(cam.world_to_camera.translation, np.float64))
    for k, v in dict(fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy, width=cam.width,
                     height=cam.height, world_to_camera=pose, z_near=cam.z_near,
                     z_far=cam.z_far).items():
        object.__setattr__(c, k, v)
    return c


def render_config(name, cfg, R, nat):
    from paper_2502_11618_b200.scenes import hall_cameras, multi_station_hall

    t0 = time.time()
    pos, col, _ = multi_station_hall(cfg["points"])
    scene = digest(pos, col)
    print(f"{name}: scan {time.time() - t0:.0f}s {scene[:16]}", flush=True)
    cams = hall_cameras(cfg.get("orbit", 8), cfg["width"], cfg["height"], f=cfg["f"])[: cfg["views"]]
    cloud = R.PointCloud(pos, col)
    del pos, col
    t0 = time.time()
    grid = R.build_grid(cloud, 1.0, backend=nat)
    print(f"{name}: reference build_grid {time.time() - t0:.0f}s", flush=True)
    frames = []
    for i, cam in enumerate(cams):
        t0 = time.time()
        rc = ref_camera(R, cam)
        fr = R.project_points(cloud, grid, rc, R.RenderParams(), backend=nat)
        fp = R.FilterParams()
        filt = R.depth_filter(fr, fp, backend=nat)
        keep = R.filter_depth_image(fr.depth, fp, backend=nat)
        cands = int(sum(e - s for s, e in zip(*grid.cell_ranges(
            R.cull_cells(grid, R.extract_frustum(rc))))))
        rec = {"rot": np.asarray(cam.world_to_camera.rotation).tolist(),
               "t": np.asarray(cam.world_to_camera.translation).tolist(),
               "candidates": cands, "filled": int(fr.alpha.sum()), "kept": int(keep.sum()),
               "raw": digest(fr.rgb, fr.depth, fr.alpha),
               "filtered": digest(filt.rgb, filt.depth, filt.alpha),
               "keep": digest(keep.astype(np.uint8)),
               "unet_in": digest(unet_input_bytes(filt.rgb, filt.depth, filt.alpha))}
        if cfg["sweep"]:
            rec["sweep"] = []
            for fs in SWEEP:
                p = R.FilterParams(filter_strength=fs)
                f2 = R.depth_filter(fr, p, backend=nat)
                k2 = R.filter_depth_image(fr.depth, p, backend=nat)
                rec["sweep"].append({"fs": fs, "keep": digest(k2.astype(np.uint8)),
                                     "filtered": digest(f2.rgb, f2.depth, f2.alpha),
                                     "kept": int(k2.sum())})
        frames.append(rec)
        print(f"{name}: frame {i} {time.time() - t0:.1f}s cands {cands} "
              f"filled {rec['filled']} kept {rec['kept']}", flush=True)
    return {"points": cfg["points"], "width": cfg["width"], "height": cfg["height"],
            "f": cfg["f"], "scene": scene, "frames": frames,
            "intr": [cams[0].fx, cams[0].fy, cams[0].cx, cams[0].cy, cams[0].z_near,
                     cams[0].z_far]}


def main():
    from make_golden import setup_reference

    R, _, _ = setup_reference()
    nat = R.get_backend("native")
    path = os.path.join(HERE, "configs.json")
    doc = {}
    if os.path.exists(path):
        with open(path) as fh:
            doc = json.load(fh)
    doc["_generator"] = ("tests/golden/make_config_golden.py (reference lidarsplat, native "
                         "backend, /root/reference/pkg)")
    for name in sys.argv[1:] or list(CONFIGS):
        doc[name] = render_config(name, CONFIGS[name], R, nat)
        with open(path, "w") as fh:
            json.dump(doc, fh, indent=1, sort_keys=True)
            fh.write("\n")


if __name__ == "__main__":
    main()
