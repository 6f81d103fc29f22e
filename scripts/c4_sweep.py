"""BASELINE configs[3]: a large scan at 3840x2160 -- grid culling + projection +
a depth-filter sweep over filter_strength (no U-Net).  Per frame: one
projection (cull, both passes, assemble), then the batched sweep
(filtering.depth_filter_sweep: pyramid once, all strengths in two launches) on
the device-resident raw frame -- or, with --batched 0, ls_depth_filter_frame
once per strength.  Strengths = SURVEY §8(d)'s list.  Prints one JSON line.

    python scripts/c4_sweep.py [--points 400000000] [--frames 10] [--batched 1]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2502_11618_b200 import FilterParams, PointCloud, RenderParams, _lib, build_grid
from paper_2502_11618_b200.filtering import depth_filter_sweep
from paper_2502_11618_b200.render import FrameBuffers, project_scene
from paper_2502_11618_b200.scenes import hall_cameras, multi_station_hall

ap = argparse.ArgumentParser()
ap.add_argument("--points", type=int, default=400_000_000)
ap.add_argument("--width", type=int, default=3840)
ap.add_argument("--height", type=int, default=2160)
ap.add_argument("--batched", type=int, default=1)
ap.add_argument("--outputs", type=int, default=1, help="0: keep masks only (batched sweep)")
ap.add_argument("--frames", type=int, default=10)
a = ap.parse_args()

t0 = time.time()
pos, col, _ = multi_station_hall(a.points, device="cuda")
t_gen = time.time() - t0
t0 = time.time()
grid = build_grid(PointCloud(pos, col), 1.0)
scene = grid.scene()
torch.cuda.synchronize()
t_grid = time.time() - t0
del pos, col
cams = hall_cameras(8, a.width, a.height, f=2000.0 * a.width / 3840)
dev = _lib.device()
h, w = a.height, a.width
bufs = FrameBuffers(w, h, dev)
strengths = [0.0, 0.05, 0.1, 0.25, 0.5, 1.0, 1e30]
fparams = [FilterParams(filter_strength=min(float(s), 1e30)) for s in strengths]
pyr = torch.empty(int(_lib.load().ls_pyramid_floats(h, w, fparams[0].levels_n)),
                  dtype=torch.float32, device=dev)
frgb = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
fdepth = torch.empty((h, w), dtype=torch.float32, device=dev)
falpha = torch.empty((h, w), dtype=torch.uint8, device=dev)
keeps = torch.empty((len(strengths), h, w), dtype=torch.uint8, device=dev)
work = None
lib = _lib.load()
rp = RenderParams()


def frame(cam):
    global work
    project_scene(scene, cam, rp.zbuffer_epsilon_rel, bufs, cull=True)
    if a.batched:
        return depth_filter_sweep(bufs.rgb, bufs.depth, bufs.alpha, strengths, fparams[0],
                                  outputs=bool(a.outputs), work=work)
    for i, fp in enumerate(fparams):
        _lib.check(lib.ls_depth_filter_frame(
            bufs.rgb.data_ptr(), bufs.depth.data_ptr(), bufs.alpha.data_ptr(), h, w,
            _lib.make_filter(fp), frgb.data_ptr(), fdepth.data_ptr(), falpha.data_ptr(),
            keeps[i].data_ptr(), pyr.data_ptr(), _lib.stream_ptr()), "depth_filter_frame")
    return None, None, None, keeps


for i in range(3):
    res = frame(cams[i % 8])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(a.frames):
    res = frame(cams[i % 8])
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.frames
# projection alone for the split
e0.record()
for i in range(a.frames):
    project_scene(scene, cams[i % 8], rp.zbuffer_epsilon_rel, bufs, cull=True)
e1.record()
torch.cuda.synchronize()
ms_proj = e0.elapsed_time(e1) / a.frames
if int(bufs.flags.item()):
    raise SystemExit("accumulator bound exceeded")
print(json.dumps({
    "config": f"{a.points / 1e6:g}M points, {w}x{h}, cull+project+filter sweep x{len(strengths)}",
    "frames_per_s": 1e3 / ms, "ms_per_frame": ms, "projection_ms": ms_proj,
    "filter_ms_per_strength": (ms - ms_proj) / len(strengths),
    "filter_sweep": ("batched (depth_filter_sweep)" if a.batched else "one filter per strength")
                    + ("" if a.outputs or not a.batched else ", keep masks only"),
    "filter_strengths": [float(s) for s in strengths],
    "kept_pixels_per_strength": [int(k.sum()) for k in res[3].to(torch.int64)],
    "setup_s": {"generate": round(t_gen, 1), "grid_build": round(t_grid, 1)},
    "note": "device-timed (CUDA events); synthetic seeded multi-station hall"}))
