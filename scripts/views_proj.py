"""Multi-view batched projection vs one projection per view (no U-Net):
K views of the multi-station hall scan rendered to filtered frames, either
as K single-view frames (project_scene) or as one ls_frame_project_views
batch.  Device-timed; prints one JSON line per (K, mode).

    python scripts/views_proj.py [--points 50000000] [--rounds 10]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2502_11618_b200 import FilterParams, PointCloud, RenderParams, _lib, build_grid
from paper_2502_11618_b200.render import (FrameBuffers, ViewBuffers, project_scene,
                                          project_scene_views)
from paper_2502_11618_b200.scenes import hall_cameras, multi_station_hall

ap = argparse.ArgumentParser()
ap.add_argument("--points", type=int, default=50_000_000)
ap.add_argument("--rounds", type=int, default=10)
a = ap.parse_args()

pos, col, _ = multi_station_hall(a.points)
grid = build_grid(PointCloud(pos, col), 1.0)
scene = grid.scene()
del pos, col
w, h = 1920, 1080
cams = hall_cameras(64, w, h)
dev = _lib.device()
fp, rp = FilterParams(), RenderParams()
pyr = torch.empty(int(_lib.load().ls_pyramid_floats(h, w, fp.levels_n)), dtype=torch.float32,
                  device=dev)


def timed(fn):
    fn(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(a.rounds):
        fn(r + 1)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.rounds


for k in (1, 2, 4, 8):
    vb = ViewBuffers(w, h, k, dev)
    bufs = FrameBuffers(w, h, dev)
    frgb = torch.empty((k, h, w, 3), dtype=torch.float32, device=dev)
    fdep = torch.empty((k, h, w), dtype=torch.float32, device=dev)
    falp = torch.empty((k, h, w), dtype=torch.uint8, device=dev)

    def single(r):
        for v in range(k):
            project_scene(scene, cams[(8 * r + v) % 64], rp.zbuffer_epsilon_rel, bufs, cull=True,
                          filter_params=fp, filtered=(frgb[v], fdep[v], falp[v]), pyramid=pyr)

    def batched(r):
        project_scene_views(scene, [cams[(8 * r + v) % 64] for v in range(k)],
                            rp.zbuffer_epsilon_rel, vb, cull=True, filter_params=fp,
                            filtered=(frgb, fdep, falp), pyramid=pyr)

    for mode, fn in (("single", single), ("multi-view", batched)):
        ms = timed(fn)
        print(json.dumps({"points": a.points, "views": k, "mode": mode,
                          "ms_per_batch": ms, "ms_per_view": ms / k,
                          "views_per_s": 1e3 * k / ms}), flush=True)
    if int(bufs.flags.item()) or int(vb.flags.max().item()):
        raise SystemExit("accumulator bound exceeded")
