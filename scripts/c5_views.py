"""BASELINE configs[4] per GPU: a batch of camera views of a 50M-point scan,
each projected + filtered into one slot of a batched U-Net input, then one
batched U-Net forward (view-parallel reconstruction; 8 GPUs each take 8 of
the 64 views as independent replicas).  Prints one JSON line per batch size.

    python scripts/c5_views.py [--points 50000000] [--views 8]
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
from paper_2502_11618_b200.unet import UNet

ap = argparse.ArgumentParser()
ap.add_argument("--points", type=int, default=50_000_000)
ap.add_argument("--views", type=int, default=8)
ap.add_argument("--rounds", type=int, default=5)
ap.add_argument("--batched-projection", type=int, default=1,
                help="1: one multi-view pass pair per U-Net batch (ls_frame_project_views)")
a = ap.parse_args()

pos, col, _ = multi_station_hall(a.points, device="cuda")
grid = build_grid(PointCloud(pos, col), 1.0)
scene = grid.scene()
del pos, col
w, h = 1920, 1080
cams = hall_cameras(64, w, h)
dev = _lib.device()
net = UNet.from_config("default", seed=7)
uh = (h + net.divisor - 1) // net.divisor * net.divisor
fp, rp = FilterParams(), RenderParams()
bufs = FrameBuffers(w, h, dev)
pyr = torch.empty(int(_lib.load().ls_pyramid_floats(h, w, fp.levels_n)), dtype=torch.float32,
                  device=dev)
for batch in (1, 4, 8):
    x = torch.zeros((batch, uh, w, net.in_pad), dtype=torch.bfloat16, device=dev)
    out = torch.empty((batch, uh, w, 3), dtype=torch.float32, device=dev)

    vb = ViewBuffers(w, h, batch, dev) if a.batched_projection else None

    def views(start):
        for v0 in range(0, a.views, batch):
            if vb is not None:
                project_scene_views(scene, [cams[(start + v0 + b) % 64] for b in range(batch)],
                                    rp.zbuffer_epsilon_rel, vb, cull=True, filter_params=fp,
                                    filtered=None, unet_in=x, pyramid=pyr)
                net.forward(x, out)
                continue
            for b in range(batch):
                project_scene(scene, cams[(start + v0 + b) % 64], rp.zbuffer_epsilon_rel, bufs,
                              cull=True, filter_params=fp, filtered=(None, None, None),
                              unet_in=x[b], pyramid=pyr)
            net.forward(x, out)

    views(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(a.rounds):
        views(8 * r)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (a.rounds * a.views)
    if int(bufs.flags.item()) or (vb is not None and int(vb.flags.max().item())):
        raise SystemExit("accumulator bound exceeded")
    print(json.dumps({"config": f"{a.points / 1e6:g}M points, 1920x1080, {a.views} views per GPU, "
                                f"U-Net batch {batch}" + (", multi-view projection"
                                                          if vb is not None else ""),
                      "views_per_s_per_gpu": 1e3 / ms, "ms_per_view": ms,
                      "note": "device-timed; 64 views over 8 GPUs = 8 independent replicas"}),
          flush=True)
    del x, out
    net._plans.clear()
    net._bufs.clear()
