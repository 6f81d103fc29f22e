"""Run a few pipeline frames for ncu captures (no timing printed here).

    python scripts/profile_frame.py [--points N] [--frames F] [--unet none|default]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2502_11618_b200 import PointCloud, build_grid, cull_cells, extract_frustum
from paper_2502_11618_b200.engine import FrameRenderer
from paper_2502_11618_b200.scenes import hall_cameras, multi_station_hall

ap = argparse.ArgumentParser()
ap.add_argument("--points", type=int, default=100_000_000)
ap.add_argument("--frames", type=int, default=3)
ap.add_argument("--unet", default="none")
a = ap.parse_args()
pos, col, _ = multi_station_hall(a.points, device="cuda")
grid = build_grid(PointCloud(pos, col), 1.0)
unet = None
if a.unet != "none":
    from paper_2502_11618_b200.unet import UNet

    unet = UNet.from_config(a.unet, seed=7, device=torch.device("cuda"))
cams = hall_cameras(8)
r = FrameRenderer(grid, 1920, 1080, unet=unet, filtered_outputs=unet is None)
for i in range(a.frames):
    r.enqueue(cams[i % len(cams)])
torch.cuda.synchronize()
r.check_flags()
cand = []
for i in range(a.frames):
    s, e = grid.cell_ranges(cull_cells(grid, extract_frustum(cams[i % len(cams)])))
    cand.append(int((e - s).sum()))
print("candidates per frame:", cand)
