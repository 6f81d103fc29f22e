"""Experiment: does the projection of frame i+1 overlap the U-Net of frame i on
the same GPU?  Times N projection+filter frames (FrameRenderer without U-Net,
stream A) and N DEFAULT U-Net forwards (stream B) separately and concurrently."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

from paper_2502_11618_b200 import PointCloud, build_grid
from paper_2502_11618_b200.engine import FrameRenderer
from paper_2502_11618_b200.scenes import hall_cameras, multi_station_hall
from paper_2502_11618_b200.unet import UNet

pts = int(os.environ.get("POINTS", "100000000"))
pos, col, _ = multi_station_hall(pts, device="cuda")
grid = build_grid(PointCloud(pos, col), 1.0)
del pos, col
cams = hall_cameras(8)
N = 20
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
with torch.cuda.stream(sa):
    r = FrameRenderer(grid, 1920, 1080, filtered_outputs=True)
net = UNet.from_config("default", seed=7)
x = torch.rand((1, 1088, 1920, UNet.in_pad), device="cuda").to(torch.bfloat16)
out = torch.empty((1, 1088, 1920, 3), device="cuda")


def proj(n):
    with torch.cuda.stream(sa):
        for i in range(n):
            r.enqueue(cams[i % 8])


def unet(n):
    with torch.cuda.stream(sb):
        for i in range(n):
            net.forward(x, out)


def timed(f):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    f()
    for s in (sa, sb):
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


proj(3); unet(3)
torch.cuda.synchronize()
tp = timed(lambda: proj(N))
tu = timed(lambda: unet(N))
tb = timed(lambda: (proj(N), unet(N)))
print(f"projection {tp / N * 1e3:.1f} us/frame, unet {tu / N * 1e3:.1f} us/frame, "
      f"sum {(tp + tu) / N * 1e3:.1f}, concurrent {tb / N * 1e3:.1f} us/frame "
      f"({tb / (tp + tu):.3f} of the sum)")
