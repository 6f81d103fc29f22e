"""How much of the frame path is launch overhead?  Times N frames of the
device path (fixed camera) enqueued eagerly vs replayed from a CUDA graph."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2502_11618_b200 import PointCloud, build_grid
from paper_2502_11618_b200.engine import FrameRenderer
from paper_2502_11618_b200.scenes import hall_cameras, multi_station_hall

unet = None
if len(sys.argv) > 1 and sys.argv[1] != "none":
    from paper_2502_11618_b200.unet import UNet

    unet = UNet.from_config(sys.argv[1], seed=7)
pos, col, _ = multi_station_hall(20_000_000)
grid = build_grid(PointCloud(pos, col), 1.0)
cam = hall_cameras(8)[0]
r = FrameRenderer(grid, 1920, 1080, unet=unet)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(5):
        r.enqueue(cam)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 50
    e0.record()
    for _ in range(n):
        r.enqueue(cam)
    e1.record()
    torch.cuda.synchronize()
    eager = e0.elapsed_time(e1) / n
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        r.enqueue(cam)
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / n
print(f"frame ({'unet ' + sys.argv[1] if unet else 'no unet'}): eager {eager * 1e3:.1f} us, "
      f"graph {graph * 1e3:.1f} us")
