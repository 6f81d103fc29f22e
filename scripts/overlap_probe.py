"""Prototype: frame i+1's projection/filter (low-priority stream) overlapping
frame i's U-Net (high-priority stream), double-buffered U-Net input."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2502_11618_b200 import PointCloud, build_grid
from paper_2502_11618_b200.engine import FrameRenderer
from paper_2502_11618_b200.render import project_scene
from paper_2502_11618_b200.scenes import hall_cameras, multi_station_hall
from paper_2502_11618_b200.unet import UNet

pts = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
pos, col, _ = multi_station_hall(pts)
grid = build_grid(PointCloud(pos, col), 1.0)
cams = hall_cameras(8)
net = UNet.from_config("default", seed=7)
r = FrameRenderer(grid, 1920, 1080, unet=net)
n = 40


def serial():
    for i in range(n):
        r.enqueue(cams[i % 8])


lo = torch.cuda.Stream(priority=0)
hi_pri = torch.cuda.Stream(priority=-1)
unet_in = [r.unet_in, torch.zeros_like(r.unet_in)]
outs = [r.rgb_out, torch.empty_like(r.rgb_out)]
done = [None, None]


def overlapped():
    for i in range(n):
        k = i % 2
        with torch.cuda.stream(lo):
            if done[k] is not None:
                lo.wait_event(done[k])
            project_scene(r.scene, cams[i % 8], r.rp.zbuffer_epsilon_rel, r.bufs, cull=True,
                          filter_params=r.fp, filtered=(r.frgb, r.fdepth, r.falpha),
                          unet_in=unet_in[k][0], pyramid=r.pyramid)
            ev = torch.cuda.Event()
            ev.record(lo)
        hi_pri.wait_event(ev)
        with torch.cuda.stream(hi_pri):
            net.forward(unet_in[k], outs[k])
            d = torch.cuda.Event()
            d.record(hi_pri)
        done[k] = d


for name, fn in (("serial", serial), ("overlap", overlapped), ("serial", serial),
                 ("overlap", overlapped)):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    s = torch.cuda.current_stream()
    s.wait_stream(lo)
    s.wait_stream(hi_pri)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{name}: {ms * 1e3:.1f} us/frame, {1e3 / ms:.1f} frames/s")
