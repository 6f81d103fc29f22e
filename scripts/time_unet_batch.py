"""Per-frame U-Net cost at 1920x1088 for batch sizes 1..8 (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2502_11618_b200.unet import UNet

net = UNet.from_config("default", seed=7)
h, w = 1088, 1920
for b in (1, 2, 4, 8):
    x = torch.rand((b, h, w, UNet.in_pad), device="cuda").to(torch.bfloat16)
    out = torch.empty((b, h, w, 3), device="cuda")
    for _ in range(3):
        net.forward(x, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n):
        net.forward(x, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    fl = net.flops(w, h) * b
    print(f"batch {b}: {ms:.3f} ms/forward, {ms / b:.3f} ms/frame, {fl / ms / 1e9:.1f} TFLOP/s")
    del x, out
    net._plans.clear()
    net._bufs.clear()
    torch.cuda.empty_cache()
