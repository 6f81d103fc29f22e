"""Time the device U-Net at 1920x1088 (CUDA events) and per-layer launches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_11618_b200.unet import UNet
net = UNet.from_config(sys.argv[1] if len(sys.argv) > 1 else "default", seed=7)
h, w = 1088, 1920
x = torch.rand((1, h, w, UNet.in_pad), device="cuda").to(torch.bfloat16)
out = torch.empty((1, h, w, 3), device="cuda")
for _ in range(3):
    net.forward(x, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = int(os.environ.get("N", "20"))
e0.record()
for _ in range(n):
    net.forward(x, out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
fl = net.flops(w, h)
print(f"unet {ms:.3f} ms/frame  {fl/ms/1e9:.1f} TFLOP/s  ({fl/1e12:.3f} TFLOP)")
