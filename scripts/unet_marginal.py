"""In-chain marginal cost of each U-Net layer at 1920x1088: time the first k
plan launches (k = 1..22, PDL-chained, repeated) and difference the totals."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2502_11618_b200 import _lib
from paper_2502_11618_b200.unet import UNet

NAMES = ["e0c1", "e0c2", "e1c1", "e1c2", "e2c1", "e2c2", "e3c1", "e3c2", "b1", "b2",
         "d3up", "d3c1", "d3c2", "d2up", "d2c1", "d2c2", "d1up", "d1c1", "d1c2", "d0up",
         "d0c1", "d0c2h"]
net = UNet.from_config("default", seed=7)
h, w = 1088, 1920
x = torch.rand((1, h, w, UNet.in_pad), device="cuda").to(torch.bfloat16)
out = torch.empty((1, h, w, 3), device="cuda")
plans = net._plan(x, out)
lib = _lib.load()
st = _lib.stream_ptr()
reps = 30
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
prev = 0.0
for k in range(1, len(plans.plans) + 1):
    for _ in range(3):
        for pl in plans.plans[:k]:
            lib.ls_conv_plan_launch(pl, st)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        for pl in plans.plans[:k]:
            lib.ls_conv_plan_launch(pl, st)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e3
    name = NAMES[k - 1] if k - 1 < len(NAMES) else f"l{k}"
    print(f"{name:6s} +{t - prev:7.1f} us   cumulative {t:8.1f} us")
    prev = t
