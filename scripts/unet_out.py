"""Write the DEFAULT U-Net's output on a seeded random input (1920x1088) to a
.npy file -- used to compare kernel configurations bit for bit across
processes (the LS_CONV_* switches are read once per process)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2502_11618_b200.unet import UNet

h, w = int(os.environ.get("H", "1088")), int(os.environ.get("W", "1920"))
b = int(os.environ.get("B", "1"))  # batch (images of independent random inputs)
net = UNet.from_config("default", seed=7)
g = torch.Generator(device="cpu").manual_seed(3)
x = torch.rand((b, h, w, UNet.in_pad), generator=g).to("cuda", torch.bfloat16)
out = torch.empty((b, h, w, 3), device="cuda")
net.forward(x, out)
torch.cuda.synchronize()
np.save(sys.argv[1], out.cpu().numpy())
