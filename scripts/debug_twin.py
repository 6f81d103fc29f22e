import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
sys.path.insert(0, 'tests')
from conftest import golden, plain_camera
from oracle import oracle as O
from paper_2502_11618_b200._kernels import cuda as cu
from paper_2502_11618_b200 import _lib
kg = golden("kernels.npz")
p = "proj0_"
rot, t, fx, fy, cx, cy, w, h, zn, zf = O.cam_tuple(plain_camera(kg, p))
starts, ends = kg[p + "starts"], kg[p + "ends"]
lib = _lib.load()
d_pos = torch.from_numpy(kg[p+"pos"]).cuda()
d_s = torch.from_numpy(starts).cuda(); d_e = torch.from_numpy(ends).cuda()
ws = torch.full((5,), -7, dtype=torch.int64, device='cuda')
minz = torch.full((h*w,), float('inf'), dtype=torch.float64, device='cuda')
pix = torch.full((4000,), -5, dtype=torch.int64, device='cuda')
z = torch.full((4000,), -5.0, dtype=torch.float64, device='cuda')
cam = cu._cam(rot, t, fx, fy, cx, cy, w, h, zn, zf)
rc = lib.ls_project_min_depth(d_pos.data_ptr(), d_s.data_ptr(), d_e.data_ptr(), 4, cam, minz.data_ptr(), pix.data_ptr(), z.data_ptr(), ws.data_ptr(), 40, 0)
torch.cuda.synchronize()
print("rc", rc, "prefix", ws.tolist(), "pix", pix[:5].tolist(), "z", z[:5].tolist())
print(cam.width, cam.height, cam.z_near, cam.z_far, list(cam.rot))
