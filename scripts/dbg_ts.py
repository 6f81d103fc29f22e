import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2502_11618_b200 import _lib
lib = _lib.load()
dev = torch.device("cuda")
h, w, c = 1088, 1920, 32
x0 = torch.randn(1, h, w, c, device=dev).to(torch.bfloat16)
wt = (torch.randn(9, c, c, device=dev) * 0.05).to(torch.bfloat16)
sc = torch.ones(c, device=dev); sh = torch.zeros(c, device=dev)
y = torch.empty(1, h, w, c, dtype=torch.bfloat16, device=dev)
pl = torch.empty(1, h // 2, w // 2, c, dtype=torch.bfloat16, device=dev)
st = ctypes.c_int32(0)
plan = lib.ls_conv_plan_create(x0.data_ptr(), c, None, 0, 1, h, w, wt.data_ptr(), 3, c, 0,
                               sc.data_ptr(), sh.data_ptr(), 1, 0.1, y.data_ptr(), None,
                               pl.data_ptr(), None, None, 0, None, ctypes.byref(st))
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    lib.ls_conv_plan_launch(plan, s)
torch.cuda.synchronize()
buf = np.zeros(148 * 4 * 64, np.uint64)
lib.ls_conv_plan_debug_ts.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
lib.ls_conv_plan_debug_ts(plan, buf.ctypes.data, buf.size)
t = buf.reshape(148, 4, 64).astype(np.int64)
t0 = t[:, :, 0].min()
for cta in (0, 77):
    print("cta", cta)
    for ev, name in enumerate(["mma tile start", "mma tempty ok", "prod tile start", "epi tfull ok"]):
        print(f"  {name:16s}", ((t[cta, ev, :12] - t0) / 1000.0).round(2).tolist())
d = np.diff(t[:, 0, 2:60], axis=1)
print("mma per-tile period us: median", np.median(d) / 1000, "p90", np.percentile(d, 90) / 1000)
d = np.diff(t[:, 2, 2:60], axis=1)
print("prod per-tile period us: median", np.median(d) / 1000)
lag = (t[:, 3, 2:60] - t[:, 0, 2:60])
print("mma start -> epi tfull lag us: median", np.median(lag) / 1000)
if int(os.environ.get("LS_CONV_DBG", "0")) & 16:
    a = t[:, 2, 2:60]; b = t[:, 3, 2:60]; st = t[:, 1, 2:60]
    print("MMA: tempty-ok -> full(stage0)-ok us", np.median(a - st) / 1000, " full-ok -> after commit us", np.median(b - a) / 1000)
