"""Time single conv layers (CUDA events), e.g. the full-res U-Net layers."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_11618_b200 import _lib
lib = _lib.load()
dev = torch.device("cuda")

def layer(c0, c1, cout, h, w, pool=False, transposed=False, reps=10):
    cin = c0 + c1
    x0 = torch.randn(1, h, w, c0, device=dev).to(torch.bfloat16)
    x1 = torch.randn(1, h, w, c1, device=dev).to(torch.bfloat16) if c1 else None
    n = 4 * cout if transposed else cout
    taps = 1 if transposed else 9
    wt = (torch.randn(taps, n, cin, device=dev) * 0.05).to(torch.bfloat16)
    sc = torch.ones(n, device=dev); sh = torch.zeros(n, device=dev)
    oh, ow = (2 * h, 2 * w) if transposed else (h, w)
    y = torch.empty(1, oh, ow, cout, dtype=torch.bfloat16, device=dev)
    pl = torch.empty(1, h // 2, w // 2, cout, dtype=torch.bfloat16, device=dev) if pool else None
    import ctypes
    st = ctypes.c_int32(0)
    plan = lib.ls_conv_plan_create(x0.data_ptr(), c0, None if x1 is None else x1.data_ptr(), c1, 1, h, w,
                                   wt.data_ptr(), 1 if transposed else 3, cout, 1 if transposed else 0,
                                   sc.data_ptr(), sh.data_ptr(), 1, 0.1, y.data_ptr(), None,
                                   _lib.ptr(pl), None, None, 0, None, ctypes.byref(st))
    assert plan, st.value
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        lib.ls_conv_plan_launch(plan, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        lib.ls_conv_plan_launch(plan, s)
    e1.record(); torch.cuda.synchronize()
    lib.ls_conv_plan_destroy(plan)
    return e0.elapsed_time(e1) / reps * 1e3

H, W = 1088, 1920
if os.environ.get("LS_TIME_LAYER_NO_MAIN") != "1":
  print(os.environ.get("LS_CONV_MAX_STAGES"), os.environ.get("LS_CONV_CTAS_PER_SM"),
      "e0c2 %.1f us" % layer(32, 0, 32, H, W, pool=True),
      "d0c1 %.1f us" % layer(32, 32, 32, H, W),
      "e1c2 %.1f us" % layer(64, 0, 64, H // 2, W // 2, pool=True),
      "d0up %.1f us" % layer(64, 0, 32, H // 2, W // 2, transposed=True),
      "small-L2 e0c2 %.1f us" % layer(32, 0, 32, 272, 480, pool=True), flush=True)
