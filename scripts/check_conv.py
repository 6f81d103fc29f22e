"""Single-layer check of the tcgen05 conv kernels vs torch f32 (GPU)."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.nn.functional as F
from paper_2502_11618_b200 import _lib

torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False
lib = _lib.load()
dev = torch.device("cuda")


def conv_case(c0, c1, cout, h, w, act, pool=False, head=False, batch=1, seed=0, f32_out=True):
    """One ls_conv2d layer against torch f32.  f32_out=False: no f32 copy of the
    output is requested (so 32-channel pixel-pair layers take their staged TMA
    stores) and the raw outputs are returned instead of error figures."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    cin = c0 + c1
    x0 = torch.randn(batch, h, w, c0, generator=g).to(dev, torch.bfloat16)
    x1 = torch.randn(batch, h, w, c1, generator=g).to(dev, torch.bfloat16) if c1 else None
    wt = (torch.randn(cout, 9, cin, generator=g) * (2.0 / (9 * cin)) ** 0.5).to(dev, torch.bfloat16)
    scale = (torch.rand(cout, generator=g) + 0.5).to(dev)
    shift = (torch.randn(cout, generator=g) * 0.1).to(dev)
    y = torch.empty(batch, h, w, cout, dtype=torch.bfloat16, device=dev)
    yf = torch.empty(batch, h, w, cout, dtype=torch.float32, device=dev)
    pl = torch.zeros(batch, h // 2, w // 2, cout, dtype=torch.bfloat16, device=dev) if pool else None
    hw = (torch.randn(3, cout, generator=g) * 0.2).to(dev) if head else None
    hb = (torch.randn(3, generator=g) * 0.1).to(dev) if head else None
    ho = torch.empty(batch, h, w, 3, dtype=torch.float32, device=dev) if head else None
    wdev = wt.reshape(cout, 3, 3, cin).permute(2, 1, 0, 3).contiguous()  # [kx][ky][o][c]
    if c0 == 8 and c1 == 0:  # 8-channel input: weight rows hold the 16-wide K chunk
        wdev = torch.cat([wdev, torch.zeros_like(wdev)], -1).contiguous()
    rc = lib.ls_conv2d(x0.data_ptr(), c0, None if x1 is None else x1.data_ptr(), c1, batch, h, w,
                       wdev.data_ptr(), 3, cout, scale.data_ptr(), shift.data_ptr(), act, 0.1,
                       y.data_ptr(), yf.data_ptr() if f32_out else None, _lib.ptr(pl), _lib.ptr(hw),
                       _lib.ptr(hb), 3 if head else 0, _lib.ptr(ho), 0)
    torch.cuda.synchronize()
    assert rc == 0, rc
    if not f32_out:
        return {"y": y.cpu(), "pool": pl.cpu() if pool else None, "head": ho.cpu() if head else None}
    X = x0.float() if x1 is None else torch.cat([x0.float(), x1.float()], -1)
    W = wt.float().reshape(cout, 3, 3, cin).permute(0, 3, 1, 2)
    r = F.conv2d(X.permute(0, 3, 1, 2), W, padding=1).permute(0, 2, 3, 1)
    r = r * scale + shift
    if act == 1:
        r = torch.relu(r)
    elif act == 2:
        r = torch.where(r > 0, r, 0.1 * r)
    err = (yf - r).abs().max().item() / max(r.abs().max().item(), 1e-6)
    out = {"rel_err_f32": err, "bf16_err": (y.float() - r).abs().max().item()}
    if pool:
        rp = F.max_pool2d(y.float().permute(0, 3, 1, 2), 2).permute(0, 2, 3, 1)
        out["pool_eq"] = bool(torch.equal(rp, pl.float()))
    if head:
        rh = torch.sigmoid(r @ hw.t() + hb)
        out["head_err"] = (rh - ho).abs().max().item()
    return out


def convT_case(cin, cout, h, w, seed=0, batch=1):
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = torch.randn(batch, h, w, cin, generator=g).to(dev, torch.bfloat16)
    k = (torch.randn(2, 2, cout, cin, generator=g) * (2.0 / (4 * cin)) ** 0.5)
    wt = k.reshape(4 * cout, cin).to(dev, torch.bfloat16)
    b = torch.randn(cout, generator=g) * 0.1
    shift = b.repeat(4).to(dev)
    scale = torch.ones(4 * cout, device=dev)
    y = torch.empty(batch, 2 * h, 2 * w, cout, dtype=torch.bfloat16, device=dev)
    rc = lib.ls_conv_transpose2x2(x.data_ptr(), cin, batch, h, w, wt.data_ptr(), cout,
                                  scale.data_ptr(), shift.data_ptr(), y.data_ptr(), 0)
    torch.cuda.synchronize()
    assert rc == 0, rc
    Wt = wt.float().reshape(2, 2, cout, cin).permute(3, 2, 0, 1)  # [ci, co, dy, dx]
    r = F.conv_transpose2d(x.float().permute(0, 3, 1, 2), Wt, b.to(dev), stride=2).permute(0, 2, 3, 1)
    return {"bf16_err": (y.float() - r).abs().max().item(), "ref_max": r.abs().max().item()}


if __name__ == "__main__":
    cases = [
        dict(c0=64, c1=0, cout=64, h=32, w=64, act=0),
        dict(c0=16, c1=0, cout=32, h=64, w=128, act=1),
        dict(c0=8, c1=0, cout=32, h=64, w=128, act=1),
        dict(c0=32, c1=0, cout=32, h=64, w=128, act=1, pool=True),
        dict(c0=32, c1=32, cout=32, h=64, w=128, act=2, head=True),
        dict(c0=128, c1=128, cout=128, h=16, w=32, act=2),
        dict(c0=256, c1=0, cout=512, h=8, w=24, act=1),
        dict(c0=64, c1=0, cout=64, h=20, w=120, act=1, pool=True),
        dict(c0=64, c1=0, cout=16, h=16, w=16, act=0, batch=2),
    ]
    for c in cases:
        try:
            print(c, conv_case(**c), flush=True)
        except Exception as e:
            print(c, "FAILED", repr(e), flush=True)
    for cin, cout, h, w in [(512, 256, 8, 16), (64, 32, 32, 64), (128, 64, 16, 40)]:
        print("convT", cin, cout, h, w, convT_case(cin, cout, h, w), flush=True)
