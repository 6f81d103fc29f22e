"""Host-independence check of scenes.multi_station_hall: digest on CPU and on
the GPU, plus a per-stage comparison of one chunk's intermediates."""
import hashlib
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2502_11618_b200.scenes import multi_station_hall

for dev in (None, "cuda"):
    t = time.time()
    p, c, _ = multi_station_hall(4_000_000, device=dev)
    h = hashlib.sha256(p.tobytes())
    h.update(c.tobytes())
    print(dev, h.hexdigest()[:16], f"{time.time() - t:.1f}s", flush=True)

gen = torch.Generator().manual_seed(1)
m = 200_000
zmin = -math.sqrt(3.0) / 2.0
cz0 = zmin + (1.0 - zmin) * torch.rand(m, generator=gen)
xy = 2.0 * torch.rand(m, 2, generator=gen) - 1.0
o0 = torch.tensor([12.3, 7.7, 1.5])
hall0 = torch.tensor([40.0, 30.0, 8.0])
res = {}
for dev in ("cpu", "cuda"):
    cz, cs, o, hall = cz0.to(dev), xy.to(dev), o0.to(dev), hall0.to(dev)
    r = {}
    r2 = cs[:, 0] * cs[:, 0] + cs[:, 1] * cs[:, 1]
    r["r2"] = r2
    r["sq"] = torch.sqrt(r2.double()).float()
    r["div"] = (cs.double() / torch.sqrt(r2.double())[:, None]).float()
    cz64 = cz.double()
    rxy = torch.sqrt(torch.clamp(1 - cz64 * cz64, min=0)).float()
    r["rxy"] = rxy
    d = torch.stack([rxy * cs[:, 0], rxy * cs[:, 1], cz], dim=1)
    r["d"] = d
    inv = (1.0 / d.double()).float()
    r["inv"] = inv
    tt = torch.where(d > 0, (hall - o) * inv, (0.0 - o) * inv)
    r["tt"] = tt
    t, surf = tt.min(dim=1)
    r["t"], r["surf"] = t, surf
    p = o + d * t[:, None]
    r["p"] = p
    res[dev] = {k: v.cpu() for k, v in r.items()}
for k in res["cpu"]:
    a, b = res["cpu"][k], res["cuda"][k]
    print(k, "equal" if torch.equal(a, b) else f"DIFF {(a != b).sum().item()}", flush=True)
