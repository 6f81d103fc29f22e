"""Seeded synthetic scans for the benchmark configurations.

C1  ``uniform_box``: the reference's own 1M-point bench scene
    (pkg/benchmarks/compare_backends.py:23-33, test_acceptance.py:176-186).
C2+ ``multi_station_hall``: a 40 x 30 x 8 m hall (floor, ceiling, four walls)
    with 12 box occluders, scanned from S stations at 1.5 m; every station casts
    N/S rays uniform in solid angle over elevation [-60 deg, +90 deg] and keeps
    the first hit, so density falls off as 1/r^2 like a terrestrial scanner.
    Colour = procedural texture x per-station gain in [0.85, 1.15] (the
    brightness inconsistency between stations the paper describes).

Every random number comes from a seeded CPU torch generator and the geometry
uses only IEEE-exact operations, so every consumer (GPU path, CPU oracle,
reference arm, the golden digests) sees identical arrays on any host; the
per-chunk arithmetic can run on the GPU (``device="cuda"``) with the same
bytes.
"""

from __future__ import annotations

import math

import numpy as np

HALL = (40.0, 30.0, 8.0)


def uniform_box(n: int = 1_000_000, seed: int = 404):
    rng = np.random.default_rng(seed)
    pts = np.empty((n, 3), np.float32)
    pts[:, 0] = rng.uniform(-2, 2, n)
    pts[:, 1] = rng.uniform(-2, 2, n)
    pts[:, 2] = rng.uniform(5, 13, n)
    cols = rng.integers(0, 256, (n, 3), dtype=np.uint8)
    return pts, cols


def _boxes(gen, count=12):
    import torch

    lo = torch.empty(count, 3, dtype=torch.float64)
    hi = torch.empty(count, 3, dtype=torch.float64)
    for b in range(count):
        size = 1.0 + 3.0 * torch.rand(3, generator=gen, dtype=torch.float64)
        size[2] = 0.5 + 2.5 * torch.rand(1, generator=gen, dtype=torch.float64).item()
        cx = 2.0 + (HALL[0] - 4.0 - size[0]) * torch.rand(1, generator=gen, dtype=torch.float64)
        cy = 2.0 + (HALL[1] - 4.0 - size[1]) * torch.rand(1, generator=gen, dtype=torch.float64)
        lo[b] = torch.tensor([cx.item(), cy.item(), 0.0], dtype=torch.float64)
        hi[b] = lo[b] + size
    return lo, hi


def _inside_any(p, lo, hi, margin=0.3):
    return bool((((p >= lo - margin) & (p <= hi + margin)).all(dim=1)).any())


def _hue_table(n_surfaces: int = 15):
    """Per-surface box colour (host f64 -> f32 once): 0.3 + 0.6 * frac(hue + k/3)."""
    import torch

    t = np.empty((n_surfaces, 3), np.float32)
    for sidx in range(n_surfaces):
        h = (sidx * 0.61803) % 1.0
        for k, off in enumerate((0.0, 0.33, 0.66)):
            t[sidx, k] = np.float32(0.3) + np.float32(0.6) * np.float32((np.float32(h) + off) % 1.0)
    return torch.from_numpy(t)


def _unit_disc(gen, m: int):
    """(cos az, sin az) of m azimuths uniform on [0, 2 pi): points drawn
    uniformly in the square, kept inside the unit disc, normalised with an
    IEEE sqrt + divide -- no transcendental functions, so the scan is
    bit-identical on every host CPU (vectorised sin/cos differ across ISAs)."""
    import torch

    out = []
    have = 0
    while have < m:
        k = (m - have) * 4 // 3 + 1024
        xy = 2.0 * torch.rand(k, 2, generator=gen) - 1.0
        r2 = xy[:, 0] * xy[:, 0] + xy[:, 1] * xy[:, 1]
        ok = (r2 <= 1.0) & (r2 > 1e-6)
        xy, r2 = xy[ok], r2[ok]
        take = min(m - have, int(xy.shape[0]))
        out.append((xy[:take].double() / torch.sqrt(r2[:take].double())[:, None]).float())
        have += take
    return torch.cat(out)


def multi_station_hall(n_points: int, n_stations: int = 6, seed: int = 2025,
                       chunk: int = 2_000_000, device=None):
    """Returns (positions f32 (N,3), colors u8 (N,3), stations f64 (S,3)).

    Every random number comes from one seeded CPU torch generator (integer
    Mersenne twister); the geometry uses only IEEE-exact operations (+ - * /,
    sqrt, floor, min/max, compare), so the same seed gives the same bytes on
    any host -- and, with ``device="cuda"``, on the GPU, where the per-chunk
    arithmetic runs much faster (a 400M-point scan in seconds).  The golden
    digests in tests/golden/configs.json rely on this."""
    import torch

    dev = torch.device(device) if device is not None else torch.device("cpu")
    gen = torch.Generator().manual_seed(seed)
    lo, hi = _boxes(gen)
    stations = []
    while len(stations) < n_stations:
        p = torch.tensor([3.0 + (HALL[0] - 6.0) * torch.rand(1, generator=gen).item(),
                          3.0 + (HALL[1] - 6.0) * torch.rand(1, generator=gen).item(), 1.5],
                         dtype=torch.float64)
        if not _inside_any(p, lo, hi):
            stations.append(p)
    gains = 0.85 + 0.3 * torch.rand(n_stations, 3, generator=gen, dtype=torch.float64)
    pos = np.empty((n_points, 3), np.float32)
    col = np.empty((n_points, 3), np.uint8)
    per = [n_points // n_stations + (1 if s < n_points % n_stations else 0)
           for s in range(n_stations)]
    out = 0
    hall = torch.tensor(HALL, dtype=torch.float32, device=dev)
    lo32, hi32 = lo.float().to(dev), hi.float().to(dev)
    box_c_tab = _hue_table().to(dev)
    floor0 = torch.tensor([0.35, 0.30, 0.25], device=dev)
    floor1 = torch.tensor([0.3, 0.25, 0.2], device=dev)
    wall0 = torch.tensor([0.55, 0.5, 0.45], device=dev)
    wall1 = torch.tensor([0.1, 0.05, 0.15], device=dev)
    ceil_c = torch.tensor([0.85, 0.85, 0.8], device=dev)
    zmin = -math.sqrt(3.0) / 2.0  # sin(-60 deg)
    for s in range(n_stations):
        o = stations[s].float().to(dev)
        g = gains[s].float().to(dev)
        left = per[s]
        while left > 0:
            m = min(chunk, left)
            # all draws on the CPU generator, in a fixed order
            cz = zmin + (1.0 - zmin) * torch.rand(m, generator=gen)
            cs = _unit_disc(gen, m)
            un = torch.rand(m, 3, 2, generator=gen)
            cz, cs, un = cz.to(dev), cs.to(dev), un.to(dev)
            # sqrt and division in f64, rounded once to f32: IEEE on every
            # device (torch's f32 sqrt / reciprocal on CUDA are not)
            cz64 = cz.double()
            rxy = torch.sqrt(torch.clamp(1 - cz64 * cz64, min=0)).float()
            d = torch.stack([rxy * cs[:, 0], rxy * cs[:, 1], cz], dim=1)
            d = torch.where(d.abs() < 1e-9, torch.full_like(d, 1e-9), d)
            inv = (1.0 / d.double()).float()
            # exit of the hall box from inside
            t, surf = torch.where(d > 0, (hall - o) * inv, (0.0 - o) * inv).min(dim=1)
            t0 = (lo32[None] - o) * inv[:, None, :]          # (m, B, 3)
            t1 = (hi32[None] - o) * inv[:, None, :]
            tn = torch.minimum(t0, t1).amax(dim=2)              # (m, B)
            tf = torch.maximum(t0, t1).amin(dim=2)
            tn = torch.where((tn <= tf) & (tn > 0), tn, torch.full_like(tn, float("inf")))
            tb, bi = tn.min(dim=1)
            hit = tb < t
            t = torch.where(hit, tb, t)
            surf = torch.where(hit, bi + 3, surf)
            p = o + d * t[:, None]
            # procedural texture: floor checker, wall stripes, per-box hue
            # (integer parity / remainder: exact on every device)
            fx = torch.floor(p[:, 0] * 2.0).to(torch.int64)
            fy = torch.floor(p[:, 1] * 2.0).to(torch.int64)
            chk = ((fx + fy) & 1).to(torch.float32)[:, None]
            sz = torch.floor(p[:, 2] * 4.0).to(torch.int64)
            sxy = torch.floor((p[:, 0] + p[:, 1]) * 0.5).to(torch.int64)
            stripe = torch.remainder(sz + sxy, 3).to(torch.float32)[:, None]
            floor_c = floor0 + chk * floor1
            wall_c = wall0 + stripe * wall1
            box_c = box_c_tab[surf]
            sv = surf[:, None]
            base = torch.where(sv >= 3, box_c, torch.where(sv < 2, wall_c,
                               torch.where(p[:, 2:3] < 0.5, floor_c, ceil_c.expand(m, 3))))
            noise = 0.1 * (un[:, :, 0] + un[:, :, 1] - 1.0)  # triangular, sd 0.041
            c = torch.clamp((base + noise) * g, 0.0, 1.0) * 255.0
            pos[out:out + m] = p.cpu().numpy()
            col[out:out + m] = torch.round(c).to(torch.uint8).cpu().numpy()
            out += m
            left -= m
    return pos, col, torch.stack(stations).numpy()


def hall_cameras(count: int, width: int = 1920, height: int = 1080, f: float = 1000.0,
                 seed: int = 7):
    """Seeded poses inside the hall (eye at 1.4-1.8 m, looking across it)."""
    from .geometry import CameraModel, RigidTransform

    rng = np.random.default_rng(seed)
    cams = []
    for i in range(count):
        ang = 2 * math.pi * i / max(count, 1) + rng.uniform(-0.2, 0.2)
        eye = np.array([HALL[0] / 2 + 8 * math.cos(ang), HALL[1] / 2 + 6 * math.sin(ang),
                        rng.uniform(1.4, 1.8)])
        target = np.array([HALL[0] / 2 - 10 * math.cos(ang), HALL[1] / 2 - 8 * math.sin(ang),
                           rng.uniform(0.8, 2.0)])
        fwd = target - eye
        fwd /= np.linalg.norm(fwd)
        right = np.cross(np.array([0.0, 0.0, -1.0]), fwd)
        right /= np.linalg.norm(right)
        down = np.cross(fwd, right)
        rot = np.stack([right, down, fwd])
        pose = RigidTransform(rot, -(rot @ eye))
        cams.append(CameraModel.unchecked(f, f, width / 2.0, height / 2.0, width, height, pose,
                                          0.1, 100.0))
    return cams
