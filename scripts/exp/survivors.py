"""Pass-1 survivor statistics (experiment build): of the candidates with a
pixel, how many satisfy zc <= RN(stale_min * 1.01) at pass-1 time (could be
kept in pass 2) and how many improve the stale minimum (issue red.min)."""
import ctypes
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from paper_2502_11618_b200 import _lib

_lib.LIB_PATH = os.path.join(HERE, "liblidarsplat_stats.so")
lib = _lib.load()
lib.ls_debug_stats.argtypes = [ctypes.c_void_p, ctypes.c_int]
import torch

from paper_2502_11618_b200 import PointCloud, build_grid
from paper_2502_11618_b200.engine import FrameRenderer
from paper_2502_11618_b200.scenes import hall_cameras, multi_station_hall

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
pos, col, _ = multi_station_hall(n, device="cuda")
grid = build_grid(PointCloud(pos, col), 1.0)
r = FrameRenderer(grid, 1920, 1080)
out = (ctypes.c_ulonglong * 4)()
for i, cam in enumerate(hall_cameras(8)):
    lib.ls_debug_stats(out, 1)
    r.enqueue(cam)
    torch.cuda.synchronize()
    lib.ls_debug_stats(out, 1)
    c, s, m = out[0], out[1], out[2]
    print(f"view {i}: in-image candidates {c}, survivors {s} ({s / c:.3f}), improving {m} ({m / c:.3f})")
