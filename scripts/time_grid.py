"""Per-step timing of the per-scan grid build (build_grid + the Morton-ordered
device scene) at a given scan size."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2502_11618_b200 import PointCloud, _lib, build_grid
from paper_2502_11618_b200.scenes import multi_station_hall

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
pos, col, _ = multi_station_hall(n, device="cuda")
c = PointCloud(pos, col)
d_pos, d_col = c.device_arrays()
torch.cuda.synchronize()
lib = _lib.load()


def timed(name, fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print(f"{name:28s} {(time.perf_counter() - t) * 1e3:8.1f} ms", flush=True)
    return r


lo = timed("host min/max", lambda: (c.positions.min(axis=0), c.positions.max(axis=0)))[0]
origin = lo.astype(np.float64)
dims = np.array([40, 30, 8], np.int64)
ids = torch.empty(n, dtype=torch.int64, device="cuda")
timed("assign_cells", lambda: lib.ls_assign_cells(d_pos.data_ptr(), n, origin.ctypes.data, 1.0,
                                                  dims.ctypes.data, ids.data_ptr(),
                                                  _lib.stream_ptr()))
ws_b = lib.ls_counting_sort_workspace(n, int(dims.prod()))
ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
off = torch.empty(int(dims.prod()) + 1, dtype=torch.int64, device="cuda")
order = torch.empty(n, dtype=torch.int64, device="cuda")
timed("counting_sort (radix)", lambda: lib.ls_counting_sort(ids.data_ptr(), n, int(dims.prod()),
                                                             off.data_ptr(), order.data_ptr(),
                                                             ws.data_ptr(), ws_b,
                                                             _lib.stream_ptr()))
del ws
ws_b = lib.ls_morton_order_workspace(n, int(dims.prod()))
ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
timed("morton_order (radix)", lambda: lib.ls_morton_order(d_pos.data_ptr(), n, origin.ctypes.data,
                                                           1.0, dims.ctypes.data, order.data_ptr(),
                                                           ws.data_ptr(), ws_b, _lib.stream_ptr()))
del ws
sp, sc = torch.empty_like(d_pos), torch.empty_like(d_col)
timed("gather_points", lambda: lib.ls_gather_points(d_pos.data_ptr(), d_col.data_ptr(),
                                                     order.data_ptr(), n, sp.data_ptr(),
                                                     sc.data_ptr(), _lib.stream_ptr()))
g = timed("build_grid (whole)", lambda: build_grid(c, 1.0))
timed("grid.scene() (Morton scene)", lambda: g.scene())
