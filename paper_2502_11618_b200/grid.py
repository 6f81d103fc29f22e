"""Uniform grid + frustum culling (reference grid.py:19-151), built and culled
on the GPU.

``build_grid`` runs the bit-exact f64 cell assignment, a stable device sort
and the cell-major gathers in HBM; the resulting ``UniformGrid`` keeps the
device arrays resident (the per-frame passes stream them) and materialises the
reference's host fields (cell_offsets, point_order, sorted_positions,
sorted_colors) lazily, on first access.  ``cull_cells`` is the warp-ballot
culling kernel followed by an ordered compaction; it returns the same
ascending cell ids as the reference.
"""

from __future__ import annotations

import os
import threading

import numpy as np

from . import _lib
from .cloud import PointCloud
from .errors import InvalidCloudError
from .geometry import Frustum

MAX_CELLS = 1 << 31
USE_MORTON = os.environ.get("LS_MORTON", "1") != "0"
CULL_SLACK = 1e-7  # reference grid.py:22


class DeviceScene:
    """Device-resident cell-major scan + per-scan tile index (ls_scene)."""

    def __init__(self, positions, colors, cell_offsets, origin, cell_size, dims):
        import torch

        lib = _lib.load()
        dev = positions.device
        st = _lib.stream_ptr()
        self.positions, self.colors = positions, colors
        self.n_points = int(positions.shape[0])
        n_cells = int(cell_offsets.shape[0]) - 1
        ws_bytes = lib.ls_occupied_workspace(n_cells)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        occ_cells = torch.empty(n_cells, dtype=torch.int64, device=dev)
        occ_off = torch.empty(n_cells + 1, dtype=torch.int64, device=dev)
        n_occ_d = torch.empty(1, dtype=torch.int64, device=dev)
        _lib.check(lib.ls_occupied_cells(cell_offsets.data_ptr(), n_cells, occ_cells.data_ptr(),
                                         occ_off.data_ptr(), n_occ_d.data_ptr(), ws.data_ptr(),
                                         ws_bytes, st), "occupied_cells")
        n_occ = int(n_occ_d.item())
        self.n_occ = n_occ
        self.occ_cells = occ_cells[:n_occ].clone()
        self.occ_offsets = occ_off[: n_occ + 1].clone()
        self.n_tiles = (self.n_points + _lib.LS_TILE_POINTS - 1) // _lib.LS_TILE_POINTS
        self.tile_c0 = torch.empty(max(self.n_tiles, 1), dtype=torch.int32, device=dev)
        self.tile_c1 = torch.empty(max(self.n_tiles, 1), dtype=torch.int32, device=dev)
        if n_occ > 0:
            _lib.check(lib.ls_scene_tile_index(self.occ_offsets.data_ptr(), n_occ,
                                               self.n_points, self.tile_c0.data_ptr(),
                                               self.tile_c1.data_ptr(), st), "scene_tile_index")
        self.words = max((n_occ + 31) // 32, 1)
        # per-frame scratch of one-shot synchronous calls (project_points,
        # cull_cells ...), serialised by ``lock``; renderers own their own
        # FrameScratch so concurrent frames never share cull bits, work
        # lists or pass-1 caches
        self.lock = threading.RLock()
        self.scratch = FrameScratch(self)
        s = _lib.LsScene()
        s.d_positions, s.d_colors, s.n_points = (positions.data_ptr(), colors.data_ptr(),
                                                 self.n_points)
        s.d_occ_cells, s.d_occ_offsets, s.n_occ = (self.occ_cells.data_ptr(),
                                                   self.occ_offsets.data_ptr(), n_occ)
        s.d_tile_c0, s.d_tile_c1, s.n_tiles = (self.tile_c0.data_ptr(), self.tile_c1.data_ptr(),
                                               self.n_tiles)
        s.origin[:] = [float(v) for v in origin]
        s.cell_size = float(cell_size)
        s.dims[:] = [int(v) for v in dims]
        self.struct = s

    # the default scratch's buffers (tests and one-shot calls)
    keep_bits = property(lambda self: self.scratch.keep_bits)
    tile_list = property(lambda self: self.scratch.tile_list)
    tile_count = property(lambda self: self.scratch.tile_count)

    def new_scratch(self) -> "FrameScratch":
        return FrameScratch(self)

    def cull_bits(self, planes: np.ndarray, out=None, scratch=None):
        """Warp-ballot cull of every occupied cell; returns the u32 keep bits
        (written to ``out``, else to the scratch's keep bits)."""
        bits = (scratch or self.scratch).keep_bits if out is None else out
        pl = np.ascontiguousarray(planes, np.float64)
        _lib.check(_lib.load().ls_cull(self.struct, pl.ctypes.data, CULL_SLACK, bits.data_ptr(),
                                       _lib.stream_ptr()), "cull")
        return bits

    def view_buffers(self, scratch=None):
        return (scratch or self.scratch).view_buffers()

    def worklist(self, scratch=None):
        """Frame work list of non-culled tiles from the scratch's keep bits."""
        sc = scratch or self.scratch
        _lib.check(_lib.load().ls_tile_worklist(self.struct, sc.keep_bits.data_ptr(),
                                                sc.tile_list.data_ptr(),
                                                sc.tile_count.data_ptr(), _lib.stream_ptr()),
                   "tile_worklist")
        return sc.tile_list, sc.tile_count


class FrameScratch:
    """Per-frame device scratch of one frame stream over a DeviceScene: keep
    bits, tile work list + counter, the pass-1 -> pass-2 caches and the
    multi-view cull buffers.  Frames enqueued on different streams must use
    different scratch objects (each renderer owns one)."""

    def __init__(self, scene: DeviceScene):
        import torch

        dev = scene.positions.device
        self.scene_n_tiles = scene.n_tiles
        self.words = scene.words
        self.keep_bits = torch.empty(scene.words, dtype=torch.int32, device=dev)
        self.tile_list = torch.empty(max(scene.n_tiles, 1), dtype=torch.int32, device=dev)
        self.tile_count = torch.zeros(1, dtype=torch.int32, device=dev)
        self.frame_cache = None   # lazily sized by render.frame_cache
        self.views_cache = None   # lazily sized by render.views_cache
        self._view_bufs = None

    def view_buffers(self):
        """Multi-view cull/work-list buffers (allocated on first use):
        (LS_MAX_VIEWS, words) keep bits, work list, per-entry view status, count."""
        if self._view_bufs is None:
            import torch

            dev = self.keep_bits.device
            n = max(self.scene_n_tiles, 1)
            self._view_bufs = (
                torch.empty((_lib.LS_MAX_VIEWS, self.words), dtype=torch.int32, device=dev),
                torch.empty(n, dtype=torch.int32, device=dev),
                torch.empty(n, dtype=torch.int32, device=dev),
                torch.zeros(1, dtype=torch.int32, device=dev))
        return self._view_bufs


class UniformGrid:
    """Cell partition of a cloud (reference grid.py:25-91).

    Fields match the reference's frozen dataclass; the array fields are backed
    by device tensors and copied to the host only when read.
    """

    def __init__(self, origin, cell_size, dims, cell_offsets, point_order, sorted_positions,
                 sorted_colors):
        self._origin = np.asarray(origin, np.float64)
        self._cell_size = float(cell_size)
        self._dims = np.asarray(dims, np.int64)
        self._host = {"cell_offsets": cell_offsets, "point_order": point_order,
                      "sorted_positions": sorted_positions, "sorted_colors": sorted_colors}
        self._dev = {}
        self._scene = None

    @classmethod
    def _from_device(cls, origin, cell_size, dims, d_offsets, d_order, d_pos, d_col):
        g = cls(origin, cell_size, dims, None, None, None, None)
        g._dev = {"cell_offsets": d_offsets, "point_order": d_order,
                  "sorted_positions": d_pos, "sorted_colors": d_col}
        return g

    # -- reference fields -------------------------------------------------------
    origin = property(lambda self: self._origin)
    cell_size = property(lambda self: self._cell_size)
    dims = property(lambda self: self._dims)

    def _field(self, key):
        arr = self._host.get(key)
        if arr is None:
            arr = self._dev[key].cpu().numpy()
            arr.setflags(write=False)
            self._host[key] = arr
        return arr

    cell_offsets = property(lambda self: self._field("cell_offsets"))
    point_order = property(lambda self: self._field("point_order"))
    sorted_positions = property(lambda self: self._field("sorted_positions"))
    sorted_colors = property(lambda self: self._field("sorted_colors"))

    @property
    def n_cells(self) -> int:
        return int(self._dims[0] * self._dims[1] * self._dims[2])

    # -- host-side helpers (reference grid.py:47-91) -------------------------------
    def occupied_cells(self) -> np.ndarray:
        return np.nonzero(np.diff(self.cell_offsets) > 0)[0]

    def cell_points(self, cell: int) -> np.ndarray:
        off = self.cell_offsets
        return self.point_order[off[cell]: off[cell + 1]]

    def gather_points(self, cells) -> np.ndarray:
        cells = np.asarray(cells, dtype=np.int64)
        off = self.cell_offsets
        pieces = [np.arange(off[c], off[c + 1], dtype=np.int64) for c in cells]
        flat = np.concatenate(pieces) if pieces else np.empty(0, np.int64)
        return self.point_order[flat]

    def cell_boxes(self, cells):
        cells = np.asarray(cells, dtype=np.int64)
        dy, dz = int(self._dims[1]), int(self._dims[2])
        idx = np.stack([cells // (dy * dz), (cells // dz) % dy, cells % dz], axis=1)
        lo = self._origin + idx.astype(np.float64) * self._cell_size
        return lo, lo + self._cell_size

    def cell_ranges(self, cells):
        """(starts, ends) into the sorted arrays, adjacent ranges merged."""
        cells = np.asarray(cells, dtype=np.int64)
        off = self.cell_offsets
        s, e = off[cells], off[cells + 1]
        nz = e > s
        s, e = s[nz], e[nz]
        if s.size == 0:
            return s, e
        cut = np.flatnonzero(s[1:] != e[:-1]) + 1
        first = np.concatenate(([0], cut))
        last = np.concatenate((cut - 1, [e.size - 1]))
        return s[first], e[last]

    # -- device side -------------------------------------------------------------
    def _device_field(self, key, dtype):
        import torch

        t = self._dev.get(key)
        if t is None:
            t = torch.from_numpy(np.ascontiguousarray(self._host[key], dtype)).to(_lib.device())
            self._dev[key] = t
        return t

    def scene(self) -> DeviceScene:
        """The resident device scan used by the frame passes: cell-major like
        the public fields, and inside each cell in Morton order of the point's
        in-cell position (ls_morton_order), so a warp tile is spatially compact
        (LS_MORTON=0 keeps the reference's in-cell order; frames are identical
        either way -- both frame reductions are order-free)."""
        if self._scene is None:
            import torch

            pos = self._device_field("sorted_positions", np.float32)
            col = self._device_field("sorted_colors", np.uint8)
            n = int(pos.shape[0])
            if USE_MORTON and n > 0:
                lib = _lib.load()
                dims = np.ascontiguousarray(self._dims, np.int64)
                origin = np.ascontiguousarray(self._origin, np.float64)
                ws_bytes = lib.ls_morton_order_workspace(n, int(dims.prod()))
                if ws_bytes:
                    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=pos.device)
                    order = torch.empty(n, dtype=torch.int64, device=pos.device)
                    st = _lib.stream_ptr()
                    _lib.check(lib.ls_morton_order(pos.data_ptr(), n, origin.ctypes.data,
                                                   float(self._cell_size), dims.ctypes.data,
                                                   order.data_ptr(), ws.data_ptr(), ws_bytes, st),
                               "morton_order")
                    del ws
                    mpos, mcol = torch.empty_like(pos), torch.empty_like(col)
                    _lib.check(lib.ls_gather_points(pos.data_ptr(), col.data_ptr(),
                                                    order.data_ptr(), n, mpos.data_ptr(),
                                                    mcol.data_ptr(), st), "gather_points")
                    pos, col = mpos, mcol
            self._scene = DeviceScene(pos, col, self._device_field("cell_offsets", np.int64),
                                      self._origin, self._cell_size, self._dims)
        return self._scene


def build_grid(cloud: PointCloud, cell_size: float, backend=None) -> UniformGrid:
    """Partition ``cloud`` into cubic cells of ``cell_size`` metres on the GPU
    (origin = component-wise min, dims = max(ceil(extent/size), 1); the point
    order inside a cell follows the input order)."""
    import torch

    if cloud.count == 0:
        raise InvalidCloudError("empty cloud")
    if cell_size <= 0:
        raise ValueError("cell_size must be > 0")
    # component-wise extent (min/max are exact): on the device when there is
    # one (numpy's strided axis-0 reduction takes seconds at 100M points), so
    # the argument checks below still run first on a GPU-less host
    if torch.cuda.is_available():
        pos, col = cloud.device_arrays()
        lo = torch.amin(pos, dim=0).cpu().numpy().astype(np.float64)
        hi = torch.amax(pos, dim=0).cpu().numpy().astype(np.float64)
    else:
        p = cloud.positions
        lo = np.array([p[:, i].min() for i in range(3)], np.float64)
        hi = np.array([p[:, i].max() for i in range(3)], np.float64)
    dims_f = np.maximum(np.ceil((hi - lo) / cell_size), 1.0)
    if dims_f.prod() > MAX_CELLS:
        raise InvalidCloudError(
            f"grid of {dims_f.astype(int)} cells exceeds {MAX_CELLS}; increase cell_size")
    dims = dims_f.astype(np.int64)
    n, n_cells = cloud.count, int(dims.prod())
    lib = _lib.load()
    st = _lib.stream_ptr()
    pos, col = cloud.device_arrays()
    dev = pos.device
    ids = torch.empty(n, dtype=torch.int64, device=dev)
    _lib.check(lib.ls_assign_cells(pos.data_ptr(), n, lo.ctypes.data, float(cell_size),
                                   dims.ctypes.data, ids.data_ptr(), st), "assign_cells")
    ws_bytes = lib.ls_counting_sort_workspace(n, n_cells)
    if ws_bytes == 0:
        raise InvalidCloudError(f"cloud of {n} points is too large for one grid build")
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    offsets = torch.empty(n_cells + 1, dtype=torch.int64, device=dev)
    order = torch.empty(n, dtype=torch.int64, device=dev)
    _lib.check(lib.ls_counting_sort(ids.data_ptr(), n, n_cells, offsets.data_ptr(),
                                    order.data_ptr(), ws.data_ptr(), ws_bytes, st),
               "counting_sort")
    del ws, ids
    spos = torch.empty_like(pos)
    scol = torch.empty_like(col)
    _lib.check(lib.ls_gather_points(pos.data_ptr(), col.data_ptr(), order.data_ptr(), n,
                                    spos.data_ptr(), scol.data_ptr(), st), "gather_points")
    return UniformGrid._from_device(lo, float(cell_size), dims, offsets, order, spos, scol)


def cull_cells(grid: UniformGrid, frustum: Frustum) -> np.ndarray:
    """Occupied cells whose CULL_SLACK-inflated boxes meet the frustum,
    ascending (conservative superset of every cell with a visible point)."""
    import torch

    scene = grid.scene()
    if scene.n_occ == 0:
        return np.empty(0, np.int64)
    bits = scene.cull_bits(frustum.planes, out=torch.empty_like(scene.keep_bits))
    lib = _lib.load()
    ws_bytes = lib.ls_compact_workspace(scene.n_occ)
    dev = bits.device
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    out = torch.empty(scene.n_occ, dtype=torch.int64, device=dev)
    cnt = torch.empty(1, dtype=torch.int64, device=dev)
    _lib.check(lib.ls_cull_compact(bits.data_ptr(), scene.occ_cells.data_ptr(), scene.n_occ,
                                   out.data_ptr(), cnt.data_ptr(), ws.data_ptr(), ws_bytes,
                                   _lib.stream_ptr()), "cull_compact")
    return out[: int(cnt.item())].cpu().numpy()
