"""Point-sharded multi-GPU rendering.

The cell-major scan is split into contiguous, point-balanced shards, one per
rank (the reference's worker split, render.py:69-81, across GPUs instead of
threads).  Per frame:

  every rank : cull its shard (its own occupied cells), build the tile work
               list, pass 1 into a local minz
  collective : all-reduce MIN of minz -- u64 bit patterns of positive f64
               depths order like the doubles, and like int64 (< 2^63)
  every rank : pass 2 against the GLOBAL minz into local f32 accumulators
  collective : reduce SUM of the accumulators to the frame's root
               (root = frame index mod world size, so consecutive frames'
               filter + U-Net run on different GPUs)
  root       : assemble + depth filter + U-Net input + U-Net
  others     : reset their pass buffers for the next frame

Min and integer addition are order-free, so the frame is bit-identical to the
single-GPU frame for any shard count.  The collectives are torch.distributed
(NCCL over NVLink on the GPU box; gloo in the CPU tests).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .filtering import FilterParams
from .frame import RenderParams
from .geometry import extract_frustum
from .grid import DeviceScene
from .render import frame_cache


def shard_bounds(n_points: int, rank: int, world: int):
    """[start, end) of rank's contiguous, point-balanced share; interior
    boundaries fall on multiples of LS_TILE_POINTS, so every shard's arrays
    keep the 16 B (xyz) / 4 B (rgb) alignment of the vectorised frame passes
    and its warp tiles coincide with the global ones."""
    t = _lib.LS_TILE_POINTS

    def cut(r):
        if r <= 0:
            return 0
        if r >= world:
            return n_points
        return min(n_points, ((n_points * r) // world + t // 2) // t * t)

    return cut(rank), cut(rank + 1)


def shard_cell_offsets(cell_offsets, start: int, end: int):
    """Cell offsets of the sub-array [start, end) (same cell ids, clamped)."""
    return (cell_offsets.clamp(min=start, max=end) - start).contiguous()


def merge_minz(minz_bits, group=None):
    """All-reduce MIN of per-shard pass-1 minima (int64 view of the f64 bits)."""
    import torch.distributed as dist

    dist.all_reduce(minz_bits, op=dist.ReduceOp.MIN, group=group)
    return minz_bits


def merge_accum(accum, root: int, group=None):
    """Reduce SUM of the {r, g, b, count} f32 accumulators to ``root``.  Every
    field is an integer; f32 addition of integers is exact (hence order-free)
    while the sums stay below 2^24, and a sum that reached 2^24 stays >= 2^24,
    which ls_frame_finish flags."""
    import torch.distributed as dist

    dist.reduce(accum, dst=root, op=dist.ReduceOp.SUM, group=group)
    return accum


class ShardedRenderer:
    """FrameRenderer over one shard of the scan, merged across ranks.

    Streams: cull, passes and both collectives run on the caller's stream;
    the root's assemble/filter/U-Net run on a side stream, so the next frame's
    projection (and its collectives, in which every rank takes part) never
    waits for a U-Net.  The per-frame pass buffers (minz, accum) alternate
    between two sets; set k is reused only after the side stream has consumed
    (and reset) it."""

    def __init__(self, grid, width: int, height: int, rank: int, world: int,
                 render_params: RenderParams | None = None,
                 filter_params: FilterParams | None = None, unet=None, group=None):
        import torch

        from .render import FrameBuffers

        self.rank, self.world, self.group = rank, world, group
        self.device = _lib.device()
        self.rp = render_params or RenderParams()
        self.fp = filter_params or FilterParams()
        self.width, self.height = int(width), int(height)
        full = grid.scene()
        start, end = shard_bounds(full.n_points, rank, world)
        offs = shard_cell_offsets(grid._device_field("cell_offsets", np.int64), start, end)
        self.scene = DeviceScene(full.positions[start:end], full.colors[start:end], offs,
                                 grid.origin, grid.cell_size, grid.dims)
        self.scratch = self.scene.scratch  # the shard scene is this renderer's own
        self.sets = [FrameBuffers(width, height, self.device) for _ in range(2)]
        self.bufs = self.sets[0]
        h, w, dev = self.height, self.width, self.device
        self.frgb = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
        self.fdepth = torch.empty((h, w), dtype=torch.float32, device=dev)
        self.falpha = torch.empty((h, w), dtype=torch.uint8, device=dev)
        self.pyramid = torch.empty(int(_lib.load().ls_pyramid_floats(h, w, self.fp.levels_n)),
                                   dtype=torch.float32, device=dev)
        self.unet = unet
        self.unet_in = self.rgb_out = None
        if unet is not None:
            uh = (h + unet.divisor - 1) // unet.divisor * unet.divisor
            self.unet_in = torch.zeros((1, uh, w, unet.in_pad), dtype=torch.bfloat16, device=dev)
            self.rgb_out = torch.empty((1, uh, w, 3), dtype=torch.float32, device=dev)
        self.side = torch.cuda.Stream()
        self._consumed = [None, None]  # side-stream event: set k finished + reset
        self.frame_index = 0

    @property
    def launches_per_frame(self) -> int:
        # cull, counter reset, work list, pass 1, pass 2 on every rank; finish +
        # filter + U-Net on the root (1/world of the frames)
        from .engine import filter_launches

        unet_n = (self.unet.launches_for(self.unet_in.shape[1], self.unet_in.shape[2])
                  if self.unet else 0)
        n = 5 + (1 + filter_launches(self.fp.levels_n) + unet_n) / self.world
        return int(round(n))

    def enqueue(self, camera) -> None:
        """Enqueue one frame (this rank's share) on the current stream."""
        import torch

        lib = _lib.load()
        main = torch.cuda.current_stream()
        k = self.frame_index % 2
        root = self.frame_index % self.world
        self.frame_index += 1
        b = self.sets[k]
        if self._consumed[k] is not None:
            main.wait_event(self._consumed[k])
        cam = _lib.make_camera(camera)
        sc = self.scene
        st = _lib.stream_ptr()
        bits = sc.cull_bits(extract_frustum(camera).planes).data_ptr()
        tl, tc = sc.worklist()
        cache = _lib.ptr(frame_cache(sc, camera))
        _lib.check(lib.ls_frame_pass1(sc.struct, bits, tl.data_ptr(), tc.data_ptr(), cam,
                                      b.minz.data_ptr(), cache, st), "frame_pass1")
        merge_minz(b.minz, self.group)
        _lib.check(lib.ls_frame_pass2(sc.struct, bits, tl.data_ptr(), tc.data_ptr(), cam,
                                      float(self.rp.zbuffer_epsilon_rel), b.minz.data_ptr(),
                                      cache, b.accum.data_ptr(), st), "frame_pass2")
        merge_accum(b.accum, root, self.group)
        if self.rank != root:
            b.minz.fill_(_lib.INF_BITS)
            b.accum.zero_()
            self._consumed[k] = None
            return
        merged = torch.cuda.Event()
        merged.record(main)
        self.side.wait_event(merged)
        with torch.cuda.stream(self.side):
            _lib.check(lib.ls_frame_finish(
                b.minz.data_ptr(), b.accum.data_ptr(), b.width, b.height,
                _lib.make_filter(self.fp), b.rgb.data_ptr(), b.depth.data_ptr(),
                b.alpha.data_ptr(), self.frgb.data_ptr(), self.fdepth.data_ptr(),
                self.falpha.data_ptr(), None, _lib.ptr(None if self.unet_in is None
                                                       else self.unet_in[0]),
                0 if self.unet_in is None else int(self.unet_in.shape[1]),
                0 if self.unet_in is None else int(self.unet_in.shape[3]), 0.1,
                self.pyramid.data_ptr(), b.flags.data_ptr(), _lib.stream_ptr()),
                "frame_finish")
            done = torch.cuda.Event()
            done.record(self.side)
            self._consumed[k] = done
            if self.unet is not None:
                self.unet.forward(self.unet_in, self.rgb_out)

    def synchronize(self) -> None:
        """Wait for this rank's side-stream work (the frames it is root of)."""
        self.side.synchronize()

    def check_flags(self) -> None:
        self.side.synchronize()
        if any(int(b.flags.item()) for b in self.sets):
            raise RuntimeError("f32 accumulator bound exceeded")
