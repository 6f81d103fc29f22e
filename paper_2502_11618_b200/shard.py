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


def merge_accum(accum, root: int, group=None, async_op: bool = False):
    """Reduce SUM of the {r, g, b, count} f32 accumulators to ``root``.  Every
    field is an integer; f32 addition of integers is exact (hence order-free)
    while the sums stay below 2^24, and a sum that reached 2^24 stays >= 2^24,
    which ls_frame_finish flags.  ``async_op``: return the collective's work
    handle without making the current stream wait for it."""
    import torch.distributed as dist

    work = dist.reduce(accum, dst=root, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
    return work if async_op else accum


class DistComm:
    """The collectives of a sharded frame over torch.distributed (NCCL on the
    GPU box: NVLink/NVSwitch; gloo in the CPU tests)."""

    def __init__(self, group=None):
        self.group = group

    def all_min(self, minz_bits) -> None:
        merge_minz(minz_bits, self.group)

    def all_min_async(self, minz_bits):
        """All-reduce MIN without making the current stream wait (work handle)."""
        import torch.distributed as dist

        return dist.all_reduce(minz_bits, op=dist.ReduceOp.MIN, group=self.group, async_op=True)

    def reduce_sum(self, accum, root: int) -> None:
        merge_accum(accum, root, self.group)

    def reduce_sum_async(self, accum, root: int):
        """Enqueue the SUM reduce without making the current stream wait; the
        returned work handle's ``wait()`` orders a later stream after it."""
        return merge_accum(accum, root, self.group, async_op=True)


class ShardedRenderer:
    """FrameRenderer over one shard of the scan, merged across ranks.

    Streams: cull and passes run on the caller's stream, the collectives on
    NCCL's stream; the root's assemble/filter/U-Net run on a side stream, so
    the next frame's projection (and its collectives, in which every rank
    takes part) never waits for a U-Net.  Frames are software-pipelined by one
    stage: ``enqueue(camera_i)`` culls and runs pass 1 of frame i, starts its
    minz all-reduce asynchronously, and only then runs pass 2 of frame i-1
    (after waiting for ITS all-reduce) and starts frame i-1's accumulator
    reduce -- so each MIN all-reduce overlaps the next frame's pass 1 and each
    SUM reduce the frame after's.  ``flush()`` completes the last frame.  The
    pass buffers rotate over three sets (a set is reused only after its frame
    was consumed and reset) and the cull / work-list / pass-1 cache scratch
    over two.

    A frame is three phases around the two collectives -- ``_project_min``
    (cull, work list, pass 1), ``_accumulate`` (pass 2 against the merged
    minimum), ``_finish`` (root: assemble, filter, U-Net; others: reset) --
    so ``VirtualShards`` can drive several ranks' renderers in one process."""

    def __init__(self, grid, width: int, height: int, rank: int, world: int,
                 render_params: RenderParams | None = None,
                 filter_params: FilterParams | None = None, unet=None, group=None, comm=None):
        import torch

        from .render import FrameBuffers

        self.rank, self.world, self.group = rank, world, group
        self.comm = comm or DistComm(group)
        self.device = _lib.device()
        self.rp = render_params or RenderParams()
        self.fp = filter_params or FilterParams()
        self.width, self.height = int(width), int(height)
        full = grid.scene()
        start, end = shard_bounds(full.n_points, rank, world)
        self.shard = (start, end)
        offs = shard_cell_offsets(grid._device_field("cell_offsets", np.int64), start, end)
        self.scene = DeviceScene(full.positions[start:end], full.colors[start:end], offs,
                                 grid.origin, grid.cell_size, grid.dims)
        self.scratch = self.scene.scratch  # the shard scene is this renderer's own
        # frame i's pass 2 runs after frame i+1's pass 1: two scratch sets
        self.scratches = [self.scene.scratch, self.scene.new_scratch()]
        self.sets = [FrameBuffers(width, height, self.device) for _ in range(3)]
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
        self.aux = torch.cuda.Stream()  # non-root resets behind the async reduce
        self._consumed = [None, None, None]  # event: set k finished + reset
        self._pending = None  # (camera, set, scratch, root, all-reduce work) of the last frame
        self.frame_index = 0
        self.finished = None  # side-stream event of the last frame this rank finished

    @property
    def launches_per_frame(self) -> int:
        # cull, counter reset, work list, pass 1, pass 2 on every rank; finish +
        # filter + U-Net on the root (1/world of the frames)
        from .engine import filter_launches

        unet_n = (self.unet.launches_for(self.unet_in.shape[1], self.unet_in.shape[2])
                  if self.unet else 0)
        n = 5 + (1 + filter_launches(self.fp.levels_n) + unet_n) / self.world
        return int(round(n))

    def _next(self):
        """(pass-buffer set, root) of the next frame; waits (on the current
        stream) until the set's previous frame was consumed."""
        import torch

        k = self.frame_index % len(self.sets)
        root = self.frame_index % self.world
        self.frame_index += 1
        if self._consumed[k] is not None:
            torch.cuda.current_stream().wait_event(self._consumed[k])
        return k, root

    def _project_min(self, camera, k, si: int = 0) -> None:
        """Cull this shard's cells, build its work list, pass 1 into set k
        (scratch set si: cull bits, work list, pass-1 cache)."""
        sc, b, scr = self.scene, self.sets[k], self.scratches[si]
        bits = sc.cull_bits(extract_frustum(camera).planes, scratch=scr).data_ptr()
        tl, tc = sc.worklist(scr)
        cache = _lib.ptr(frame_cache(sc, camera, scr))
        _lib.check(_lib.load().ls_frame_pass1(sc.struct, bits, tl.data_ptr(), tc.data_ptr(),
                                              _lib.make_camera(camera), b.minz.data_ptr(), cache,
                                              _lib.stream_ptr()), "frame_pass1")

    def _accumulate(self, camera, k, si: int = 0) -> None:
        """Pass 2 of this shard against set k's (merged) minimum."""
        sc, b, scr = self.scene, self.sets[k], self.scratches[si]
        _lib.check(_lib.load().ls_frame_pass2(
            sc.struct, scr.keep_bits.data_ptr(), scr.tile_list.data_ptr(),
            scr.tile_count.data_ptr(), _lib.make_camera(camera),
            float(self.rp.zbuffer_epsilon_rel), b.minz.data_ptr(),
            _lib.ptr(frame_cache(sc, camera, scr)), b.accum.data_ptr(), _lib.stream_ptr()),
            "frame_pass2")

    def _finish(self, k, root, work=None) -> None:
        """Root: assemble + filter (+ U-Net) from set k on the side stream.
        Others: reset set k for the frame after next.  ``work``: the pending
        (asynchronous) accumulator reduce of set k -- the side stream waits
        for it, the caller's stream does not, so the reduce overlaps the next
        frame's cull and pass 1."""
        import torch

        b = self.sets[k]
        merged = torch.cuda.Event()
        merged.record(torch.cuda.current_stream())
        if self.rank != root:
            if work is None:
                b.minz.fill_(_lib.INF_BITS)
                b.accum.zero_()
                self._consumed[k] = None
                return
            # the reset runs on its own stream: the side stream may be busy
            # with a U-Net this rank is root of, which the next frames' passes
            # must not wait for
            self.aux.wait_event(merged)
            with torch.cuda.stream(self.aux):
                work.wait()  # the reduce has read this rank's accumulators
                b.minz.fill_(_lib.INF_BITS)
                b.accum.zero_()
                done = torch.cuda.Event()
                done.record(self.aux)
                self._consumed[k] = done
            return
        self.side.wait_event(merged)
        with torch.cuda.stream(self.side):
            if work is not None:
                work.wait()
            _lib.check(_lib.load().ls_frame_finish(
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
            fin = torch.cuda.Event()
            fin.record(self.side)
            self.finished = fin

    def enqueue(self, camera) -> None:
        """Enqueue one frame (this rank's share) on the current stream.  The
        frame completes on the next ``enqueue`` or on ``flush()``."""
        k, root = self._next()
        si = (self.frame_index - 1) % 2
        self._project_min(camera, k, si)
        all_min_async = getattr(self.comm, "all_min_async", None)
        if all_min_async is not None:
            work = all_min_async(self.sets[k].minz)
        else:
            self.comm.all_min(self.sets[k].minz)
            work = None
        prev, self._pending = self._pending, (camera, k, si, root, work)
        if prev is not None:
            self._complete(prev)

    def flush(self) -> None:
        """Complete the last enqueued frame (its pass 2, reduce and finish)."""
        if self._pending is not None:
            prev, self._pending = self._pending, None
            self._complete(prev)

    def _complete(self, pending) -> None:
        camera, k, si, root, work = pending
        if work is not None:
            work.wait()  # the current stream waits for the frame's MIN all-reduce
        self._accumulate(camera, k, si)
        reduce_async = getattr(self.comm, "reduce_sum_async", None)
        if reduce_async is not None:
            self._finish(k, root, reduce_async(self.sets[k].accum, root))
        else:
            self.comm.reduce_sum(self.sets[k].accum, root)
            self._finish(k, root)

    def synchronize(self) -> None:
        """Complete the pending frame and wait for this rank's side-stream work
        (the frames it is root of) and its resets."""
        self.flush()
        import torch

        torch.cuda.current_stream().synchronize()
        self.side.synchronize()
        self.aux.synchronize()

    def check_flags(self) -> None:
        self.synchronize()
        bad = any(int(b.flags.item()) for b in self.sets)
        for b in self.sets:
            b.flags.zero_()
        if bad:
            raise RuntimeError("f32 accumulator bound exceeded")


class VirtualShards:
    """All ranks of a point-sharded frame in ONE process (tests, and a world
    larger than the visible GPUs): each rank's ShardedRenderer runs its
    phases on the current stream and the two collectives are done in memory
    (MIN over the ranks' minima written back to every rank, SUM of the
    accumulators into the root's set) -- the same data flow as ``enqueue``
    over NCCL, with no rank ever waiting on another rank's kernel."""

    def __init__(self, grid, width: int, height: int, world: int, **kw):
        self.ranks = [ShardedRenderer(grid, width, height, r, world, comm=_NoComm(), **kw)
                      for r in range(world)]
        self.world = world

    def enqueue(self, camera) -> int:
        """One frame across every virtual rank; returns the root rank."""
        import torch

        ks = [r._next() for r in self.ranks]
        k, root = ks[0]
        for r in self.ranks:
            r._project_min(camera, k)
        gmin = torch.stack([r.sets[k].minz for r in self.ranks]).amin(0)
        for r in self.ranks:
            r.sets[k].minz.copy_(gmin)
            r._accumulate(camera, k)
        total = torch.stack([r.sets[k].accum for r in self.ranks]).sum(0)
        self.ranks[root].sets[k].accum.copy_(total)
        for r in self.ranks:
            r._finish(k, root)
        return root

    def synchronize(self) -> None:
        for r in self.ranks:
            r.synchronize()


class _NoComm:
    def all_min(self, t):
        raise RuntimeError("virtual ranks merge in VirtualShards.enqueue")

    reduce_sum = all_min
