"""FrameRenderer: the device-resident per-frame pipeline.

What the reference's render service / CLI do per frame (serve.py:55-79,
cli.py:151-170, bench.py:85-99) -- cull, project, filter, reconstruct -- on a
scan that stays resident in HBM.  Buffers are allocated once per resolution;
a frame is a fixed sequence of launches on one stream with no host sync, so
frames pipeline back to back.  ``render`` is the public end-to-end call (host
result in pinned memory); ``enqueue`` is the device-only form used for the
kernel-level throughput number.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .filtering import FilterParams
from .frame import FrameRGBDA, RenderParams
from .render import (FrameBuffers, ViewBuffers, _exact_frame, project_scene,
                     project_scene_views)

# kernel launches per frame of the fused path: cull, work-list counter reset,
# tile work list, pass 1, pass 2, assemble+pyramid, the filter steps (+ U-Net
# layers when attached)
BASE_LAUNCHES = 6


def filter_launches(levels_n: int) -> int:
    """Launches of the filter steps: the L-1 non-final steps run as one fused
    launch when 2 <= L <= 5 (csrc/filter.cu k_filter_coarse_fused), then the
    final step; LS_FILTER_FUSED=0 restores one launch per step."""
    import os

    if 2 <= levels_n <= 5 and os.environ.get("LS_FILTER_FUSED", "1") != "0":
        return 2
    return levels_n


class FrameRenderer:
    def __init__(self, grid, width: int, height: int, render_params: RenderParams | None = None,
                 filter_params: FilterParams | None = None, unet=None,
                 filtered_outputs: bool = True, keep_mask: bool = False,
                 graph: bool = False):
        """``filtered_outputs=False`` (only with a U-Net): the f32 filtered frame
        (frgb/fdepth/falpha, 17 B/px) is not materialised -- the U-Net reads
        the packed bf16 input the same filter kernel writes.  ``keep_mask``:
        also write the filter's keep mask (u8, ``self.keep``) every frame.
        ``graph``: enqueue each frame as ONE CUDA-graph launch (captured once
        per output slot, re-targeted to every frame's camera by
        ``ls_frame_graph_set_camera``) instead of ~50 individual launches --
        for launch-bound small frames; results are identical."""
        import torch

        self.device = _lib.device()
        self.grid = grid
        self.scene = grid.scene()
        # this renderer's own cull bits / work list / pass-1 cache: renderers
        # sharing a grid (one per host thread / stream) never share scratch
        self.scratch = self.scene.new_scratch()
        self.width, self.height = int(width), int(height)
        self.rp = render_params or RenderParams()
        self.fp = filter_params or FilterParams()
        self.bufs = FrameBuffers(width, height, self.device)
        # accumulator-bound flag of each output slot (render / render_stream
        # read it back with the slot's result and reset it)
        self.slot_flags = torch.zeros(2, dtype=torch.int32, device=self.device)
        h, w, dev = self.height, self.width, self.device
        self.frgb = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
        self.fdepth = torch.empty((h, w), dtype=torch.float32, device=dev)
        self.falpha = torch.empty((h, w), dtype=torch.uint8, device=dev)
        self.keep = torch.empty((h, w), dtype=torch.uint8, device=dev) if keep_mask else None
        n = _lib.load().ls_pyramid_floats(h, w, self.fp.levels_n)
        if n < 0:
            raise ValueError(f"image {w}x{h} too small for {self.fp.levels_n} pyramid levels")
        self.pyramid = torch.empty(int(n), dtype=torch.float32, device=dev)
        self.unet = unet
        self.filtered_outputs = bool(filtered_outputs) or unet is None
        self.unet_in = None
        self.rgb_out = None
        if unet is not None:
            uh = (h + unet.divisor - 1) // unet.divisor * unet.divisor
            uw = (w + unet.divisor - 1) // unet.divisor * unet.divisor
            if uw != w:
                raise ValueError("frame width must be divisible by 2^depth for the U-Net")
            self.unet_in = torch.zeros((1, uh, w, unet.in_pad), dtype=torch.bfloat16, device=dev)
            self.rgb_out = torch.empty((1, uh, w, 3), dtype=torch.float32, device=dev)
        self._pinned = None
        # render_stream state: a second device output set (frame i's copy-out
        # overlaps frame i+1's compute), a copy stream, per-slot copy events
        self._alt = None
        self._copy_stream = None
        self._copy_done = [None, None]
        self._ring = None
        self._exact_bufs = None
        self.use_graph = bool(graph)
        self._graphs = [None, None]
        self._cap_stream = None

    @property
    def launches_per_frame(self) -> int:
        n = BASE_LAUNCHES + filter_launches(self.fp.levels_n)
        if self.unet is not None:
            n += self.unet.launches_for(self.unet_in.shape[1], self.width)
        return n

    def _outputs(self, slot: int):
        """Device result tensors of output slot 0 or 1: the U-Net RGB, or the
        filtered (rgb, depth, alpha) frame."""
        import torch

        if slot == 0:
            if self.unet is not None:
                return (self.rgb_out,)
            return (self.frgb, self.fdepth, self.falpha)
        if self._alt is None:
            self._alt = tuple(torch.empty_like(t) for t in self._outputs(0))
        return self._alt

    def enqueue(self, camera, events=None, slot: int = 0) -> None:
        """Enqueue one full frame on the current stream (no host sync).
        ``events`` (optional list of 3 CUDA events) marks project / filter /
        U-Net boundaries for per-stage timing.  ``slot`` selects the output
        buffer set (render_stream alternates two)."""
        if self.use_graph and events is None:
            self._replay(camera, slot)
            return
        self._enqueue_launches(camera, events, slot)

    def _replay(self, camera, slot: int) -> None:
        """The frame as one graph launch on the current stream."""
        import torch

        from .geometry import extract_frustum

        g = self._graphs[slot]
        if g is None:
            # warm-up frame on the capture stream (allocates the pass-1 cache
            # and the U-Net's per-stream plans / activations outside the
            # capture), then the capture itself
            if self._cap_stream is None:
                self._cap_stream = torch.cuda.Stream()
            cap = self._cap_stream
            cap.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cap):
                self._enqueue_launches(camera, None, slot)
            cap.synchronize()
            g = torch.cuda.CUDAGraph(keep_graph=True)
            with torch.cuda.graph(g, stream=cap):
                self._enqueue_launches(camera, None, slot)
            g.instantiate()
            self._graphs[slot] = g
        planes = np.ascontiguousarray(extract_frustum(camera).planes, np.float64)
        _lib.check(_lib.load().ls_frame_graph_set_camera(
            g.raw_cuda_graph(), g.raw_cuda_graph_exec(), _lib.make_camera(camera),
            planes.ctypes.data), "frame_graph_set_camera")
        g.replay()

    def _enqueue_launches(self, camera, events, slot: int) -> None:
        outs = self._outputs(slot)
        if self.unet is None:
            filtered = outs
        elif self.filtered_outputs:
            filtered = (self.frgb, self.fdepth, self.falpha)
        else:
            filtered = (None, None, None)
        project_scene(self.scene, camera, self.rp.zbuffer_epsilon_rel, self.bufs, cull=True,
                      filter_params=self.fp, filtered=filtered, keep=self.keep,
                      unet_in=None if self.unet is None else self.unet_in[0],
                      pyramid=self.pyramid, stage_events=events,
                      raw=self.unet is None or self.filtered_outputs, scratch=self.scratch,
                      flags=self.slot_flags[slot:slot + 1])
        if self.unet is not None:
            self.unet.forward(self.unet_in, outs[0])
        if events is not None:
            events[-1].record()

    def check_flags(self) -> None:
        """Raise if a frame ``enqueue``d since the last check kept more points
        in one pixel than the f32 accumulators hold exactly (> 65,793); its
        device result is then not exact.  ``render`` / ``render_stream``
        check every frame themselves and recompute such frames exactly."""
        bad = int(self.slot_flags.max().item())
        self.slot_flags.zero_()
        if bad:
            raise RuntimeError("f32 accumulator bound exceeded; use render() / "
                               "project_points() for the exact path")

    def _exact_outputs(self, camera):
        """Recompute ``camera``'s frame on the exact u64 x 4 accumulator path
        (the reference-interface twins) and return device result tensors shaped
        like ``_outputs`` (U-Net rgb, or the filtered frame).  Stream-ordered on
        the current stream after every frame enqueued before it."""
        import torch

        from .filtering import depth_filter

        raw = _exact_frame(None, self.grid, camera, self.rp)
        filt = depth_filter(raw, self.fp)
        dev = self.device
        if self.unet is None:
            return tuple(torch.from_numpy(np.ascontiguousarray(a)).to(dev)
                         for a in (filt.rgb, filt.depth, filt.alpha))
        if self.filtered_outputs:
            for dst, a in zip((self.frgb, self.fdepth, self.falpha),
                              (filt.rgb, filt.depth, filt.alpha)):
                dst.copy_(torch.from_numpy(np.ascontiguousarray(a)))
        if self._exact_bufs is None:
            self._exact_bufs = (torch.zeros_like(self.unet_in), torch.empty_like(self.rgb_out))
        x, out = self._exact_bufs
        planes = torch.from_numpy(np.ascontiguousarray(np.concatenate(
            [filt.rgb.transpose(2, 0, 1), filt.depth[None],
             filt.alpha[None].astype(np.float32)]), dtype=np.float32)).to(dev)
        _lib.check(_lib.load().ls_unet_pack_rgbda(
            planes.data_ptr(), self.height, self.width, self.unet.in_pad,
            float(self.unet.cfg.depthZNear), x.data_ptr(), _lib.stream_ptr()),
            "unet_pack_rgbda")
        self.unet.forward(x, out)
        return (out,)

    def render(self, camera):
        """Public end-to-end call: one frame, result copied to host memory.
        Returns the reconstructed RGB (H,W,3) f32 when a U-Net is attached,
        else the filtered FrameRGBDA.  The arrays are fresh copies (the
        reference returns new arrays too).  A frame in which one pixel kept
        more than 65,793 points is recomputed on the exact u64 path, so the
        result is always the reference's."""
        import torch

        if self._pinned is None:
            self._pinned = self._host_set() + (torch.zeros(1, dtype=torch.int32,
                                                           pin_memory=True),)
        *host, hflag = self._pinned
        self.slot_flags[0:1].zero_()
        self.enqueue(camera, slot=0)
        hflag.copy_(self.slot_flags[0:1], non_blocking=True)
        for dst, src in zip(host, self._outputs(0)):
            dst.copy_(src[0, : self.height] if src.dim() == 4 else src, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        if int(hflag[0]):
            self.slot_flags[0:1].zero_()
            for dst, src in zip(host, self._exact_outputs(camera)):
                dst.copy_(src[0, : self.height] if src.dim() == 4 else src)
        if self.unet is not None:
            return host[0].numpy().copy()
        return FrameRGBDA(*(t.numpy().copy() for t in host))

    def _host_set(self):
        """One set of pinned host buffers matching the device results."""
        import torch

        if self.unet is not None:
            return (torch.empty((self.height, self.width, 3), dtype=torch.float32,
                                pin_memory=True),)
        return tuple(torch.empty_like(t, device="cpu", pin_memory=True)
                     for t in (self.frgb, self.fdepth, self.falpha))

    def render_stream(self, cameras, depth: int = 2):
        """Pipelined public call: yields each camera's host result, in order.

        Frame i's device->host copy runs on a copy stream from one of two
        device output sets while frame i+1 (and i+2) compute, so a stream of
        frames costs max(compute, copy) per frame instead of their sum.  Each
        yielded array lives in a ring of ``depth + 2`` pinned host buffers and
        stays valid until the next frame has been yielded -- copy it to keep
        it longer."""
        import collections

        import torch

        comp = torch.cuda.current_stream()
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream()
        copy = self._copy_stream
        if self._ring is None or len(self._ring) != depth + 2:  # pinned once, reused
            self._ring = [self._host_set() for _ in range(depth + 2)]
            self._ring_flags = torch.zeros(depth + 2, dtype=torch.int32, pin_memory=True)
        ring, rflags = self._ring, self._ring_flags
        pending = collections.deque()

        def result(item):
            done, hs, cam = item
            done.synchronize()
            if int(rflags[hs]):  # accumulator bound hit: recompute exactly
                for dst, src in zip(ring[hs], self._exact_outputs(cam)):
                    dst.copy_(src[0, : self.height] if src.dim() == 4 else src)
            if self.unet is not None:
                return ring[hs][0].numpy()
            return FrameRGBDA(*(t.numpy() for t in ring[hs]))

        for i, cam in enumerate(cameras):
            slot, hs = i % 2, i % (depth + 2)
            if self._copy_done[slot] is not None:
                comp.wait_event(self._copy_done[slot])  # slot's previous copy-out read it
            self.enqueue(cam, slot=slot)
            ready = torch.cuda.Event()
            ready.record(comp)
            copy.wait_event(ready)
            with torch.cuda.stream(copy):
                for dst, src in zip(ring[hs], self._outputs(slot)):
                    dst.copy_(src[0, : self.height] if src.dim() == 4 else src, non_blocking=True)
                # the slot's flag goes out with its result and is reset before
                # the slot is reused (comp waits for this copy-out)
                rflags[hs:hs + 1].copy_(self.slot_flags[slot:slot + 1], non_blocking=True)
                self.slot_flags[slot:slot + 1].zero_()
                done = torch.cuda.Event()
                done.record(copy)
            self._copy_done[slot] = done
            pending.append((done, hs, cam))
            if len(pending) > depth:
                yield result(pending.popleft())
        while pending:
            yield result(pending.popleft())

    @property
    def d2h_bytes(self) -> int:
        if self.unet is not None:
            return self.height * self.width * 3 * 4
        return self.height * self.width * (3 * 4 + 4 + 1)


class ViewBatchRenderer:
    """A batch of camera views of one resident scan per call (BASELINE
    configs[4]: view-parallel reconstruction).  Each call culls every view,
    runs ONE multi-view pass pair over the scan (ls_frame_project_views: a
    tile is read once for all views), one assemble/filter per view into row v
    of a batched U-Net input, and one batched U-Net forward.  Every view's
    frame is identical to ``FrameRenderer`` rendering it alone."""

    def __init__(self, grid, width: int, height: int, n_views: int,
                 render_params: RenderParams | None = None,
                 filter_params: FilterParams | None = None, unet=None):
        import torch

        self.device = _lib.device()
        self.grid = grid
        self.scene = grid.scene()
        self.scratch = self.scene.new_scratch()
        self.width, self.height, self.n_views = int(width), int(height), int(n_views)
        self.rp = render_params or RenderParams()
        self.fp = filter_params or FilterParams()
        self.vbufs = ViewBuffers(width, height, n_views, self.device)
        h, w, k, dev = self.height, self.width, self.n_views, self.device
        n = _lib.load().ls_pyramid_floats(h, w, self.fp.levels_n)
        if n < 0:
            raise ValueError(f"image {w}x{h} too small for {self.fp.levels_n} pyramid levels")
        self.pyramid = torch.empty(int(n), dtype=torch.float32, device=dev)
        self.unet = unet
        self.frgb = self.fdepth = self.falpha = None
        self.unet_in = self.rgb_out = None
        if unet is None:
            self.frgb = torch.empty((k, h, w, 3), dtype=torch.float32, device=dev)
            self.fdepth = torch.empty((k, h, w), dtype=torch.float32, device=dev)
            self.falpha = torch.empty((k, h, w), dtype=torch.uint8, device=dev)
        else:
            uh = (h + unet.divisor - 1) // unet.divisor * unet.divisor
            if w % unet.divisor:
                raise ValueError("frame width must be divisible by 2^depth for the U-Net")
            self.unet_in = torch.zeros((k, uh, w, unet.in_pad), dtype=torch.bfloat16, device=dev)
            self.rgb_out = torch.empty((k, uh, w, 3), dtype=torch.float32, device=dev)

    @property
    def launches_per_batch(self) -> int:
        # per view: cull, assemble+pyramid, L filter steps; per batch: count
        # reset, work list, 2 passes (+ U-Net layers)
        n = self.n_views * (2 + filter_launches(self.fp.levels_n)) + 4
        if self.unet is not None:
            n += self.unet.launches_for(self.unet_in.shape[1], self.width, self.n_views)
        return n

    def enqueue(self, cameras) -> None:
        """Enqueue one batch (len(cameras) == n_views) on the current stream."""
        filtered = None if self.unet is not None else (self.frgb, self.fdepth, self.falpha)
        project_scene_views(self.scene, cameras, self.rp.zbuffer_epsilon_rel, self.vbufs,
                            cull=True, filter_params=self.fp, filtered=filtered,
                            unet_in=self.unet_in, pyramid=self.pyramid,
                            raw=self.unet is None, scratch=self.scratch)
        if self.unet is not None:
            self.unet.forward(self.unet_in, self.rgb_out)

    def check_flags(self) -> None:
        """Raise if a batch ``enqueue``d since the last check had a view whose
        pixel kept more points than the f32 accumulators hold exactly."""
        bad = int(self.vbufs.flags.max().item())
        self.vbufs.flags.zero_()
        if bad:
            raise RuntimeError("f32 accumulator bound exceeded; use render() / "
                               "project_points() for the exact path")

    def render(self, cameras):
        """Public call: one batch, results on the host.  Returns a list of
        (H,W,3) f32 U-Net outputs, or of filtered FrameRGBDA frames.  A view
        in which one pixel kept more than 65,793 points is recomputed on the
        exact u64 path (same result as rendering it with FrameRenderer)."""
        cameras = list(cameras)
        self.vbufs.flags.zero_()
        self.enqueue(cameras)
        flags = self.vbufs.flags.cpu().numpy()
        if self.unet is not None:
            out = self.rgb_out[:, : self.height].cpu().numpy()
            res = [out[v] for v in range(self.n_views)]
        else:
            rgb, depth, alpha = (t.cpu().numpy() for t in (self.frgb, self.fdepth, self.falpha))
            res = [FrameRGBDA(rgb[v], depth[v], alpha[v]) for v in range(self.n_views)]
        if flags.any():
            self.vbufs.flags.zero_()
            exact = FrameRenderer(self.grid, self.width, self.height, self.rp, self.fp,
                                  unet=self.unet, filtered_outputs=self.unet is None)
            for v in np.flatnonzero(flags):
                outs = exact._exact_outputs(cameras[v])
                if self.unet is not None:
                    res[v] = outs[0][0, : self.height].cpu().numpy()
                else:
                    res[v] = FrameRGBDA(*(t.cpu().numpy() for t in outs))
        return res
