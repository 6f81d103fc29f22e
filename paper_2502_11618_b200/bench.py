"""Per-stage frame timing (R:bench.py:1-108): ``run_bench`` / ``BenchReport``.

Same call, report fields and soft gates as the reference; the stages are
timed with CUDA events on the device instead of the host clock:

  culling_ms    : cull kernel + tile work list
  projection_ms : pass 1 + pass 2
  filter_ms     : fused assemble + depth-filter pyramid (the reference times
                  assembly inside projection and the filter separately; here
                  the two are one kernel chain, so assembly lands in filter_ms)
  total_ms      : the whole frame

Frames run back to back on one stream with this call's own buffers and
scratch (no host sync between frames), so the numbers are the pipeline's
device times, not launch latency.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .cloud import PointCloud
from .filtering import FilterParams
from .frame import RenderParams
from .grid import UniformGrid

STAGES = ("culling_ms", "projection_ms", "filter_ms", "total_ms")

# soft performance gates (ms), the reference's acceptance budgets (R:bench.py:19-21)
CULL_BUDGET_MS_PER_MPOINT = 60.0
FRAME_BUDGET_MS = 33.0


@dataclass
class BenchReport:
    points_total: int
    resolution: tuple
    frames: int
    backend: str
    stats: dict          # stage -> {"mean": ms, "p50": ms, "p95": ms}
    fps: float

    def to_dict(self) -> dict:
        """The reference's JSON shape (schemas/bench_report.schema.json)."""
        return {"points_total": self.points_total,
                "resolution": {"width": self.resolution[0], "height": self.resolution[1]},
                "frames": self.frames, "backend": self.backend, "stats": self.stats,
                "fps": self.fps}

    def gate_warnings(self) -> list:
        """Human-readable soft-gate violations (empty when within budget)."""
        out = []
        budget = CULL_BUDGET_MS_PER_MPOINT * max(self.points_total / 1e6, 1.0)
        cull = self.stats["culling_ms"]["mean"]
        if cull > budget:
            out.append(f"culling {cull:.2f} ms exceeds {budget:.0f} ms budget "
                       f"for {self.points_total} points")
        total = self.stats["total_ms"]["mean"]
        if total > FRAME_BUDGET_MS:
            out.append(f"raw+filter frame {total:.2f} ms exceeds {FRAME_BUDGET_MS:.0f} ms budget")
        return out


def _summary(samples) -> dict:
    a = np.asarray(samples, dtype=np.float64)
    return {"mean": float(a.mean()), "p50": float(np.percentile(a, 50)),
            "p95": float(np.percentile(a, 95))}


class _Target:
    """Device buffers of one resolution (pass buffers, filtered frame, pyramid)."""

    def __init__(self, width, height, fparams, dev):
        import torch

        from .render import FrameBuffers

        self.bufs = FrameBuffers(width, height, dev)
        self.out = (torch.empty((height, width, 3), dtype=torch.float32, device=dev),
                    torch.empty((height, width), dtype=torch.float32, device=dev),
                    torch.empty((height, width), dtype=torch.uint8, device=dev))
        n = int(_lib.load().ls_pyramid_floats(height, width, fparams.levels_n))
        if n < 0:
            raise ValueError(f"image {width}x{height} too small for {fparams.levels_n} "
                             "pyramid levels")
        self.pyramid = torch.empty(n, dtype=torch.float32, device=dev)


def run_bench(cloud: PointCloud, grid: UniformGrid | None, cameras, rparams: RenderParams,
              fparams: FilterParams, n_frames: int, backend=None,
              backend_name: str = "default", workers=None) -> BenchReport:
    """Render ``n_frames`` (cycling through ``cameras``: cull -> project ->
    depth filter) and time each stage (R:bench.py:70-108)."""
    import torch

    from .render import _brute_scene, project_scene

    if n_frames < 1:
        raise ValueError("need at least one frame")
    if backend is not None and getattr(backend, "name", "cuda") != "cuda":
        raise ValueError(f"unknown backend {backend!r}")
    cams = list(cameras)
    dev = _lib.device()
    if grid is None:
        pos, col = cloud.device_arrays()
        scene, cull, scratch = _brute_scene(cloud, pos, col), False, None
    else:
        scene, cull = grid.scene(), True
        scratch = scene.new_scratch()
    targets = {}
    events = []
    for i in range(n_frames):
        cam = cams[i % len(cams)]
        key = (cam.width, cam.height)
        if key not in targets:
            targets[key] = _Target(cam.width, cam.height, fparams, dev)
        t = targets[key]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record()
        if scene.n_points:
            if scratch is None:
                scene.lock.acquire()
            try:
                project_scene(scene, cam, rparams.zbuffer_epsilon_rel, t.bufs, cull=cull,
                              filter_params=fparams, filtered=t.out, pyramid=t.pyramid,
                              stage_events=ev[1:], scratch=scratch)
                if scratch is None:
                    torch.cuda.current_stream().synchronize()
            finally:
                if scratch is None:
                    scene.lock.release()
        else:
            for e in ev[1:]:
                e.record()
        events.append(ev)
    torch.cuda.current_stream().synchronize()
    samples = {s: [] for s in STAGES}
    for ev in events:
        samples["culling_ms"].append(ev[0].elapsed_time(ev[1]))
        samples["projection_ms"].append(ev[1].elapsed_time(ev[3]))
        samples["filter_ms"].append(ev[3].elapsed_time(ev[4]))
        samples["total_ms"].append(ev[0].elapsed_time(ev[4]))
    stats = {s: _summary(v) for s, v in samples.items()}
    return BenchReport(points_total=cloud.count, resolution=(cams[0].width, cams[0].height),
                       frames=n_frames, backend=backend_name, stats=stats,
                       fps=1000.0 / stats["total_ms"]["mean"])
