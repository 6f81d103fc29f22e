#!/usr/bin/env python3
"""Per-frame rendering pipeline throughput on B200 (BASELINE.json metric:
"frames/sec at 1920x1080 for N-M-point scan (1/2/4/8 B200); Gpoints/s projected").

Workload (default) = BASELINE configs[1]: synthetic 20M-point multi-station
scan (paper_2502_11618_b200.scenes.multi_station_hall, seeded), 1920x1080,
full pipeline per frame: grid-cell culling -> two-pass projection -> assemble
-> depth-filter pyramid (L=4) -> U-Net input -> U-Net (when --unet != none).
A step = one frame of a seeded camera path inside the hall.  The scan
(300 MB) is larger than L2, so no extra L2 flush is needed between frames.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N > 1 (torchrun): the scan is sharded by cell-major point ranges; per frame
every rank projects its shard, minz is all-reduced (MIN), pass 2 accumulators
are reduced (SUM) to the frame's root (round-robin), which finishes the frame.

--impl reference times the reference's own CPU kernels (oracle/_ref, compiled
from /root/reference's _native.pyx; else the C port) driven by the oracle's
restatement of the reference host code, on this box's host cores.
"""

from __future__ import annotations

import argparse
import faulthandler
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/sec at 1920x1080 for N-M-point scan (1/2/4/8 B200); Gpoints/s projected"


def parse():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--points", type=int, default=20_000_000)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--unet", choices=["default", "reduced", "none"], default="default")
    ap.add_argument("--cpu-frames", type=int, default=2, help="cpu_baseline sample frames")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--views", type=int, default=8, help="camera poses cycled")
    ap.add_argument("--mode", choices=["replicas", "sharded"], default="replicas",
                    help="N>1: frame-parallel replicas of the scan (default; each rank renders "
                         "whole frames) or point-sharded frames (min/sum merges, root-side "
                         "filter + U-Net)")
    return ap.parse_args()


def workload_name(args):
    return (f"multi-station hall scan {args.points / 1e6:g}M points, {args.width}x{args.height}, "
            "cull+project+filter" + ("" if args.unet == "none" else f"+unet({args.unet})"))


# ------------------------------------------------------------------ clocks ---
class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line).  Polls NVML every ~2 ms from a thread
    (the timed region can be tens of milliseconds, too short for
    nvidia-smi's 100 ms loop)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, cuda_index: int):
        self.cuda_index = cuda_index
        self.samples = []
        self.smax = None
        self._stop = threading.Event()
        self._thread = None
        self.error = None

    def _handle(self, nv):
        """NVML handle of the CUDA device (matched by UUID; index fallback)."""
        try:
            import torch

            want = str(torch.cuda.get_device_properties(self.cuda_index).uuid)
            for i in range(nv.nvmlDeviceGetCount()):
                h = nv.nvmlDeviceGetHandleByIndex(i)
                uuid = nv.nvmlDeviceGetUUID(h)
                uuid = uuid.decode() if isinstance(uuid, bytes) else uuid
                if want in uuid:
                    return h
        except Exception:  # noqa: BLE001
            pass
        return nv.nvmlDeviceGetHandleByIndex(self.cuda_index)

    def start(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = self._handle(nv)
            self.smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.error = f"nvml unavailable: {e}"
            return

        def poll():
            while not self._stop.is_set():
                try:
                    self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                         nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
                except Exception:  # noqa: BLE001
                    pass
                time.sleep(0.002)

        self._thread = threading.Thread(target=poll, daemon=True)
        self._thread.start()

    def stop(self):
        self._stop.set()
        if self._thread is not None:
            self._thread.join(timeout=1)
        if self.error:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.error], "samples": 0}
        reasons = set()
        for _, mask in self.samples:
            for name, bit in self.REASONS.items():
                if mask & bit:
                    reasons.add(name)
        sm = [c for c, _ in self.samples]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ scene ----
def make_scene(args):
    from paper_2502_11618_b200.scenes import hall_cameras, multi_station_hall

    pos, col, _ = multi_station_hall(args.points)
    cams = hall_cameras(args.views, args.width, args.height)
    return pos, col, cams


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(
            d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


# --------------------------------------------------------------- CPU legs ---
def cpu_frames(pos, col, cams, args, n_frames, with_unet):
    """Reference CPU pipeline (oracle/_ref kernels, else the C port) on the
    host cores; returns (seconds per frame list, kind, cores, note)."""
    from oracle import oracle as O

    kind = "reference" if O.reference_module_path() else "port"
    kern = O.kernels(kind)
    port = O.PortKernels()
    grid = O.OracleGrid(pos, col, 1.0, kern)
    workers = os.cpu_count() or 1
    unet_ref = None
    if with_unet:
        from oracle.unet_ref import CpuUNet

        unet_ref = CpuUNet(args.unet, threads=workers)
    times = []
    for i in range(n_frames):
        cam = cams[i % len(cams)]
        t0 = time.perf_counter()
        rgb, depth, alpha, keep = O.render_frame(grid, cam, 0.01, 4, 0.1, 0.25, kern, port,
                                                 workers=workers)
        if unet_ref is not None:
            unet_ref.reconstruct(rgb, depth, alpha)
        times.append(time.perf_counter() - t0)
    return times, kind, workers


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    pos, col, cams = make_scene(args)
    with_unet = args.unet != "none"
    # bounded sample: the CPU path costs ~seconds per frame; time `steps`
    # frames after `warmup` warm-up frames (both capped so the run stays
    # within minutes)
    n_warm = min(max(1, args.warmup), 10)
    n_time = min(max(1, args.steps), 6)
    times, kind, cores = cpu_frames(pos, col, cams, args, n_warm + n_time, with_unet)
    times = times[n_warm:]
    fps = len(times) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s",
        "n_gpus": args.gpus, "steps": len(times), "warmup": n_warm,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded multi-station hall scan)",
        "config": {"workload": workload_name(args), "points": args.points,
                   "width": args.width, "height": args.height},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": kind,
                         "sample": f"{len(times)} full frames (cull+project+filter"
                                   f"{'+unet f32 torch-cpu' if with_unet else ''})"},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU arm ---
def run_b200(args):
    import torch

    from paper_2502_11618_b200 import PointCloud, build_grid, cull_cells, extract_frustum
    from paper_2502_11618_b200.engine import FrameRenderer

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    pos, col, cams = make_scene(args)
    cloud = PointCloud(pos, col)
    grid = build_grid(cloud, 1.0)
    torch.cuda.synchronize()
    unet = None
    if args.unet != "none":
        from paper_2502_11618_b200.unet import UNet

        unet = UNet.from_config(args.unet, seed=7, device=torch.device("cuda", local))
    sharded = world > 1 and args.mode == "sharded"
    if sharded:
        from paper_2502_11618_b200.shard import ShardedRenderer

        renderer = ShardedRenderer(grid, args.width, args.height, rank, world, unet=unet)
    else:
        # with a U-Net the f32 filtered frame is an intermediate the U-Net does
        # not read (it reads the packed bf16 input of the same filter kernel)
        renderer = FrameRenderer(grid, args.width, args.height, unet=unet,
                                 filtered_outputs=unet is None)
    # replicas: rank r renders its own frames (views offset by rank)
    view0 = 0 if sharded else rank * args.steps
    # candidate counts per view (algorithmic bytes of the projection passes)
    n_cand = []
    for cam in cams:
        cells = cull_cells(grid, extract_frustum(cam))
        s, e = grid.cell_ranges(cells)
        n_cand.append(int((e - s).sum()))

    for i in range(args.warmup):
        renderer.enqueue(cams[(view0 + i) % len(cams)])
    torch.cuda.synchronize()
    # ---- device-timed region (inputs resident in HBM) ----
    # The K timed frames run uninstrumented: an event recorded between two
    # kernels ends the programmatic-dependent-launch overlap at that boundary
    # (~3% of a frame).  The per-stage breakdown used for the rooflines comes
    # from a second, instrumented pass over the same frames afterwards.
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record()
    for i in range(args.steps):
        renderer.enqueue(cams[(view0 + args.warmup + i) % len(cams)])
    if sharded:
        torch.cuda.current_stream().wait_stream(renderer.side)
    t_end.record()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clk = clocks.stop()
    total_ms = t_start.elapsed_time(t_end)
    if world > 1:
        t = torch.tensor([total_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    # instrumented pass (stage events), not part of the timed value
    nst = 5
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nst + 1)]
           for _ in range(args.steps)]
    if not sharded:  # root-side work is on a side stream: no per-stage events
        for i in range(args.steps):
            evs[i][0].record()
            renderer.enqueue(cams[(view0 + args.warmup + i) % len(cams)], events=evs[i][1:])
        torch.cuda.synchronize()
    renderer.check_flags()
    stage = {k: [] for k in ("cull", "pass1", "pass2", "filter", "unet")}
    for e in ([] if sharded else evs):
        stage["cull"].append(e[0].elapsed_time(e[1]))
        stage["pass1"].append(e[1].elapsed_time(e[2]))
        stage["pass2"].append(e[2].elapsed_time(e[3]))
        stage["filter"].append(e[3].elapsed_time(e[4]))
        stage["unet"].append(e[4].elapsed_time(e[5]))
    # frames completed by the whole job in the timed region
    frames = args.steps * (1 if sharded or world == 1 else world)
    ms = total_ms / args.steps
    fps = frames * 1e3 / total_ms
    cand = [n_cand[(view0 + args.warmup + i) % len(cams)] for i in range(args.steps)]
    mean_cand = float(np.mean(cand))
    hbm, bf16, bf16s, peak_kind = measured_peaks()
    proj_gbs = 0.0
    if not sharded:
        t_proj = np.array(stage["pass1"]) + np.array(stage["pass2"])
        proj_bytes = 27.0 * np.array(cand)  # 12 B pass 1 + 15 B pass 2 per candidate
        proj_gbs = float(np.mean(proj_bytes / (t_proj * 1e-3)) / 1e9)
    stages_ms = {k: float(np.mean(v)) for k, v in stage.items()} if not sharded else None
    # per-frame device time, mean / p50 / p95 as the reference's run_bench
    # reports them (R:bench.py:61-67), from the instrumented pass
    frame_ms = None
    if not sharded and args.steps > 0:
        ft = np.array([e[0].elapsed_time(e[5]) for e in evs])
        frame_ms = {"mean": float(ft.mean()), "p50": float(np.percentile(ft, 50)),
                    "p95": float(np.percentile(ft, 95)),
                    "source": "instrumented pass, CUDA events around each frame"}
    roofline = None if sharded else {
                "kernel": "projection (k_frame_pass1 + k_frame_pass2)", "bound": "hbm",
                "achieved": proj_gbs, "peak": hbm, "unit": "GB/s", "frac": proj_gbs / hbm,
                "traffic": None, "peak_kind": peak_kind,
                "algorithmic": "27 B per candidate point"}
    # DRAM traffic of the same kernels from a committed ncu capture (bench.py
    # cannot profile itself): profiles/r01_traffic.json
    traffic = {}
    tpath = os.path.join(ROOT, "profiles", "r01_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            traffic = json.load(fh)
    if roofline is not None and "projection_dram_bytes_per_candidate" in traffic:
        roofline["traffic"] = traffic["projection_dram_bytes_per_candidate"] * mean_cand
        roofline["traffic_source"] = "profiles/r01_traffic.json (ncu dram bytes per candidate x candidates)"
    if unet is not None and not sharded:
        flops = unet.flops(args.width, renderer.unet_in.shape[1])
        tflops = flops / (stages_ms["unet"] * 1e-3) / 1e12
        roofline_unet = {"kernel": "U-Net (tcgen05 implicit-GEMM convs)", "bound": "tensor",
                         "achieved": tflops, "peak": bf16, "unit": "TFLOP/s",
                         "frac": tflops / bf16,
                         "traffic": traffic.get("unet_dram_bytes_per_frame"),
                         "traffic_source": "profiles/r01_traffic.json (ncu dram bytes, 22 launches)",
                         "peak_kind": peak_kind,
                         "algorithmic": f"{flops / 1e12:.4f} TFLOP per frame"}
        if stages_ms["unet"] > stages_ms["pass1"] + stages_ms["pass2"]:
            roofline, roofline_unet = roofline_unet, roofline
        roofline["other"] = roofline_unet
    # ---- end to end through the public API (host result every frame) ----
    # FrameRenderer.render_stream: every frame's camera goes in from the host
    # and its full result comes back to pinned host memory; the copy-out of
    # frame i overlaps the compute of frame i+1 (wall clock over K frames)
    e2e = None
    if not sharded:
        for _ in renderer.render_stream([cams[(view0 + i) % len(cams)] for i in range(3)]):
            pass
        torch.cuda.synchronize()
        seq = [cams[(view0 + args.warmup + i) % len(cams)] for i in range(args.steps)]
        if world > 1:
            torch.distributed.barrier()
        e0 = time.perf_counter()
        n_out = 0
        for _ in renderer.render_stream(seq):
            n_out += 1
        e_s = time.perf_counter() - e0
        if world > 1:  # slowest rank; every rank delivered n_out frames
            t = torch.tensor([e_s], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e_s = float(t.item())
        e2e = {"value": n_out * world / e_s, "unit": "frames/s",
               "api": "FrameRenderer.render_stream",
               "h2d_bytes_per_step": 320,  # camera struct + 6 frustum planes (kernel params)
               "d2h_bytes_per_step": renderer.d2h_bytes}
    line = {
        "metric": METRIC, "value": fps, "unit": "frames/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong" if sharded else "weak",
        "vs_baseline": None,
        "dtype": "f64" if unet is None else "f64+bf16",
        "data": "synthetic (seeded multi-station hall scan, random-init U-Net weights)",
        "config": {"workload": workload_name(args), "points": args.points,
                   "width": args.width, "height": args.height, "views": len(cams),
                   "parallelism": (f"point-shard{world}" if sharded else
                                   f"frame-replicas{world}" if world > 1 else "single"),
                   "l2": "inputs larger than L2 (scan 15 B/pt)"},
        "gpoints_per_s": mean_cand * fps / 1e9,
        "candidates_mean": mean_cand,
        "stages_ms": stages_ms,
        "frame_ms": frame_ms,
        "stages_note": "per-stage CUDA events from a second, instrumented pass over the same "
                       "frames; value / ms_per_step come from the uninstrumented timed pass",
        "roofline": roofline,
        "clocks": clk,
        "e2e": e2e,
        "gpu_launches": renderer.launches_per_frame * args.steps,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        times, kind, cores = cpu_frames(pos, col, cams, args, 1 + args.cpu_frames,
                                        args.unet != "none")
        times = times[1:]
        line["cpu_baseline"] = {"value": len(times) / sum(times), "unit": "frames/s",
                                "cores": cores, "kind": kind,
                                "sample": f"{len(times)} full frames of the same workload"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    faulthandler.enable()
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
