"""bench.py's JSON-line contract, on a tiny workload.

CPU: the reference arm (`--impl reference`, the oracle pipeline on host cores)
prints one line with the contract keys, honours --steps/--warmup and stays
silent on ranks other than 0.  GPU: the b200 arm's line carries `roofline`,
`cpu_baseline`, `e2e`, `clocks` and a non-zero `gpu_launches`.
"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TINY = ["--points", "20000", "--width", "64", "--height", "64", "--unet", "reduced"]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, env=None, timeout=300, rc=0):
    e = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        e.pop(k, None)
    e.update(env or {})
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                       env=e, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == rc, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.strip().startswith("{")]
    return lines


def test_reference_arm_line():
    lines = _run(["--impl", "reference", "--steps", "2", "--warmup", "3"] + TINY)
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference"
    assert d["steps"] == 2 and d["warmup"] == 3
    assert d["value"] > 0 and d["unit"] == "frames/s" and d["higher_is_better"] is True
    assert d["config"]["points"] == 20000 and d["config"]["width"] == 64
    assert d["e2e"] == {"value": d["value"], "unit": "frames/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["kind"] in ("reference", "port") and cb["cores"] >= 1


def test_reference_arm_other_ranks_silent():
    assert _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1"] + TINY,
                env={"RANK": "1", "WORLD_SIZE": "2"}) == []


def test_world_size_must_match_gpus():
    assert _run(["--impl", "reference", "--gpus", "4", "--steps", "1"] + TINY,
                env={"RANK": "0", "WORLD_SIZE": "2"}, rc=2) == []


def test_gpus_flag_launches_ranks():
    """--gpus 2 without torchrun re-executes bench.py as 2 ranks
    (torch.distributed.run); the reference arm prints once, from rank 0, with
    n_gpus 2 and the same config dict the b200 arm prints."""
    lines = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1"] + TINY)
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "point-shard2"
    sys.path.insert(0, ROOT)
    import bench

    class A:
        points, width, height, views, unet, mode = 20000, 64, 64, 8, "reduced", "sharded"

    assert d["config"] == bench.bench_config(A, 2)


@pytest.mark.gpu
def test_b200_arm_line():
    lines = _run(["--steps", "3", "--warmup", "3"] + TINY)
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert BASE_KEYS | {"roofline", "clocks", "gpu_launches", "cpu_baseline"} <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["gpu_launches"] > 0
    rf = d["roofline"]
    assert rf["bound"] in ("hbm", "tensor") and rf["peak"] > 0
    assert rf["frac"] == pytest.approx(rf["achieved"] / rf["peak"])
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["clocks"]["sm_max_mhz"] > 0
    par = d["parity"]
    assert par["bit_exact"] is True and par["frames"] >= 1
    assert par["unet_within_tolerance"] is True
    ref = json.loads(_run(["--impl", "reference", "--steps", "1", "--warmup", "1"] + TINY)[0])
    assert ref["config"] == d["config"]
