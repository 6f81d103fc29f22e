"""Host-side API parity (no GPU): the package root exports the reference's
__all__, and psnr / ssim / augment_brightness_contrast / the frame and
manifest files reproduce the reference's outputs (fixtures from
tests/golden/make_api_golden.py, run against the reference itself)."""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN

sys.path.insert(0, GOLDEN)
from make_api_golden import augment_cases, metric_cases  # noqa: E402

with open(os.path.join(GOLDEN, "api.json")) as _fh:
    API = json.load(_fh)


def test_root_exports_reference_all():
    import lidarsplat

    missing = [n for n in API["all"] if not hasattr(lidarsplat, n)]
    assert not missing, f"names the reference exports but lidarsplat lacks: {missing}"
    assert set(API["all"]) <= set(lidarsplat.__all__)


@pytest.mark.parametrize("i", range(5))
def test_metrics_match_reference(i):
    from lidarsplat import psnr, ssim

    p, t = metric_cases()[i]
    want = API["metrics"][i]
    assert psnr(p, t) == pytest.approx(want["psnr"], rel=1e-12, abs=1e-12)
    assert ssim(p, t) == pytest.approx(want["ssim"], rel=1e-12, abs=1e-12)


def test_metrics_errors():
    from lidarsplat import psnr, ssim

    a = np.zeros((12, 12, 3), np.float32)
    assert psnr(a, a) == 99.0
    with pytest.raises(ValueError, match="shapes differ"):
        psnr(a, np.zeros((12, 13, 3)))
    with pytest.raises(ValueError, match="at least 11px"):
        ssim(np.zeros((10, 30, 3)), np.zeros((10, 30, 3)))
    with pytest.raises(ValueError, match="expected an image"):
        psnr(np.zeros(5), np.zeros(5))


@pytest.mark.parametrize("i", range(3))
def test_augment_matches_reference_bytes(i):
    from lidarsplat import AugmentParams, augment_brightness_contrast

    img, alpha, params, spawn = augment_cases()[i]
    ss = None if spawn is None else np.random.SeedSequence(entropy=spawn[0],
                                                           spawn_key=(spawn[1],))
    out = augment_brightness_contrast(img, alpha, AugmentParams(**params), ss)
    assert out.dtype == np.float32 and out.shape == img.shape
    assert hashlib.sha256(np.ascontiguousarray(out).tobytes()).hexdigest() == API["augment"][i]
    assert np.array_equal(out[alpha == 0], img[alpha == 0])


def test_augment_params_validation():
    from lidarsplat import AugmentParams

    with pytest.raises(ValueError, match="not ordered"):
        AugmentParams(contrast_scale_range=(1.2, 0.9))
    with pytest.raises(ValueError, match=">= 1"):
        AugmentParams(group_count_range=(0, 2))
    with pytest.raises(ValueError, match="64 unsigned"):
        AugmentParams(seed=-1)


def test_frame_files_round_trip(tmp_path):
    from lidarsplat import FrameRGBDA
    from lidarsplat.io import read_frame, read_pfm, write_frame, write_pfm

    rng = np.random.default_rng(3)
    alpha = (rng.random((9, 13)) < 0.5).astype(np.uint8)
    depth = np.where(alpha, rng.random((9, 13)) * 10 + 0.1, 0).astype(np.float32)
    rgb = np.where(alpha[:, :, None], rng.random((9, 13, 3)), 0).astype(np.float32)
    f = FrameRGBDA(rgb, depth, alpha)
    write_frame(f, tmp_path / "x")
    g = read_frame(tmp_path / "x")
    assert np.array_equal(g.depth, depth) and np.array_equal(g.alpha, alpha)
    assert np.abs(g.rgb - rgb).max() <= 0.5 / 255 + 1e-7
    write_pfm(tmp_path / "d.pfm", depth)
    assert np.array_equal(read_pfm(tmp_path / "d.pfm"), depth)


def test_manifest_and_cameras_round_trip(tmp_path):
    from lidarsplat.errors import CameraError, DatasetError
    from lidarsplat.io import (DatasetManifest, load_cameras, load_manifest, save_cameras,
                               save_manifest)

    m = DatasetManifest(mode="leaky", ids=("a", "b"), params={"x": 1}, seed=5)
    save_manifest(tmp_path, m)
    assert load_manifest(tmp_path) == m
    with pytest.raises(DatasetError, match="unique"):
        DatasetManifest(mode="leaky", ids=("a", "a"), params={}, seed=0)
    c2w = np.eye(4)
    c2w[:3, 3] = [1.0, 2.0, 3.0]
    save_cameras(tmp_path / "c.json", dict(fx=10, fy=10, cx=8, cy=8, width=16, height=16),
                 [("f0", c2w)])
    cams = load_cameras(tmp_path / "c.json")
    assert list(cams) == ["f0"]
    assert np.allclose(cams["f0"].world_to_camera.translation, [-1.0, -2.0, -3.0])
    (tmp_path / "bad.json").write_text("{")
    with pytest.raises(CameraError, match="not valid JSON"):
        load_cameras(tmp_path / "bad.json")


def test_bench_report_shape_matches_reference_schema():
    """BenchReport.to_dict of a report satisfies the reference's JSON schema."""
    import jsonschema

    from lidarsplat import BenchReport

    stats = {s: {"mean": 1.0, "p50": 1.0, "p95": 2.0}
             for s in ("culling_ms", "projection_ms", "filter_ms", "total_ms")}
    r = BenchReport(points_total=10, resolution=(64, 48), frames=3, backend="cuda",
                    stats=stats, fps=1000.0)
    jsonschema.validate(r.to_dict(), API["bench_schema"])
    assert r.gate_warnings() == []
    slow = BenchReport(points_total=10, resolution=(64, 48), frames=3, backend="cuda",
                       stats={**stats, "total_ms": {"mean": 40.0, "p50": 40.0, "p95": 40.0},
                              "culling_ms": {"mean": 61.0, "p50": 1.0, "p95": 1.0}}, fps=25.0)
    w = slow.gate_warnings()
    assert len(w) == 2 and "culling" in w[0] and "33 ms budget" in w[1]
