"""FrameRenderer public calls on the B200: the pipelined render_stream (copy
of frame i overlapping compute of frame i+1, double-buffered device outputs,
pinned host ring) returns exactly what per-frame render() returns."""

import numpy as np
import pytest

from conftest import random_cloud, random_view

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu(cuda_ready):
    return cuda_ready


@pytest.mark.parametrize("with_unet", [False, True])
def test_render_stream_equals_render(with_unet):
    from paper_2502_11618_b200 import build_grid
    from paper_2502_11618_b200.engine import FrameRenderer
    from paper_2502_11618_b200.unet import UNet

    rng = np.random.default_rng(11)
    cloud = random_cloud(rng, 200_000, extent=10.0, offset=-5.0)
    views = [random_view(rng, cloud, width=256, height=192) for _ in range(7)]
    unet = UNet.from_config("reduced", seed=2) if with_unet else None
    r = FrameRenderer(build_grid(cloud, 1.0), 256, 192, unet=unet)
    single = []
    for v in views:
        out = r.render(v)
        single.append(out.copy() if with_unet else
                      (out.rgb.copy(), out.depth.copy(), out.alpha.copy()))
    streamed = []
    for out in r.render_stream(views, depth=2):
        streamed.append(out.copy() if with_unet else
                        (out.rgb.copy(), out.depth.copy(), out.alpha.copy()))
    r.check_flags()
    assert len(streamed) == len(views)
    for a, b in zip(single, streamed):
        if with_unet:
            assert np.array_equal(a, b)
        else:
            assert all(np.array_equal(x, y) for x, y in zip(a, b))
    # frames differ from one another (the ring really carried distinct results)
    first = streamed[0] if with_unet else streamed[0][1]
    assert any(not np.array_equal(first, s if with_unet else s[1]) for s in streamed[1:])


def test_ply_load_stages_device_copy(tmp_path):
    """load_ply(device=True) leaves the scan resident: build_grid reuses the
    staged tensors and renders the same frame as a host-loaded cloud."""
    from paper_2502_11618_b200 import build_grid, project_points
    from paper_2502_11618_b200.io import load_ply, save_ply

    rng = np.random.default_rng(8)
    cloud = random_cloud(rng, 50_000, extent=8.0, offset=-4.0)
    save_ply(cloud, tmp_path / "c.ply")
    staged = load_ply(tmp_path / "c.ply", device=True)
    assert staged._device, "device copy not staged"
    pos, _ = staged.device_arrays()
    assert pos.is_cuda and pos.shape == (50_000, 3)
    cam = random_view(rng, cloud)
    a = project_points(staged, build_grid(staged, 1.0), cam)
    b = project_points(cloud, build_grid(cloud, 1.0), cam)
    assert np.array_equal(a.rgb, b.rgb) and np.array_equal(a.depth, b.depth)


def test_unfiltered_outputs_same_reconstruction():
    """filtered_outputs=False (the f32 filtered frame is not written) gives a
    bit-identical U-Net reconstruction."""
    from paper_2502_11618_b200 import build_grid
    from paper_2502_11618_b200.engine import FrameRenderer
    from paper_2502_11618_b200.unet import UNet

    rng = np.random.default_rng(12)
    cloud = random_cloud(rng, 150_000, extent=10.0, offset=-5.0)
    views = [random_view(rng, cloud, width=256, height=192) for _ in range(3)]
    grid = build_grid(cloud, 1.0)
    unet = UNet.from_config("reduced", seed=2)
    a = FrameRenderer(grid, 256, 192, unet=unet)
    b = FrameRenderer(grid, 256, 192, unet=unet, filtered_outputs=False)
    for v in views:
        assert np.array_equal(a.render(v), b.render(v))
        # b's assembly writes the U-Net input directly (no raw f32 rgb) and its
        # final filter step clears the rejected pixels: the same input tensor
        assert bool((a.unet_in == b.unet_in).all())


def test_concurrent_host_threads_separate_streams():
    """The ABI keeps no per-call global state (include/lidarsplat_cuda.h):
    two host threads, each with its own renderer on its own stream, issue
    frames concurrently (first-use attribute/occupancy caches raced) and get
    exactly the frames a single thread renders."""
    import threading

    import torch

    from paper_2502_11618_b200 import build_grid
    from paper_2502_11618_b200.engine import FrameRenderer
    from paper_2502_11618_b200.unet import UNet

    rng = np.random.default_rng(21)
    cloud = random_cloud(rng, 150_000, extent=10.0, offset=-5.0)
    views = [random_view(rng, cloud, width=256, height=192) for _ in range(6)]
    grid = build_grid(cloud, 1.0)
    # activation buffers belong to a UNet instance: one instance per thread
    unets = [UNet.from_config("reduced", seed=4) for _ in range(3)]
    results = {}
    errors = []
    start = threading.Barrier(2)

    def worker(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                r = FrameRenderer(grid, 256, 192, unet=unets[k])
                start.wait()
                results[k] = [r.render(v).copy() for v in views[k::2]]
                r.check_flags()
        except Exception as e:  # surfaced in the main thread
            errors.append(e)

    ts = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    ref = FrameRenderer(grid, 256, 192, unet=unets[2])
    for k in range(2):
        for v, got in zip(views[k::2], results[k]):
            assert np.array_equal(ref.render(v), got)


def _hot_pixel_cloud(rng, n_hot=70_000):
    """A random scene plus ``n_hot`` white points on one pixel-centre ray at
    the same depth: that pixel keeps them all, so its f32 colour sums pass
    2^24 (> 65,793 points) and the fast path must flag the frame."""
    from paper_2502_11618_b200 import PointCloud

    base = random_cloud(rng, 60_000, extent=6.0, offset=-3.0)
    hot = np.tile(np.array([[0.01, 0.01, 1.5]], np.float32), (n_hot, 1))
    pos = np.concatenate([base.positions + np.float32([0, 0, 6.0]), hot])
    col = np.concatenate([base.colors, np.full((n_hot, 3), 255, np.uint8)])
    return PointCloud(pos, col)


def _oracle_filtered(cloud, cam):
    from oracle import oracle as O

    port = O.PortKernels()
    og = O.OracleGrid(cloud.positions, cloud.colors, 1.0, port)
    return O.render_frame(og, cam, 0.01, 4, 0.1, 0.25, port, port)


@pytest.mark.parametrize("with_unet", [False, True])
def test_render_honours_accumulator_bound(with_unet):
    """FrameRenderer.render / render_stream and ViewBatchRenderer.render on a
    frame where one pixel keeps 70,000 points: the device frame is flagged and
    the public calls return the exact (u64-path) result, bit-identical to the
    oracle's frame (and, with a U-Net, to the U-Net of the oracle's frame)."""
    from conftest import make_camera

    from paper_2502_11618_b200 import build_grid
    from paper_2502_11618_b200.bridge import UNetBridgeModel
    from paper_2502_11618_b200.engine import FrameRenderer, ViewBatchRenderer
    from paper_2502_11618_b200.frame import FrameRGBDA
    from paper_2502_11618_b200.io.tensor import frame_to_tensor
    from paper_2502_11618_b200.unet import UNet

    rng = np.random.default_rng(31)
    cloud = _hot_pixel_cloud(rng)
    cam = make_camera(width=128, height=96, fx=80.0, fy=80.0)
    grid = build_grid(cloud, 1.0)
    rgb, depth, alpha, _ = _oracle_filtered(cloud, cam)
    unet = UNet.from_config("reduced", seed=5) if with_unet else None
    r = FrameRenderer(grid, cam.width, cam.height, unet=unet)
    # the device-only form flags the frame
    r.enqueue(cam)
    with pytest.raises(RuntimeError, match="accumulator bound"):
        r.check_flags()
    if with_unet:
        want = UNetBridgeModel(unet).reconstruct(
            frame_to_tensor(FrameRGBDA(rgb, depth, alpha))).transpose(1, 2, 0)
    got = [r.render(cam)] + list(r.render_stream([cam, cam, cam]))
    vb = ViewBatchRenderer(grid, cam.width, cam.height, 2, unet=unet)
    got += vb.render([cam, cam])
    for g in got:
        if with_unet:
            assert np.array_equal(g, want)
        else:
            assert np.array_equal(g.rgb, rgb) and np.array_equal(g.depth, depth)
            assert np.array_equal(g.alpha, alpha)
    r.check_flags()  # public calls consumed their flags


def test_render_returns_fresh_arrays():
    """render() returns new arrays each call (the reference returns new
    arrays): a later call does not overwrite an earlier result."""
    from paper_2502_11618_b200 import build_grid
    from paper_2502_11618_b200.engine import FrameRenderer

    rng = np.random.default_rng(5)
    cloud = random_cloud(rng, 80_000, extent=10.0, offset=-5.0)
    v1, v2 = (random_view(rng, cloud, width=128, height=96) for _ in range(2))
    r = FrameRenderer(build_grid(cloud, 1.0), 128, 96)
    a = r.render(v1)
    a_depth = a.depth.copy()
    b = r.render(v2)
    assert not np.array_equal(a_depth, b.depth)
    assert np.array_equal(a.depth, a_depth)


def test_concurrent_renderers_share_grid_and_unet():
    """Renderers of different resolutions on one grid and ONE UNet, driven
    from two host threads on their own streams with many frames in flight:
    each renderer owns its cull bits / work list / pass-1 cache, and the U-Net
    keeps activations per stream, so every frame equals a serial render."""
    import threading

    import torch

    from paper_2502_11618_b200 import build_grid
    from paper_2502_11618_b200.engine import FrameRenderer
    from paper_2502_11618_b200.unet import UNet

    rng = np.random.default_rng(22)
    cloud = random_cloud(rng, 300_000, extent=10.0, offset=-5.0)
    sizes = [(256, 192), (160, 128)]
    views = {k: [random_view(rng, cloud, width=w, height=h) for _ in range(10)]
             for k, (w, h) in enumerate(sizes)}
    grid = build_grid(cloud, 1.0)
    unet = UNet.from_config("reduced", seed=4)
    results, errors = {}, []
    start = threading.Barrier(2)

    def worker(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                r = FrameRenderer(grid, *sizes[k], unet=unet)
                start.wait()
                results[k] = [o.copy() for o in r.render_stream(views[k], depth=3)]
        except Exception as e:  # surfaced in the main thread
            errors.append(e)

    ts = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for k, (w, h) in enumerate(sizes):
        ref = FrameRenderer(grid, w, h, unet=unet)
        for v, got in zip(views[k], results[k]):
            assert np.array_equal(ref.render(v), got)


def test_run_bench_report_matches_reference_schema():
    """lidarsplat.run_bench (R:bench.py:70-108): device stage timing, report
    valid against the reference's schema, grid and brute-force paths."""
    import json
    import os

    import jsonschema

    from conftest import GOLDEN

    from lidarsplat import FilterParams, RenderParams, build_grid, run_bench

    with open(os.path.join(GOLDEN, "api.json")) as fh:
        schema = json.load(fh)["bench_schema"]
    rng = np.random.default_rng(9)
    cloud = random_cloud(rng, 100_000, extent=10.0, offset=-5.0)
    cams = [random_view(rng, cloud, width=128, height=96) for _ in range(3)]
    for grid in (build_grid(cloud, 1.0), None):
        rep = run_bench(cloud, grid, cams, RenderParams(), FilterParams(), 5,
                        backend_name="cuda")
        jsonschema.validate(rep.to_dict(), schema)
        st = rep.stats
        assert rep.frames == 5 and rep.resolution == (128, 96)
        assert st["total_ms"]["mean"] >= st["projection_ms"]["mean"] > 0
        assert rep.fps == pytest.approx(1000.0 / st["total_ms"]["mean"])
    with pytest.raises(ValueError, match="at least one frame"):
        run_bench(cloud, None, cams, RenderParams(), FilterParams(), 0)


def test_generate_dataset_deterministic(tmp_path):
    """generate_dataset: one pair per frame written with the manifest; two
    runs give byte-identical trees, and the stored input depth/alpha equal the
    device pair recipe's."""
    import filecmp

    from lidarsplat import (AugmentParams, FilterParams, RenderParams, build_grid,
                            generate_dataset, make_leaky_pair)
    from lidarsplat.io import load_manifest, read_frame

    rng = np.random.default_rng(13)
    cloud = random_cloud(rng, 80_000, extent=10.0, offset=-5.0)
    frames = []
    for i in range(3):
        cam = random_view(rng, cloud, width=64, height=48)
        frames.append((f"f{i}", cam, rng.random((48, 64, 3)).astype(np.float32)))
    grid = build_grid(cloud, 1.0)
    for d in ("a", "b"):
        generate_dataset(cloud, frames, tmp_path / d, "leaky", AugmentParams(seed=3),
                         FilterParams(), RenderParams(), grid=grid)
    m = load_manifest(tmp_path / "a")
    assert m.ids == ("f0", "f1", "f2") and m.mode == "leaky"
    cmp = filecmp.dircmp(tmp_path / "a" / "pairs", tmp_path / "b" / "pairs")
    assert not cmp.diff_files and not cmp.left_only and len(cmp.same_files) == 12
    pair = make_leaky_pair(cloud, grid, frames[1][2], frames[1][1], FilterParams(),
                           RenderParams(), "f1")
    stored = read_frame(tmp_path / "a" / "pairs" / "f1.input")
    assert np.array_equal(stored.depth, pair.input.depth)
    assert np.array_equal(stored.alpha, pair.input.alpha)


@pytest.mark.parametrize("with_unet", [False, True])
def test_graph_frames_equal_launched_frames(with_unet):
    """FrameRenderer(graph=True): each frame is one CUDA-graph launch
    re-targeted to the frame's camera (ls_frame_graph_set_camera) -- every
    frame equals the launch-by-launch frame, through render, render_stream and
    back-to-back enqueues."""
    import torch

    from paper_2502_11618_b200 import build_grid
    from paper_2502_11618_b200.engine import FrameRenderer
    from paper_2502_11618_b200.unet import UNet

    rng = np.random.default_rng(41)
    cloud = random_cloud(rng, 250_000, extent=10.0, offset=-5.0)
    views = [random_view(rng, cloud, width=256, height=192) for _ in range(6)]
    grid = build_grid(cloud, 1.0)
    unet = UNet.from_config("reduced", seed=2) if with_unet else None
    a = FrameRenderer(grid, 256, 192, unet=unet)
    b = FrameRenderer(grid, 256, 192, unet=unet, graph=True)

    def host(o):
        return o.copy() if with_unet else (o.rgb.copy(), o.depth.copy(), o.alpha.copy())

    def same(x, y):
        return np.array_equal(x, y) if with_unet else all(
            np.array_equal(p, q) for p, q in zip(x, y))

    ref = [host(a.render(v)) for v in views]
    got = [host(b.render(v)) for v in views]
    got_stream = [host(o) for o in b.render_stream(views)]
    for r, g1, g2 in zip(ref, got, got_stream):
        assert same(r, g1) and same(r, g2)
    # back-to-back graph frames on one stream, last one compared
    for v in views:
        b.enqueue(v)
    torch.cuda.synchronize()
    last = b.rgb_out[0, :192].cpu().numpy() if with_unet else b.fdepth.cpu().numpy()
    want = ref[-1] if with_unet else ref[-1][1]
    assert np.array_equal(last, want)
    b.check_flags()
