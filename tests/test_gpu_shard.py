"""Sharded rendering on the GPU (one device): every shard's cull + passes run
through the real kernels and are merged on-device; the merged frame must be
bit-identical to the unsharded frame for any shard count.
The multi-rank collectives themselves are covered by tests/test_shard_gloo.py."""

import os

import numpy as np
import pytest

from conftest import random_cloud, random_view

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu(cuda_ready):
    return cuda_ready


def _frame_setup(n=400_000, seed=3):
    from lidarsplat import CameraModel, build_grid

    rng = np.random.default_rng(seed)
    cloud = random_cloud(rng, n, extent=10.0, offset=-5.0)
    cam0 = random_view(rng, cloud)
    cam = CameraModel.unchecked(300.0, 300.0, 160.0, 120.0, 320, 240, cam0.world_to_camera)
    return cloud, cam, build_grid(cloud, 1.0)


@pytest.mark.parametrize("cached", [False, True])
@pytest.mark.parametrize("world", [2, 3, 5])
def test_virtual_shards_bit_identical(world, cached):
    """Shards projected separately, minz merged by MIN and accumulators by SUM,
    equal the single-scene frame.  Recompute mode rebuilds each shard's work
    list for pass 2 (list order is irrelevant); cached mode reuses pass 1's
    list and cache, as it must."""
    import torch

    from lidarsplat import _lib
    from lidarsplat.geometry import extract_frustum
    from lidarsplat.grid import DeviceScene
    from lidarsplat.render import FrameBuffers, frame_cache, project_scene
    from lidarsplat.shard import shard_bounds, shard_cell_offsets

    cloud, cam, grid = _frame_setup()
    dev = torch.device("cuda")
    full = grid.scene()
    ref = FrameBuffers(cam.width, cam.height, dev)
    project_scene(full, cam, 0.01, ref)
    lib = _lib.load()
    st = _lib.stream_ptr()
    c = _lib.make_camera(cam)
    scenes, bufs = [], []
    for r in range(world):
        s, e = shard_bounds(full.n_points, r, world)
        offs = shard_cell_offsets(grid._device_field("cell_offsets", np.int64), s, e)
        sc = DeviceScene(full.positions[s:e], full.colors[s:e], offs, grid.origin,
                         grid.cell_size, grid.dims)
        scenes.append(sc)
        b = FrameBuffers(cam.width, cam.height, dev)
        bufs.append(b)
        sc.cull_bits(extract_frustum(cam).planes)
        tl, tc = sc.worklist()
        cache = _lib.ptr(frame_cache(sc, cam)) if cached else None
        _lib.check(lib.ls_frame_pass1(sc.struct, sc.keep_bits.data_ptr(), tl.data_ptr(),
                                      tc.data_ptr(), c, b.minz.data_ptr(), cache, st), "pass1")
    gmin = torch.stack([b.minz for b in bufs]).min(0).values
    for sc, b in zip(scenes, bufs):
        b.minz.copy_(gmin)
        cache = None
        if cached:
            tl, tc, cache = sc.tile_list, sc.tile_count, _lib.ptr(frame_cache(sc, cam))
        else:
            sc.cull_bits(extract_frustum(cam).planes)
            tl, tc = sc.worklist()
        _lib.check(lib.ls_frame_pass2(sc.struct, sc.keep_bits.data_ptr(), tl.data_ptr(),
                                      tc.data_ptr(), c, 0.01, b.minz.data_ptr(), cache,
                                      b.accum.data_ptr(), st), "pass2")
    root = bufs[world - 1]
    root.accum.copy_(torch.stack([b.accum for b in bufs]).sum(0))
    _lib.check(lib.ls_frame_finish(root.minz.data_ptr(), root.accum.data_ptr(), cam.width,
                                   cam.height, None, root.rgb.data_ptr(), root.depth.data_ptr(),
                                   root.alpha.data_ptr(), None, None, None, None, None, 0, 0, 0.1,
                                   None, root.flags.data_ptr(), st), "finish")
    torch.cuda.synchronize()
    assert torch.equal(root.rgb, ref.rgb)
    assert torch.equal(root.depth, ref.depth)
    assert torch.equal(root.alpha, ref.alpha)


def test_sharded_renderer_single_rank_group():
    """ShardedRenderer wiring (cull -> pass 1 -> all-reduce -> pass 2 -> reduce
    -> finish) in a 1-rank NCCL group matches FrameRenderer."""
    import socket

    import torch
    import torch.distributed as dist

    from lidarsplat.engine import FrameRenderer
    from lidarsplat.shard import ShardedRenderer

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    try:
        from lidarsplat.unet import UNet

        cloud, cam, grid = _frame_setup(seed=5)
        rng = np.random.default_rng(5)
        views = [cam] + [random_view(rng, cloud, width=cam.width, height=cam.height)
                         for _ in range(3)]
        unet = UNet.from_config("reduced", seed=4)
        a = ShardedRenderer(grid, cam.width, cam.height, 0, 1, unet=unet)
        b = FrameRenderer(grid, cam.width, cam.height, unet=unet)
        for v in views:  # root-side work runs on a side stream; compare every frame
            a.enqueue(v)
            a.flush()  # frames are pipelined by one stage
            b.enqueue(v)
            torch.cuda.synchronize()
            assert torch.equal(a.frgb, b.frgb) and torch.equal(a.falpha, b.falpha)
            assert torch.equal(a.fdepth, b.fdepth)
            assert torch.equal(a.rgb_out, b.rgb_out)
        a.check_flags()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_renderer_virtual_ranks(world):
    """ShardedRenderer with world > 1: every rank's renderer (its own shard
    scene, cull, work list, pass-1 cache, double-buffered pass sets, side
    stream) driven through VirtualShards -- the frame's MIN / SUM merges done
    in memory, the root rotating per frame -- returns, on each frame's root,
    the frame and U-Net output FrameRenderer renders (bit-identical)."""
    import torch

    from lidarsplat.engine import FrameRenderer
    from lidarsplat.shard import VirtualShards
    from lidarsplat.unet import UNet

    cloud, cam, grid = _frame_setup(seed=7)
    rng = np.random.default_rng(7)
    views = [cam] + [random_view(rng, cloud, width=cam.width, height=cam.height)
                     for _ in range(2 * world)]
    unet = UNet.from_config("reduced", seed=4)
    vs = VirtualShards(grid, cam.width, cam.height, world, unet=unet)
    assert [r.shard for r in vs.ranks][0][0] == 0 and vs.ranks[-1].shard[1] == grid.scene().n_points
    ref = FrameRenderer(grid, cam.width, cam.height, unet=unet)
    roots = []
    for v in views:
        root = vs.enqueue(v)
        roots.append(root)
        ref.enqueue(v)
        vs.synchronize()
        torch.cuda.synchronize()
        r = vs.ranks[root]
        assert torch.equal(r.frgb, ref.frgb) and torch.equal(r.falpha, ref.falpha)
        assert torch.equal(r.fdepth, ref.fdepth)
        assert torch.equal(r.rgb_out, ref.rgb_out)
    assert sorted(set(roots)) == list(range(world))
    for r in vs.ranks:
        r.check_flags()


def test_sharded_renderer_pipelined_frames_single_rank():
    """Back-to-back ShardedRenderer frames without flushing in between (each
    frame's pass 2 runs after the next frame's pass 1, with three pass-buffer
    sets and two scratch sets in rotation) deliver the FrameRenderer frames:
    the root's outputs are checked after every second frame and at the end."""
    import socket

    import torch
    import torch.distributed as dist

    from lidarsplat.engine import FrameRenderer
    from lidarsplat.shard import ShardedRenderer

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    try:
        cloud, cam, grid = _frame_setup(seed=9)
        rng = np.random.default_rng(9)
        views = [random_view(rng, cloud, width=cam.width, height=cam.height) for _ in range(7)]
        a = ShardedRenderer(grid, cam.width, cam.height, 0, 1)
        b = FrameRenderer(grid, cam.width, cam.height)
        for i, v in enumerate(views):
            a.enqueue(v)  # completes frame i-1
            if i % 2 == 1:
                a.synchronize()  # flushes frame i too
                b.enqueue(v)
                torch.cuda.synchronize()
                assert torch.equal(a.frgb, b.frgb) and torch.equal(a.fdepth, b.fdepth)
                assert torch.equal(a.falpha, b.falpha)
        a.synchronize()
        b.enqueue(views[-1])
        torch.cuda.synchronize()
        assert torch.equal(a.frgb, b.frgb) and torch.equal(a.fdepth, b.fdepth)
        a.check_flags()
    finally:
        dist.destroy_process_group()
