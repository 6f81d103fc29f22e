"""Multi-view batched projection on the B200: one read of
the scan feeds up to LS_MAX_VIEWS views (ls_frame_project_views).  Every
view's frame must be bit-identical to rendering that view alone
(render.py:84-143 runs once per view in the reference) and to the oracle."""

import numpy as np
import pytest

from conftest import make_camera, random_cloud, random_view
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu(cuda_ready):
    return cuda_ready


def _eq(a, b):
    return (np.array_equal(a.rgb, b.rgb) and np.array_equal(a.depth, b.depth)
            and np.array_equal(a.alpha, b.alpha))


@pytest.mark.parametrize("cache", [False, True])
@pytest.mark.parametrize("k", [1, 2, 3, 8])
def test_views_equal_single_view_frames(rng, monkeypatch, k, cache):
    from lidarsplat import build_grid, project_points, project_points_views
    from paper_2502_11618_b200 import render

    monkeypatch.setattr(render, "USE_FRAME_CACHE", cache)
    cloud = random_cloud(rng, 120_000, extent=12.0, offset=-6.0)
    grid = build_grid(cloud, 1.0)
    cams = [random_view(rng, cloud, width=160, height=128) for _ in range(k)]
    batched = project_points_views(cloud, grid, cams)
    assert len(batched) == k
    for cam, fr in zip(cams, batched):
        assert _eq(fr, project_points(cloud, grid, cam))
        assert fr.alpha.sum() > 0


@pytest.mark.parametrize("cache", [False, True])
@pytest.mark.parametrize("eps", [0.0, 0.01])
def test_views_match_oracle_and_brute_force(rng, port, monkeypatch, eps, cache):
    """Includes points one f64 ulp apart along lines of sight and eps = 0
    (winners exactly on the threshold: the cached pass 2's exact path)."""
    from lidarsplat import PointCloud, RenderParams, build_grid, project_points_views
    from paper_2502_11618_b200 import render

    monkeypatch.setattr(render, "USE_FRAME_CACHE", cache)
    cloud = random_cloud(rng, 60_000, extent=10.0, offset=-5.0)
    base = cloud.positions[:3000].astype(np.float64)
    dup = np.concatenate([base, np.nextafter(base, np.inf)]).astype(np.float32)
    cloud = PointCloud(np.concatenate([cloud.positions, dup]),
                       np.concatenate([cloud.colors,
                                       rng.integers(0, 256, (len(dup), 3), dtype=np.uint8)]))
    cams = [random_view(rng, cloud, width=96, height=64) for _ in range(5)]
    params = RenderParams(zbuffer_epsilon_rel=eps)
    culled = project_points_views(cloud, build_grid(cloud, 0.7), cams, params)
    brute = project_points_views(cloud, None, cams, params)
    for cam, a, b in zip(cams, culled, brute):
        assert _eq(a, b)
        rgb, depth, alpha, _, _ = O.project(cloud.positions, cloud.colors, np.zeros(1, np.int64),
                                            np.array([cloud.count], np.int64), cam, eps, port)
        assert np.array_equal(a.rgb, rgb) and np.array_equal(a.depth, depth)
        assert np.array_equal(a.alpha, alpha)


def test_views_with_disjoint_and_empty_frusta():
    """Views looking in opposite directions (tiles kept by one view only,
    mixed tiles per view) and a view that sees nothing."""
    from lidarsplat import build_grid, project_points, project_points_views

    rng = np.random.default_rng(5)
    cloud = random_cloud(rng, 150_000, extent=20.0, offset=-10.0)
    grid = build_grid(cloud, 1.5)
    cams = [make_camera(eye=(0, 0, 0), target=t, width=128, height=96)
            for t in [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, 0, 1), (0.3, -1, 0.2)]]
    # far outside the cloud, looking away from it: nothing visible
    cams.append(make_camera(eye=(100, 100, 100), target=(200, 200, 200), width=128, height=96))
    frames = project_points_views(cloud, grid, cams)
    for cam, fr in zip(cams, frames):
        assert _eq(fr, project_points(cloud, grid, cam))
    assert frames[-1].alpha.sum() == 0
    assert all(f.alpha.sum() > 0 for f in frames[:-1])


def test_more_views_than_a_batch_and_validation(rng):
    from lidarsplat import build_grid, project_points, project_points_views

    cloud = random_cloud(rng, 40_000, extent=8.0, offset=-4.0)
    grid = build_grid(cloud, 1.0)
    cams = [random_view(rng, cloud, width=64, height=48) for _ in range(11)]
    frames = project_points_views(cloud, grid, cams)
    assert len(frames) == 11
    for cam, fr in zip(cams, frames):
        assert _eq(fr, project_points(cloud, grid, cam))
    other = random_view(rng, cloud, width=80, height=48)
    with pytest.raises(ValueError, match="width and height"):
        project_points_views(cloud, grid, [cams[0], other])


def test_view_batch_renderer_equals_frame_renderer(rng):
    from paper_2502_11618_b200 import build_grid
    from paper_2502_11618_b200.engine import FrameRenderer, ViewBatchRenderer
    from paper_2502_11618_b200.unet import UNet

    cloud = random_cloud(rng, 200_000, extent=10.0, offset=-5.0)
    grid = build_grid(cloud, 1.0)
    cams = [random_view(rng, cloud, width=256, height=192) for _ in range(4)]
    # filtered frames, no U-Net: bit-identical
    vr = ViewBatchRenderer(grid, 256, 192, 4)
    fr = FrameRenderer(grid, 256, 192)
    batch = vr.render(cams)
    vr.check_flags()
    for cam, out in zip(cams, batch):
        assert _eq(out, fr.render(cam))
    # batched U-Net over the 4 views vs one U-Net forward per view (same
    # weights, same kernels): identical reconstructions
    net = UNet.from_config("reduced", seed=4)
    vr = ViewBatchRenderer(grid, 256, 192, 4, unet=net)
    fr = FrameRenderer(grid, 256, 192, unet=net)
    batch = vr.render(cams)
    for cam, out in zip(cams, batch):
        single = fr.render(cam)
        assert np.abs(out - single).max() <= 1e-6
    # a second call reuses the (reset) pass buffers
    again = vr.render(cams[::-1])
    for a, b in zip(again, batch[::-1]):
        assert np.array_equal(a, b)


def test_capi_rejects_bad_view_batches(rng):
    import torch

    from paper_2502_11618_b200 import _lib, build_grid

    lib = _lib.load()
    cloud = random_cloud(rng, 5_000, extent=4.0, offset=-2.0)
    scene = build_grid(cloud, 1.0).scene()
    cam = random_view(rng, cloud, width=32, height=32)
    cams = (_lib.LsCamera * 9)(*[_lib.make_camera(cam)] * 9)
    mz = torch.empty((9, 32 * 32), dtype=torch.int64, device="cuda")
    acc = torch.zeros((9, 32 * 32, 4), dtype=torch.float32, device="cuda")
    st = _lib.stream_ptr()
    for n in (0, 9):
        assert lib.ls_frame_project_views(scene.struct, None, 0, None, None, None, cams, n, 0.01,
                                          mz.data_ptr(), None, acc.data_ptr(), st) == _lib.LS_EINVAL
    bad = (_lib.LsCamera * 2)(_lib.make_camera(cam), _lib.make_camera(cam))
    bad[1].width = 31
    assert lib.ls_frame_project_views(scene.struct, None, 0, None, None, None, bad, 2, 0.01,
                                      mz.data_ptr(), None, acc.data_ptr(), st) == _lib.LS_EINVAL
    bits, lst, status, cnt = scene.view_buffers()
    # bits_stride shorter than ceil(n_occ / 32)
    assert lib.ls_tile_worklist_views(scene.struct, bits.data_ptr(), 0, 2, lst.data_ptr(),
                                      status.data_ptr(), cnt.data_ptr(), st) == _lib.LS_EINVAL
