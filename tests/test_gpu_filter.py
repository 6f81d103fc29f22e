"""Depth filter on the B200 vs the reference (ports of pkg/tests/test_filtering.py,
test_acceptance.py:115-173) and the fused per-frame path vs the oracle --
bit-exact masks and frames."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from conftest import golden, make_camera, random_cloud, random_view, two_plane_cloud
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu(cuda_ready):
    return cuda_ready


def sparse_depth(rng, h, w, fill=0.6, lo=0.5, hi=20.0):
    d = np.zeros((h, w), np.float32)
    m = rng.random((h, w)) < fill
    d[m] = rng.uniform(lo, hi, size=int(m.sum())).astype(np.float32)
    return d


@pytest.mark.parametrize("c", range(16))
def test_filter_matches_reference_golden(c):
    from lidarsplat import FilterParams, filter_depth_image

    d = golden("filter.npz")
    p = f"c{c}_"
    levels, fs, et = d[p + "params"]
    keep = filter_depth_image(d[p + "depth"], FilterParams(int(levels), float(fs), float(et)))
    assert np.array_equal(keep, d[p + "keep"])


def test_filter_random_vs_oracle(port):
    from lidarsplat import FilterParams, filter_depth_image

    rng = np.random.default_rng(31)
    for _ in range(30):
        h, w = int(rng.integers(16, 400)), int(rng.integers(16, 400))
        L = int(rng.integers(1, 5))
        depth = sparse_depth(rng, h, w, fill=float(rng.uniform(0.05, 0.95)))
        fs, et = float(rng.uniform(0, 1.5)), float(rng.uniform(0.05, 0.6))
        keep = filter_depth_image(depth, FilterParams(L, fs, et))
        assert np.array_equal(keep, O.filter_mask(depth, L, fs, et, port))


def test_pyramid_and_steps():
    from lidarsplat import FilterParams, build_min_pyramid, upsample_filter_step

    pyr = build_min_pyramid(np.array([[1.0, 3.0], [0.0, 2.0]], np.float32), 1)
    assert pyr.levels[0].shape == (1, 1) and pyr.levels[0][0, 0] == np.float32(1.0)
    pyr = build_min_pyramid(np.zeros((8, 8), np.float32), 3)
    assert all(np.isinf(l).all() for l in pyr.levels)
    coarse = np.array([[1.0]], np.float32)
    fine = np.array([[1.0, 1.05], [5.0, np.inf]], np.float32)
    out = upsample_filter_step(coarse, fine, FilterParams(filter_strength=0.1), True)
    assert out[0, 0] == np.float32(1.0) and out[0, 1] == np.float32(1.05)
    assert np.isinf(out[1, 0]) and np.isinf(out[1, 1])


def test_vertical_step_edges():
    from lidarsplat import laplacian_edges

    img = np.full((6, 8), 1.0, np.float32)
    img[:, 4:] = 5.0
    e = laplacian_edges(img, 0.25)
    assert e[:, 3].all() and e[:, 4].all() and e[:, :3].sum() == 0 and e[:, 5:].sum() == 0


def test_two_plane_leak_removal():
    from lidarsplat import FilterParams, depth_filter, project_points

    cam = make_camera()
    cloud, checker = two_plane_cloud(cam)
    fr = project_points(cloud, None, cam)
    out = depth_filter(fr, FilterParams(levels_n=3, filter_strength=0.5))
    kept = out.alpha.astype(bool)
    assert kept[checker].all() and not kept[~checker].any()
    assert np.array_equal(out.depth[kept], fr.depth[kept])
    assert np.array_equal(out.rgb[kept], fr.rgb[kept])
    out.validate()


def test_invariant_suite_acceptance():
    """test_acceptance.py:115-162: subset, global-min survival, identity at
    fs >= max/min, monotone in fs (50 random images)."""
    from lidarsplat import FilterParams, build_min_pyramid, filter_depth_image
    from lidarsplat import upsample_filter_step

    rng = np.random.default_rng(303)
    for _ in range(50):
        h, w = int(rng.integers(8, 40)), int(rng.integers(8, 40))
        L = int(rng.integers(1, 4))
        if h < 2**L or w < 2**L:
            L = 1
        depth = sparse_depth(rng, h, w, fill=float(rng.uniform(0.15, 0.9)))
        filled = depth > 0
        fs = float(rng.uniform(0.0, 1.0))
        keep = filter_depth_image(depth, FilterParams(levels_n=L, filter_strength=fs))
        assert not (keep & ~filled).any()
        if filled.any():
            dmin = depth[filled].min()
            assert keep[depth == dmin].any()
            ratio = float(depth[filled].max() / dmin)
            assert np.array_equal(
                filter_depth_image(depth, FilterParams(levels_n=L, filter_strength=ratio)),
                filled)
        fs2 = fs + float(rng.uniform(0.0, 1.0))
        pyr = build_min_pyramid(depth, 1)
        a = np.isfinite(upsample_filter_step(pyr.levels[0], pyr.levels[1],
                                             FilterParams(1, fs), True))
        b = np.isfinite(upsample_filter_step(pyr.levels[0], pyr.levels[1],
                                             FilterParams(1, fs2), True))
        assert not (a & ~b).any()


@settings(max_examples=30, deadline=None)
@given(seed=st.integers(0, 2**31), fs=st.floats(0.0, 2.0, allow_nan=False),
       levels=st.integers(1, 3))
def test_filter_properties_hypothesis(seed, fs, levels):
    from lidarsplat import FilterParams, filter_depth_image

    rng = np.random.default_rng(seed)
    depth = sparse_depth(rng, 16, 16, fill=0.5)
    keep = filter_depth_image(depth, FilterParams(levels_n=levels, filter_strength=fs))
    filled = depth > 0
    assert not (keep & ~filled).any()
    if filled.any():
        assert keep[depth == depth[filled].min()].any()


@pytest.mark.parametrize("size", [(64, 48), (333, 257), (1920, 1080)])
def test_fused_frame_path_vs_oracle(port, size):
    """cull -> pass1 -> pass2 -> assemble+pyramid -> steps -> mask + U-Net
    input, all enqueued by render.project_scene, vs the CPU oracle."""
    import torch

    from lidarsplat import CameraModel, FilterParams, build_grid
    from lidarsplat.render import FrameBuffers, project_scene

    w, h = size
    rng = np.random.default_rng(w * 7 + h)
    cloud = random_cloud(rng, 300_000, extent=10.0, offset=-5.0)
    cam0 = random_view(rng, cloud)
    cam = CameraModel.unchecked(w * 0.8, w * 0.8, w / 2.0, h / 2.0, w, h,
                                cam0.world_to_camera, 0.1, 100.0)
    grid = build_grid(cloud, 1.0)
    scene = grid.scene()
    dev = torch.device("cuda")
    bufs = FrameBuffers(w, h, dev)
    fp = FilterParams()
    frgb = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
    fdep = torch.empty((h, w), dtype=torch.float32, device=dev)
    falp = torch.empty((h, w), dtype=torch.uint8, device=dev)
    keep = torch.empty((h, w), dtype=torch.uint8, device=dev)
    uh = (h + 15) // 16 * 16
    unet_in = torch.zeros((uh, w, 16), dtype=torch.bfloat16, device=dev)
    import ctypes

    from lidarsplat import _lib

    pyr = torch.empty(_lib.load().ls_pyramid_floats(h, w, 4), dtype=torch.float32, device=dev)
    for rep in range(2):  # second frame checks the consume-and-reset of the buffers
        project_scene(scene, cam, 0.01, bufs, cull=True, filter_params=fp,
                      filtered=(frgb, fdep, falp), keep=keep, unet_in=unet_in, pyramid=pyr)
        torch.cuda.synchronize()
        assert int(bufs.flags.item()) == 0
        s, e = grid.cell_ranges(O.cull_cells(grid, cam, port))
        rgb, depth, alpha, _, _ = O.project(grid.sorted_positions, grid.sorted_colors, s, e, cam,
                                            0.01, port)
        assert np.array_equal(bufs.rgb.cpu().numpy(), rgb)
        assert np.array_equal(bufs.depth.cpu().numpy(), depth)
        assert np.array_equal(bufs.alpha.cpu().numpy(), alpha)
        r2, d2, a2, k2 = O.depth_filter(rgb, depth, alpha, 4, 0.1, 0.25, port)
        assert np.array_equal(frgb.cpu().numpy(), r2)
        assert np.array_equal(fdep.cpu().numpy(), d2)
        assert np.array_equal(falp.cpu().numpy(), a2)
        assert np.array_equal(keep.cpu().numpy().astype(bool), k2)
        # U-Net input: [r,g,b,zNear/max(d,zNear),alpha] (weights.ts:90-95) in bf16
        dn = np.where(d2 > 0, (0.1 / np.maximum(d2.astype(np.float64), 0.1)).astype(np.float32),
                      np.float32(0))
        ref = np.concatenate([r2, dn[..., None], a2[..., None].astype(np.float32)], axis=-1)
        got = unet_in[:h, :, :5].float().cpu().numpy()
        exp = torch.from_numpy(ref).to(torch.bfloat16).float().numpy()
        assert np.array_equal(got, exp)
        assert (unet_in[:h, :, 5:].float() == 0).all() and (unet_in[h:].float() == 0).all()


@pytest.mark.parametrize("levels,size,k", [(4, (333, 257), 7), (1, (40, 30), 3),
                                           (2, (64, 48), 16), (5, (200, 150), 19),
                                           (6, (130, 97), 2), (3, (3840, 2160), 7)])
def test_depth_filter_sweep_vs_oracle(port, levels, size, k):
    """filtering.depth_filter_sweep (pyramid once, all strengths batched, >16
    strengths in chunks, L > 5 on the per-strength path): every strength's
    filtered frame and keep mask equal the oracle's depth filter."""
    import torch

    from paper_2502_11618_b200 import FilterParams
    from paper_2502_11618_b200.filtering import depth_filter_sweep

    w, h = size
    rng = np.random.default_rng(levels * 100 + k)
    depth = sparse_depth(rng, h, w, fill=0.55)
    alpha = (depth > 0).astype(np.uint8)
    rgb = (rng.random((h, w, 3)) * alpha[..., None]).astype(np.float32)
    fs_list = [0.0, 0.05, 0.1, 0.25, 0.5, 1.0, 1e30][:k] + list(rng.random(max(0, k - 7)) * 0.6)
    dev = torch.device("cuda")
    t = [torch.from_numpy(a).to(dev) for a in (rgb, depth, alpha)]
    et = 0.25 if levels != 2 else 0.1
    frgb, fdep, falp, keep = depth_filter_sweep(*t, fs_list, FilterParams(levels_n=levels,
                                                                          edge_threshold=et))
    _, _, _, keep_only = depth_filter_sweep(*t, fs_list, FilterParams(levels_n=levels,
                                                                      edge_threshold=et),
                                            outputs=False)
    assert bool((keep == keep_only).all())
    picks = range(k) if max(size) < 1000 else [0, 2, 6]
    for i in picks:
        r2, d2, a2, k2 = O.depth_filter(rgb, depth, alpha, levels, fs_list[i], et, port)
        assert np.array_equal(keep[i].cpu().numpy().astype(bool), k2), f"fs={fs_list[i]}"
        assert np.array_equal(frgb[i].cpu().numpy(), r2)
        assert np.array_equal(fdep[i].cpu().numpy(), d2)
        assert np.array_equal(falp[i].cpu().numpy(), a2)
