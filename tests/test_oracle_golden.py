"""Pin the CPU oracle (oracle/) against golden vectors produced by the
reference itself (tests/golden/make_golden.py) and against the reference's
own compiled kernels (oracle/_ref) when present.  CPU only."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden, plain_camera
from oracle import oracle as O


def _kernel_sets():
    sets = [O.PortKernels()]
    ref = O.load_reference()
    if ref is not None:
        sets.append(ref)
    return sets


@pytest.fixture(scope="module", params=[0, 1], ids=["port", "reference"])
def kern(request):
    sets = _kernel_sets()
    if request.param >= len(sets):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return sets[request.param]


@pytest.fixture(scope="module")
def kg():
    return golden("kernels.npz")


def test_assign_and_sort(kern, kg):
    ids = kern.assign_cells(kg["assign_pos"], kg["assign_origin"], float(kg["assign_cell"]),
                            kg["assign_dims"])
    assert np.array_equal(ids, kg["assign_ids"])
    off, order = kern.counting_sort(kg["sort_ids"], 50)
    assert np.array_equal(off, kg["sort_offsets"])
    assert np.array_equal(order, kg["sort_order"])
    assert np.array_equal(order, np.argsort(kg["sort_ids"], kind="stable"))


@pytest.mark.parametrize("s", range(3))
def test_projection_passes(kern, kg, s):
    p = f"proj{s}_"
    cam = plain_camera(kg, p)
    rot, t, fx, fy, cx, cy, w, h, zn, zf = O.cam_tuple(cam)
    starts, ends = kg[p + "starts"], kg[p + "ends"]
    n = int((ends - starts).sum())
    minz = np.full(h * w, np.inf)
    pix = np.empty(n, np.int64)
    z = np.empty(n, np.float64)
    kern.project_min_depth(kg[p + "pos"], starts, ends, rot, t, fx, fy, cx, cy, w, h, zn, zf,
                           minz, pix, z)
    acc = np.zeros((h * w, 4), np.uint64)
    kern.project_accumulate(kg[p + "col"], starts, ends, pix, z, 0.01, minz, acc)
    assert np.array_equal(minz, kg[p + "minz"])
    assert np.array_equal(pix, kg[p + "pix"])
    assert np.array_equal(z, kg[p + "z"])
    assert np.array_equal(acc, kg[p + "accum"])


def test_filter_kernels(kern, kg):
    for j in range(6):
        assert np.array_equal(kern.min_pool_2x2(kg[f"pool{j}_in"]), kg[f"pool{j}_out"])
    for j in range(8):
        assert np.array_equal(kern.laplacian_edges(kg[f"lap{j}_in"], float(kg[f"lap{j}_thr"])),
                              kg[f"lap{j}_out"])
        out = kern.filter_keep(kg[f"keep{j}_coarse"], kg[f"keep{j}_edges"], kg[f"keep{j}_fine"],
                               float(kg[f"keep{j}_fs"]))
        assert np.array_equal(out, kg[f"keep{j}_out"])
        out = kern.bilinear_fill(kg[f"fill{j}_coarse"], kg[f"fill{j}_fine"])
        assert np.array_equal(out, kg[f"fill{j}_out"])


@pytest.mark.parametrize("s", range(5))
def test_project_matches_ref_rasterizer(kern, s):
    """Golden = reference.py:14-72 pure-Python rasterizer (eps 0.05)."""
    d = golden("project.npz")
    p = f"s{s}_"
    pos = d[p + "pos"]
    rgb, depth, alpha, _, _ = O.project(pos, d[p + "col"], np.zeros(1, np.int64),
                                        np.array([len(pos)], np.int64), plain_camera(d, p), 0.05,
                                        kern)
    assert np.array_equal(alpha, d[p + "alpha"])
    assert np.array_equal(depth, d[p + "depth"])
    assert np.array_equal(rgb, d[p + "rgb"])


def test_assemble_port_matches_numpy(port):
    rng = np.random.default_rng(5)
    minz = np.where(rng.random(500) < 0.5, rng.uniform(0.1, 50, 500), np.inf)
    acc = np.zeros((500, 4), np.uint64)
    filled = np.isfinite(minz)
    acc[filled, 3] = rng.integers(1, 1000, filled.sum())
    acc[filled, :3] = rng.integers(0, 255, (filled.sum(), 3)) * acc[filled, 3:4]
    a = port.assemble(minz, acc)
    b = O.assemble(minz, acc)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("c", range(16))
def test_filter_mask_matches_reference(kern, c):
    """Golden = reference.py:175-198 ref_depth_filter_mask."""
    d = golden("filter.npz")
    p = f"c{c}_"
    levels, fs, et = d[p + "params"]
    keep = O.filter_mask(d[p + "depth"], int(levels), fs, et, kern)
    assert np.array_equal(keep, d[p + "keep"])


@pytest.mark.parametrize("s", range(6))
def test_grid_and_cull(port, s):
    d = golden("cull.npz")
    p = f"s{s}_"
    grid = O.OracleGrid(d[p + "pos"], d[p + "col"], float(d[p + "cell"]), port)
    assert np.array_equal(grid.point_order, d[p + "order"])
    assert np.array_equal(grid.cell_offsets, d[p + "offsets"])
    cam = plain_camera(d, p)
    assert np.array_equal(O.frustum_planes(cam), d[p + "planes"])
    assert np.array_equal(O.cull_cells(grid, cam, port), d[p + "culled"])


def test_pipeline_culled_and_two_plane(kern, port):
    d = golden("pipeline.npz")
    grid = O.OracleGrid(d["a_pos"], d["a_col"], 1.0, port)
    frgb, fdepth, falpha, _ = O.render_frame(grid, plain_camera(d, "a_"), 0.01, 4, 0.1, 0.25,
                                             kern, port)
    assert np.array_equal(frgb, d["a_frgb"])
    assert np.array_equal(fdepth, d["a_fdepth"])
    assert np.array_equal(falpha, d["a_falpha"])
    pos = d["b_pos"]
    rgb, depth, alpha, _, _ = O.project(pos, d["b_col"], np.zeros(1, np.int64),
                                        np.array([len(pos)], np.int64), plain_camera(d, "b_"),
                                        0.01, kern)
    assert np.array_equal(rgb, d["b_rgb"]) and np.array_equal(depth, d["b_depth"])
    _, _, fa, _ = O.depth_filter(rgb, depth, alpha, 3, 0.5, 0.25, kern)
    assert np.array_equal(fa, d["b_falpha"])
    assert fa[d["b_checker"]].all() and not fa[~d["b_checker"]].any()


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def c1_scene():
    """C1: the reference's 1M uniform box, seed 404 (compare_backends.py:23-33)."""
    rng = np.random.default_rng(404)
    n = 1_000_000
    pts = np.empty((n, 3), np.float32)
    pts[:, 0] = rng.uniform(-2, 2, n)
    pts[:, 1] = rng.uniform(-2, 2, n)
    pts[:, 2] = rng.uniform(5, 13, n)
    cols = rng.integers(0, 256, (n, 3), dtype=np.uint8)
    return pts, cols


def test_c1_digest(port):
    with open(os.path.join(GOLDEN, "c1.json")) as fh:
        info = json.load(fh)
    pts, cols = c1_scene()
    assert _digest(pts, cols) == info["inputs"]
    import types

    cam = types.SimpleNamespace(fx=350.0, fy=350.0, cx=256.0, cy=256.0, width=512, height=512,
                                z_near=0.1, z_far=100.0,
                                world_to_camera=types.SimpleNamespace(rotation=np.eye(3),
                                                                      translation=np.zeros(3)))
    grid = O.OracleGrid(pts, cols, 1.0, port)
    assert _digest(grid.point_order) == info["grid_order"]
    cells = O.cull_cells(grid, cam, port)
    assert _digest(cells) == info["culled"]
    s, e = grid.cell_ranges(cells)
    rgb, depth, alpha, _, _ = O.project(grid.sorted_positions, grid.sorted_colors, s, e, cam,
                                        0.01, port)
    assert _digest(rgb, depth, alpha) == info["frame"]
    fr, fd, fa, _ = O.depth_filter(rgb, depth, alpha, 4, 0.1, 0.25, port)
    assert _digest(fr, fd, fa) == info["filtered"]


def test_threaded_oracle_matches_single(kern):
    """The reference's ThreadPoolExecutor split (render.py:121-141) is
    bit-identical to the single-worker path (never exercised by the
    reference suite)."""
    import types

    rng = np.random.default_rng(3)
    pts = (rng.random((400_000, 3)) * 10 - 5).astype(np.float32)
    cols = rng.integers(0, 256, (400_000, 3), dtype=np.uint8)
    grid = O.OracleGrid(pts, cols, 1.0, O.PortKernels())
    cam = types.SimpleNamespace(fx=300.0, fy=300.0, cx=160.0, cy=120.0, width=320, height=240,
                                z_near=0.1, z_far=100.0,
                                world_to_camera=types.SimpleNamespace(
                                    rotation=np.eye(3), translation=np.array([0.0, 0.0, 9.0])))
    s, e = grid.cell_ranges(O.cull_cells(grid, cam, O.PortKernels()))
    assert len(s) > 2
    a = O.project(grid.sorted_positions, grid.sorted_colors, s, e, cam, 0.01, kern, workers=1)
    b = O.project(grid.sorted_positions, grid.sorted_colors, s, e, cam, 0.01, kern, workers=5)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_unet_init_matches_independent_restatement():
    """paper_2502_11618_b200.unet.init_params (vectorised closed-form
    mulberry32) equals the oracle's one-draw-at-a-time restatement of
    FE:rng.ts + FE:model/unet.ts: every REDUCED tensor in full, and the first
    2048 values of every DEFAULT kernel (same seeds, names, shapes, fan-ins).
    Uniform draws are bit-equal; the normals agree to 2 ulp (numpy's SIMD
    log/cos vs libm's scalar ones -- V8's Math.log/cos, the reference's, are
    a third implementation, so the last ulp is unpinnable without node)."""
    import numpy as np

    from oracle.unet_ref import ref_kernel_values, ref_layer_shapes
    from paper_2502_11618_b200.unet import DEFAULT_CONFIG, REDUCED_CONFIG, init_params

    for cfg, seed, limit in ((REDUCED_CONFIG, 3, None), (DEFAULT_CONFIG, 7, 2048)):
        p = init_params(cfg, seed)
        layers = ref_layer_shapes(cfg)
        assert {n + ".kernel" for n, _, _ in layers} == {k for k in p if k.endswith(".kernel")}
        for name, shape, fan_in in layers:
            k = p[name + ".kernel"]
            assert k.shape == shape
            n = k.size if limit is None else min(limit, k.size)
            ref = ref_kernel_values(seed, name, fan_in, n)
            np.testing.assert_allclose(k.ravel()[:n], ref, rtol=4.5e-16, atol=0, err_msg=name)
            assert not p[name + ".bias"].any()
        for s in range(cfg.depth):
            assert (p[f"enc{s}_bn1.moving_var"] == 1).all() and (p[f"enc{s}_bn2.gamma"] == 1).all()


def test_f32_division_equals_reference_mean():
    """k_assemble_pyramid's colour mean: f32(sum / (count * 255)) in f32 IEEE
    division equals the reference's f32(f64(sum) / (f64(count) * 255.0))
    (R:render.py:146-161) for every integer sum <= 255 * count < 2^24 --
    exhaustively for counts up to 1024, and on 2e7 random pairs up to the
    fast path's bound of 65,793 points per pixel."""
    import numpy as np

    rng = np.random.default_rng(5)
    for c in range(1, 1025):
        x = np.arange(0, 255 * c + 1)
        got = np.float32(x) / np.float32(c * 255)
        ref = (x / (c * 255.0)).astype(np.float32)
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), c
    for _ in range(4):
        cnt = rng.integers(1, 65794, size=5_000_000)
        x = np.minimum((rng.random(cnt.size) * (255 * cnt + 1)).astype(np.int64), 255 * cnt)
        got = np.float32(x) / np.float32(cnt * 255)
        ref = (x.astype(np.float64) / (cnt.astype(np.float64) * 255.0)).astype(np.float32)
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
