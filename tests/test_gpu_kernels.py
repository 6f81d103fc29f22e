"""CUDA backend twins vs the reference's golden per-kernel outputs and vs the
CPU oracle on fresh random inputs -- the B200 analogue of the reference's
native-vs-numpy parity suite (pkg/tests/test_kernels_parity.py:28-118).
Bit-exact throughout."""

import numpy as np
import pytest

from conftest import golden, plain_camera, random_cloud, random_view
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cu(cuda_ready):
    from paper_2502_11618_b200._kernels import get_backend

    return get_backend("cuda")


@pytest.fixture(scope="module")
def kg():
    return golden("kernels.npz")


def _sparse(rng, h, w, fill=0.5):
    img = np.full((h, w), np.inf, np.float32)
    m = rng.random((h, w)) < fill
    img[m] = rng.uniform(0.3, 25.0, size=int(m.sum())).astype(np.float32)
    return img


def test_assign_cells_and_sort_golden(cu, kg):
    ids = cu.assign_cells(kg["assign_pos"], kg["assign_origin"], float(kg["assign_cell"]),
                          kg["assign_dims"])
    assert np.array_equal(ids, kg["assign_ids"])
    off, order = cu.counting_sort(kg["sort_ids"], 50)
    assert np.array_equal(off, kg["sort_offsets"])
    assert np.array_equal(order, kg["sort_order"])


def test_counting_sort_stable_large(cu, port):
    rng = np.random.default_rng(7)
    for n_cells in (1, 37, 5000, 1 << 20):
        ids = rng.integers(0, n_cells, size=200_003).astype(np.int64)
        a = cu.counting_sort(ids, n_cells)
        b = port.counting_sort(ids, n_cells)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_assign_cells_random(cu, port, rng):
    cloud = random_cloud(rng, 100_000, extent=9.7, offset=-3.3)
    origin = cloud.positions.min(axis=0).astype(np.float64)
    dims = np.array([7, 9, 11], np.int64)
    assert np.array_equal(cu.assign_cells(cloud.positions, origin, 1.37, dims),
                          port.assign_cells(cloud.positions, origin, 1.37, dims))


@pytest.mark.parametrize("s", range(3))
def test_projection_passes_golden(cu, kg, s):
    p = f"proj{s}_"
    rot, t, fx, fy, cx, cy, w, h, zn, zf = O.cam_tuple(plain_camera(kg, p))
    starts, ends = kg[p + "starts"], kg[p + "ends"]
    n = int((ends - starts).sum())
    minz, pix, z = np.full(h * w, np.inf), np.empty(n, np.int64), np.empty(n)
    cu.project_min_depth(kg[p + "pos"], starts, ends, rot, t, fx, fy, cx, cy, w, h, zn, zf,
                         minz, pix, z)
    acc = np.zeros((h * w, 4), np.uint64)
    cu.project_accumulate(kg[p + "col"], starts, ends, pix, z, 0.01, minz, acc)
    assert np.array_equal(minz, kg[p + "minz"])
    assert np.array_equal(pix, kg[p + "pix"])
    assert np.array_equal(z, kg[p + "z"])
    assert np.array_equal(acc, kg[p + "accum"])


def test_projection_passes_random(cu, port, rng):
    for _ in range(4):
        cloud = random_cloud(rng, 60_000, extent=10.0, offset=-5.0)
        cam = random_view(rng, cloud, width=320, height=240, fx=200.0, fy=200.0)
        rot, t, fx, fy, cx, cy, w, h, zn, zf = O.cam_tuple(cam)
        starts = np.array([0, 5_000, 5_000, 12_345], np.int64)
        ends = np.array([5_000, 5_000, 12_345, cloud.count], np.int64)
        n = int((ends - starts).sum())
        outs = []
        for k in (cu, port):
            minz, pix, z = np.full(h * w, np.inf), np.empty(n, np.int64), np.empty(n)
            k.project_min_depth(cloud.positions, starts, ends, rot, t, fx, fy, cx, cy, w, h,
                                zn, zf, minz, pix, z)
            acc = np.zeros((h * w, 4), np.uint64)
            k.project_accumulate(cloud.colors, starts, ends, pix, z, 0.01, minz, acc)
            outs.append((minz, pix, z, acc))
        for a, b in zip(*outs):
            assert np.array_equal(a, b)


def test_filter_kernels_golden(cu, kg):
    for j in range(6):
        assert np.array_equal(cu.min_pool_2x2(kg[f"pool{j}_in"]), kg[f"pool{j}_out"])
    for j in range(8):
        assert np.array_equal(cu.laplacian_edges(kg[f"lap{j}_in"], float(kg[f"lap{j}_thr"])),
                              kg[f"lap{j}_out"])
        assert np.array_equal(
            cu.filter_keep(kg[f"keep{j}_coarse"], kg[f"keep{j}_edges"], kg[f"keep{j}_fine"],
                           float(kg[f"keep{j}_fs"])), kg[f"keep{j}_out"])
        assert np.array_equal(cu.bilinear_fill(kg[f"fill{j}_coarse"], kg[f"fill{j}_fine"]),
                              kg[f"fill{j}_out"])


def test_filter_kernels_random(cu, port):
    rng = np.random.default_rng(99)
    for _ in range(20):
        fh, fw = int(rng.integers(1, 300)), int(rng.integers(1, 300))
        fine = _sparse(rng, fh, fw, fill=float(rng.uniform(0.05, 0.95)))
        coarse = _sparse(rng, (fh + 1) // 2, (fw + 1) // 2, fill=0.7)
        thr, fs = float(rng.uniform(0.01, 1.0)), float(rng.uniform(0.0, 2.0))
        assert np.array_equal(cu.min_pool_2x2(fine), port.min_pool_2x2(fine))
        e1, e2 = cu.laplacian_edges(coarse, thr), port.laplacian_edges(coarse, thr)
        assert np.array_equal(e1, e2)
        assert np.array_equal(cu.filter_keep(coarse, e1, fine, fs),
                              port.filter_keep(coarse, e1, fine, fs))
        assert np.array_equal(cu.bilinear_fill(coarse, fine), port.bilinear_fill(coarse, fine))


def test_typed_buffer_errors(cu):
    with pytest.raises(ValueError, match="dtype"):
        cu.min_pool_2x2(np.zeros((4, 4), np.float64))
    with pytest.raises(ValueError, match="contiguous"):
        cu.min_pool_2x2(np.zeros((4, 8), np.float32)[:, ::2])


def test_counting_sort_hand_written_radix_edges(cu, port):
    """The hand-written stable LSD radix sort behind ls_counting_sort (no CUB):
    block boundaries (4096 keys), a single key, one hot cell holding most
    points, and a 2^31-cell grid (4 digit passes) all equal the stable
    counting sort of the oracle."""
    rng = np.random.default_rng(17)
    cases = [(np.zeros(1, np.int64), 3), (rng.integers(0, 9, size=4097), 9),
             (rng.integers(0, 300, size=8192), 300)]
    skew = rng.integers(0, 9600, size=3_000_017)
    skew[rng.random(skew.size) < 0.7] = 4242
    cases.append((skew, 9600))
    cases.append((rng.integers(0, 1 << 31, size=70_001), 1 << 31))
    for ids, n_cells in cases:
        ids = ids.astype(np.int64)
        order = np.argsort(ids, kind="stable")
        a = cu.counting_sort(ids, n_cells)
        assert np.array_equal(a[1], order), n_cells
        if n_cells <= 1 << 20:
            b = port.counting_sort(ids, n_cells)
            assert np.array_equal(a[0], b[0])


def test_morton_order_matches_stable_key_sort():
    """ls_morton_order (cell id << 30 | in-cell Morton code, hand-written
    radix sort over 44 key bits): the permutation equals numpy's stable sort
    of the same keys computed on the host."""
    import torch

    from paper_2502_11618_b200 import _lib

    rng = np.random.default_rng(23)
    n = 1_000_003
    pos = (rng.random((n, 3)) * np.array([40.0, 30.0, 8.0])).astype(np.float32)
    origin = pos.min(axis=0).astype(np.float64)
    cell = 1.0
    dims = np.maximum(np.ceil((pos.max(axis=0).astype(np.float64) - origin) / cell), 1).astype(
        np.int64)
    f = (pos.astype(np.float64) - origin) / cell
    i = np.floor(f).astype(np.int64)
    t = (f - i) * 1024.0
    q = np.where(t <= 0, 0, np.where(t >= 1023, 1023, t.astype(np.int64))).astype(np.uint64)
    ic = np.minimum(np.maximum(i, 0), dims - 1)
    cid = ((ic[:, 0] * dims[1] + ic[:, 1]) * dims[2] + ic[:, 2]).astype(np.uint64)

    def spread(v):
        out = np.zeros_like(v)
        for b in range(10):
            out |= ((v >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b)
        return out

    keys = (cid << np.uint64(30)) | spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1)) | (
        spread(q[:, 2]) << np.uint64(2))
    want = np.argsort(keys, kind="stable")
    lib = _lib.load()
    d_pos = torch.from_numpy(pos).cuda()
    ws_bytes = lib.ls_morton_order_workspace(n, int(dims.prod()))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    order = torch.empty(n, dtype=torch.int64, device="cuda")
    _lib.check(lib.ls_morton_order(d_pos.data_ptr(), n, origin.ctypes.data, cell,
                                   np.ascontiguousarray(dims).ctypes.data, order.data_ptr(),
                                   ws.data_ptr(), ws_bytes, _lib.stream_ptr()), "morton_order")
    assert np.array_equal(order.cpu().numpy(), want)
