"""Multi-rank merge of point shards, world_size 2 over gloo on the CPU.

Each rank projects its contiguous shard of the cell-major scan with the CPU
oracle kernels, then the SAME merge functions the GPU ShardedRenderer uses
(paper_2502_11618_b200.shard.merge_minz / merge_accum: all-reduce MIN of the
f64 bit patterns as int64, reduce SUM of the f32 {r,g,b,count} accumulators) combine
them; the root's frame must equal the single-process oracle frame bit for bit
(min and integer sums are order-free)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _scene():
    import types

    rng = np.random.default_rng(8)
    n = 120_000
    pos = (rng.random((n, 3)) * 10 - 5).astype(np.float32)
    col = rng.integers(0, 256, (n, 3), dtype=np.uint8)
    cam = types.SimpleNamespace(fx=200.0, fy=200.0, cx=96.0, cy=64.0, width=192, height=128,
                                z_near=0.1, z_far=100.0,
                                world_to_camera=types.SimpleNamespace(
                                    rotation=np.eye(3), translation=np.array([0.0, 0.0, 8.0])))
    return pos, col, cam


def _pack(acc4):
    """u64 x4 accumulators -> the GPU pass-2 layout, f32 {r, g, b, count}."""
    assert int(acc4.max()) < 2 ** 24
    return acc4.astype(np.float32)


def _unpack(packed):
    assert float(packed.max()) < 2 ** 24
    return packed.astype(np.uint64)


def _worker(rank, world, port, out, async_reduce=False):
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2502_11618_b200.shard import merge_accum, merge_minz, shard_bounds

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pos, col, cam = _scene()
    port_k = O.PortKernels()
    grid = O.OracleGrid(pos, col, 1.0, port_k)
    s, e = grid.cell_ranges(O.cull_cells(grid, cam, port_k))
    lo, hi = shard_bounds(len(pos), rank, world)
    ss, ee = np.clip(s, lo, hi), np.clip(e, lo, hi)
    keep = ee > ss
    ss, ee = ss[keep], ee[keep]
    rot, t, fx, fy, cx, cy, w, h, zn, zf = O.cam_tuple(cam)
    n = int((ee - ss).sum())
    minz = np.full(h * w, np.inf)
    pix, z = np.empty(n, np.int64), np.empty(n)
    port_k.project_min_depth(grid.sorted_positions, ss, ee, rot, t, fx, fy, cx, cy, w, h, zn, zf,
                             minz, pix, z)
    mz = torch.from_numpy(minz.view(np.int64).copy())
    merge_minz(mz)
    gmin = mz.numpy().view(np.float64)
    acc = np.zeros((h * w, 4), np.uint64)
    port_k.project_accumulate(grid.sorted_colors, ss, ee, pix, z, 0.01, gmin, acc)
    packed = torch.from_numpy(_pack(acc))
    root = 1  # not rank 0 on purpose (round-robin roots)
    if async_reduce:  # ShardedRenderer's form: wait on the handle later
        work = merge_accum(packed, root, async_op=True)
        work.wait()
    else:
        merge_accum(packed, root)
    if rank == root:
        rgb, depth, alpha = O.assemble(gmin, _unpack(packed.numpy()))
        ref = O.project(grid.sorted_positions, grid.sorted_colors, s, e, cam, 0.01, port_k)
        out[0] = bool(np.array_equal(rgb.reshape(h, w, 3), ref[0])
                      and np.array_equal(depth.reshape(h, w), ref[1])
                      and np.array_equal(alpha.reshape(h, w), ref[2])
                      and np.array_equal(gmin, ref[3]))
    dist.destroy_process_group()


@pytest.mark.parametrize("async_reduce", [False, True])
@pytest.mark.parametrize("world", [2])
def test_sharded_merge_matches_single_process(world, async_reduce):
    ctx = mp.get_context("spawn")
    out = ctx.Manager().list([None])
    mp.spawn(_worker, args=(world, _free_port(), out, async_reduce), nprocs=world, join=True)
    assert out[0] is True


def test_shard_bounds_partition():
    from paper_2502_11618_b200.shard import shard_bounds

    for n in (0, 1, 7, 1000, 123457):
        for world in (1, 2, 3, 8):
            b = [shard_bounds(n, r, world) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))


def test_shard_cell_offsets():
    import torch

    from paper_2502_11618_b200.shard import shard_cell_offsets

    off = torch.tensor([0, 3, 3, 10, 12, 20])
    assert shard_cell_offsets(off, 5, 12).tolist() == [0, 0, 0, 5, 7, 7]
