"""U-Net on tcgen05 tensor cores vs the CPU restatement of the reference
graph (oracle/unet_ref.py, f64 = the reference engine FE:model/grad64.ts).

U-Net parity is tolerance-based and UNPINNED (no node/tfjs here, no golden
vectors).  Stated tolerances: per-layer f32 accumulation error
<= 1e-4 relative; full network vs f64 oracle max-abs <= 1.5e-2 and PSNR >= 40 dB,
and no worse than 2x the error floor of a plain PyTorch bf16 forward of the
same weights."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LAYER_CASES = [
    dict(c0=64, c1=0, cout=64, h=32, w=64, act=0),
    dict(c0=16, c1=0, cout=32, h=64, w=128, act=1),
    dict(c0=8, c1=0, cout=32, h=64, w=128, act=1),
    dict(c0=32, c1=0, cout=32, h=64, w=128, act=1, pool=True),
    dict(c0=32, c1=32, cout=32, h=64, w=128, act=2, head=True),
    dict(c0=128, c1=128, cout=128, h=16, w=32, act=2),
    dict(c0=256, c1=0, cout=512, h=8, w=24, act=1),
    dict(c0=64, c1=0, cout=64, h=20, w=120, act=1, pool=True),
    dict(c0=64, c1=0, cout=16, h=16, w=16, act=0, batch=2),
    dict(c0=512, c1=0, cout=512, h=4, w=8, act=1),
    # k_conv_px2 (pixel pairs): ragged tiles (50 pairs = 3.6 tiles of 14), rows
    # not a multiple of 8, batches, pool and head epilogues
    dict(c0=32, c1=0, cout=32, h=20, w=100, act=2, batch=2),
    dict(c0=32, c1=32, cout=32, h=13, w=60, act=1),  # two sources: k_conv_kx
    dict(c0=32, c1=0, cout=32, h=10, w=36, act=1, pool=True, batch=3),
    dict(c0=32, c1=0, cout=32, h=18, w=58, act=2, head=True),
    # odd width: k_conv_px2 does not apply (falls back to k_conv_kx)
    dict(c0=32, c1=0, cout=32, h=9, w=31, act=1),
    # CTA pairs (>= 128 output columns): resident half-weights, ragged pair
    # tiles (rows not a multiple of 16), pooling, batches, 256-column tiles
    dict(c0=64, c1=0, cout=128, h=20, w=40, act=1),
    dict(c0=128, c1=0, cout=128, h=24, w=48, act=1, pool=True, batch=2),
    dict(c0=128, c1=0, cout=256, h=17, w=30, act=2),
    dict(c0=256, c1=0, cout=256, h=16, w=32, act=1, pool=True),
    dict(c0=64, c1=0, cout=512, h=96, w=128, act=1),  # 256-column pair tiles
    # k_conv_kx (cout = 64, K >= 128): two sources, ragged rows
    dict(c0=64, c1=64, cout=64, h=20, w=36, act=2),
    dict(c0=128, c1=0, cout=64, h=16, w=30, act=1, pool=True, batch=2),
    # 64-channel KX2 pixel pairs (32 / 64 inputs): ragged tiles (50 pairs), rows
    # not a multiple of 8, pool, batches; odd width falls back to k_conv_p
    dict(c0=32, c1=0, cout=64, h=20, w=100, act=1, batch=2),
    dict(c0=64, c1=0, cout=64, h=18, w=58, act=2),
    dict(c0=64, c1=0, cout=64, h=10, w=36, act=1, pool=True, batch=3),
    dict(c0=64, c1=0, cout=64, h=9, w=31, act=1),
]


@pytest.fixture(autouse=True)
def _gpu(cuda_ready):
    return cuda_ready


@pytest.mark.parametrize("case", LAYER_CASES, ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
def test_conv_layer_vs_torch(case):
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "scripts"))
    from check_conv import conv_case

    out = conv_case(**case)
    assert out["rel_err_f32"] <= 1e-4
    if "pool_eq" in out:
        assert out["pool_eq"]
    if "head_err" in out:
        assert out["head_err"] <= 1e-5


# 32-channel pixel-pair layers store through per-warp staging buffers and TMA
# when no f32 copy of the output is requested: bf16 outputs (and pool / head
# outputs) equal the lane-store path's bit for bit -- ragged pair tiles, rows
# not a multiple of 8, batches, the 8-channel input form
@pytest.mark.parametrize("case", [
    dict(c0=32, c1=0, cout=32, h=20, w=100, act=2, batch=2),
    dict(c0=32, c1=0, cout=32, h=10, w=36, act=1, pool=True, batch=3),
    dict(c0=32, c1=0, cout=32, h=18, w=58, act=2, head=True),
    dict(c0=8, c1=0, cout=32, h=64, w=128, act=1),
    dict(c0=8, c1=0, cout=32, h=13, w=58, act=1, batch=2),
    dict(c0=32, c1=0, cout=32, h=136, w=240, act=1, pool=True),
], ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
def test_staged_pair_stores_bit_identical(case):
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "scripts"))
    from check_conv import conv_case

    import torch

    staged = conv_case(**case, f32_out=False)  # default: two staging buffers per warp
    old = os.environ.get("LS_PX_STAGE")
    try:
        for mode in ("1", "0"):  # one staging buffer per warp; lane stores
            os.environ["LS_PX_STAGE"] = mode  # read at plan creation
            other = conv_case(**case, f32_out=False)
            for k in ("y", "pool", "head"):
                if staged[k] is not None:
                    assert torch.equal(staged[k], other[k]), (mode, k)
    finally:
        if old is None:
            os.environ.pop("LS_PX_STAGE", None)
        else:
            os.environ["LS_PX_STAGE"] = old


# (cin, cout, h, w[, batch]): 32- and 64-channel outputs take the staged TMA
# store (64: one output-row parity per n-tile), ragged rows, batches (64 with
# ragged rows and batch > 1: lane stores)
@pytest.mark.parametrize("shape", [(512, 256, 8, 16), (64, 32, 32, 64), (128, 64, 16, 40),
                                   (128, 64, 13, 40), (128, 64, 16, 24, 2), (128, 64, 13, 24, 2),
                                   (64, 32, 13, 24, 2)])
def test_conv_transpose_vs_torch(shape):
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "scripts"))
    from check_conv import convT_case

    out = convT_case(*shape[:4], batch=shape[4] if len(shape) > 4 else 1)
    assert out["bf16_err"] <= 2 ** -7 * max(out["ref_max"], 1.0)


def _input(rng, h, w):
    """A plausible filtered RGBDA frame packed as the bridge does."""
    from oracle.unet_ref import pack_input

    rgb = rng.random((h, w, 3)).astype(np.float32)
    depth = np.where(rng.random((h, w)) < 0.7, rng.uniform(0.5, 20, (h, w)), 0).astype(np.float32)
    rgb[depth == 0] = 0
    return pack_input(rgb, depth, (depth > 0).astype(np.uint8), 0.1, 16)


def _run_device(net, x, cpad=16):
    import torch

    dev = torch.device("cuda")
    b, h, w, _ = x.shape
    xin = torch.zeros((b, h, w, cpad), dtype=torch.bfloat16, device=dev)
    xin[..., :5] = torch.from_numpy(x).to(dev).to(torch.bfloat16)
    out = torch.empty((b, h, w, net.cfg.outChannels), dtype=torch.float32, device=dev)
    net.forward(xin, out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _psnr(a, b):
    mse = float(np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2))
    return 99.0 if mse == 0 else min(99.0, 10 * math.log10(1.0 / mse))


@pytest.mark.parametrize("name,h,w", [("default", 128, 192), ("reduced", 64, 96),
                                      ("default", 272, 480)])
def test_unet_vs_f64_oracle(name, h, w):
    import torch

    from oracle.unet_ref import forward
    from paper_2502_11618_b200.unet import UNet

    net = UNet.from_config(name, seed=21)
    x = _input(np.random.default_rng(h + w), h, w)
    got = _run_device(net, x)
    ref = forward(net.cfg, net.params, x).numpy()
    # error floor: the same graph as a plain PyTorch bf16 forward on the GPU
    floor_out = forward(net.cfg, net.params, torch.from_numpy(x), dtype=torch.bfloat16,
                        device=torch.device("cuda")).float().cpu().numpy()
    err = float(np.abs(got - ref).max())
    floor = float(np.abs(floor_out - ref).max())
    print(f"{name} {h}x{w}: max-abs {err:.3e} (bf16 torch floor {floor:.3e}), "
          f"PSNR {_psnr(got, ref):.1f} dB")
    assert got.shape == (1, h, w, 3)
    assert (got >= 0).all() and (got <= 1).all()
    assert err <= 1.5e-2
    assert _psnr(got, ref) >= 40.0
    assert err <= 2 * max(floor, 1e-3)


def test_eight_channel_input_matches_sixteen():
    """The engine's 8-channel input (first layer on pixel pairs, k_conv_px2 C8)
    and the 16-channel layout (k_conv_kx, TMA zero-fills channels 8..15) are two
    kernels for the same layer: outputs agree within the U-Net tolerance."""
    from paper_2502_11618_b200.unet import UNet

    net = UNet.from_config("default", seed=5)
    x = _input(np.random.default_rng(3), 64, 96)
    a, b = _run_device(net, x, 8), _run_device(net, x, 16)
    assert np.abs(a - b).max() <= 5e-3


def test_divisibility_rejected():
    import torch

    from paper_2502_11618_b200.unet import UNet

    net = UNet.from_config("reduced", seed=1)
    xin = torch.zeros((1, 102, 100, 16), dtype=torch.bfloat16, device="cuda")
    out = torch.empty((1, 102, 100, 3), dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError, match="divisible"):
        net.forward(xin, out)


def test_translation_covariance_reduced():
    """FE:tests/unet.test.ts:45-78 on the device network: shifting the input
    by 2^depth px shifts the interior output (tolerance widened from 1e-4 to
    the bf16 activation precision)."""
    from paper_2502_11618_b200.unet import UNet

    net = UNet.from_config("reduced", seed=5)
    rng = np.random.default_rng(9)
    h = w = 64
    shift = 4
    base = rng.random((1, h, w, 5)).astype(np.float32)
    shifted = np.roll(base, shift, axis=2)
    a = _run_device(net, base)
    b = _run_device(net, shifted)
    m = 24
    diff = np.abs(a[0, m:h - m, m:w - m - shift] - b[0, m:h - m, m + shift:w - m])
    assert diff.max() <= 1e-6


def test_weights_file_roundtrip(tmp_path):
    from paper_2502_11618_b200.unet import (REDUCED_CONFIG, UNet, init_params, load_weights,
                                            save_weights)

    p = init_params(REDUCED_CONFIG, 3)
    path = str(tmp_path / "w.json")
    save_weights(path, REDUCED_CONFIG, p, seed=3)
    cfg, q, meta = load_weights(path)
    assert cfg == REDUCED_CONFIG and meta["flavor"] == "untrained"
    for k in p:
        assert np.array_equal(q[k], p[k].astype(np.float32).astype(np.float64))
    x = _input(np.random.default_rng(0), 64, 64)
    a = _run_device(UNet(cfg, q), x)
    b = _run_device(UNet.from_weights(path), x)
    assert np.array_equal(a, b)


def test_full_frame_with_unet_vs_oracle(port):
    """FrameRenderer (cull -> project -> filter -> pack -> U-Net on device)
    vs the CPU oracle pipeline + f64 U-Net restatement, 320x256 frame."""
    import torch

    from oracle import oracle as O
    from oracle.unet_ref import forward, pack_input
    from paper_2502_11618_b200 import CameraModel, PointCloud, RigidTransform, build_grid
    from paper_2502_11618_b200.engine import FrameRenderer
    from paper_2502_11618_b200.unet import UNet

    rng = np.random.default_rng(17)
    n = 300_000
    pos = rng.random((n, 3)) * np.array([8.0, 6.0, 3.0]) + np.array([-4.0, -3.0, 4.0])
    cloud = PointCloud(pos.astype(np.float32), rng.integers(0, 256, (n, 3), dtype=np.uint8))
    cam = CameraModel(fx=300.0, fy=300.0, cx=160.0, cy=120.0, width=320, height=240,
                      world_to_camera=RigidTransform.identity())
    net = UNet.from_config("default", seed=3)
    r = FrameRenderer(build_grid(cloud, 1.0), 320, 240, unet=net)
    got = r.render(cam)
    r.check_flags()
    og = O.OracleGrid(cloud.positions, cloud.colors, 1.0, port)
    rgb, depth, alpha, _ = O.render_frame(og, cam, 0.01, 4, 0.1, 0.25, port, port)
    # the device path's filtered frame is bit-exact; the U-Net within tolerance
    assert np.array_equal(r.frgb.cpu().numpy(), rgb)
    ref = forward(net.cfg, net.params, pack_input(rgb, depth, alpha, 0.1, 16)).numpy()[0, :240]
    assert got.shape == (240, 320, 3)
    err = float(np.abs(got - ref).max())
    print(f"frame+unet max-abs {err:.3e} PSNR {_psnr(got, ref):.1f} dB")
    assert err <= 1.5e-2 and _psnr(got, ref) >= 40.0


def test_full_res_row_bands_identical(monkeypatch):
    """LS_UNET_BANDS: the full-resolution layers run band by band
    (ls_conv_plan_set_rows, halo rows recomputed per band) -- the same kernels
    on the same pixels, so the output is bit-identical to the unbanded run."""
    from paper_2502_11618_b200.unet import UNet

    x = _input(np.random.default_rng(8), 256, 160)
    monkeypatch.setenv("LS_UNET_BANDS", "1")
    a = _run_device(UNet.from_config("default", seed=6), x, 8)
    monkeypatch.setenv("LS_UNET_BANDS", "4")
    net = UNet.from_config("default", seed=6)
    b = _run_device(net, x, 8)
    assert net.launches_for(256, 160) == 5 * net.cfg.depth + 2 + 15  # bands keep dec0_up apart
    assert np.array_equal(a, b)


def test_conv_plan_set_rows_validation():
    """ls_conv_plan_set_rows rejects bands that do not start on a tile row or
    leave the layer; a valid band restricts the launch to its rows."""
    import ctypes

    import torch

    from paper_2502_11618_b200 import _lib

    lib = _lib.load()
    dev = torch.device("cuda")
    h, w, c = 64, 64, 32
    x = torch.randn(1, h, w, c, device=dev).to(torch.bfloat16)
    wt = (torch.randn(9, c, c, device=dev) * 0.05).to(torch.bfloat16)
    sc, sh = torch.ones(c, device=dev), torch.zeros(c, device=dev)
    y = torch.zeros(1, h, w, c, dtype=torch.bfloat16, device=dev)
    st = ctypes.c_int32(0)
    pl = lib.ls_conv_plan_create(x.data_ptr(), c, None, 0, 1, h, w, wt.data_ptr(), 3, c, 0,
                                 sc.data_ptr(), sh.data_ptr(), 1, 0.1, y.data_ptr(), None, None,
                                 None, None, 0, None, ctypes.byref(st))
    assert pl, st.value
    try:
        t = lib.ls_conv_plan_tile_rows(pl)
        assert t > 0 and h % t == 0
        assert lib.ls_conv_plan_set_rows(pl, 1, h) == _lib.LS_EINVAL      # not on a tile row
        assert lib.ls_conv_plan_set_rows(pl, 0, h + 1) == _lib.LS_EINVAL  # past the layer
        assert lib.ls_conv_plan_set_rows(pl, t, t) == _lib.LS_EINVAL      # empty band
        assert lib.ls_conv_plan_set_rows(pl, t, 2 * t) == 0
        assert lib.ls_conv_plan_launch(pl, _lib.stream_ptr()) == 0
        torch.cuda.synchronize()
        nz = (y.float().abs().sum(dim=(0, 2, 3)) > 0).cpu().numpy()
        assert nz[t:2 * t].all() and not nz[:t].any() and not nz[2 * t:].any()
    finally:
        lib.ls_conv_plan_destroy(pl)


def test_cta_pairs_bit_identical(tmp_path):
    """CTA-pair layers (cta_group::2, M = 256) accumulate every output in the
    same K order as the single-CTA kernels: the DEFAULT network's output with
    pairs (LS_CONV_PAIR=2: every eligible layer, including the bottleneck)
    equals the LS_CONV_PAIR=0 run bit for bit.  The switch is read once per
    process, so each configuration runs in its own."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for mode in ("0", "2", "1"):
        f = tmp_path / f"o{mode}.npy"
        env = dict(os.environ, LS_CONV_PAIR=mode, H="256", W="480")
        subprocess.run([sys.executable, os.path.join(root, "scripts", "unet_out.py"), str(f)],
                       env=env, check=True, timeout=300)
        outs.append(np.load(f))
    assert outs[0].shape == (1, 256, 480, 3)
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_fused_up_conv_bit_identical(tmp_path):
    """dec0_up computed per tile inside dec0_conv1 (ls_conv_plan_create_upfused:
    the up tensor never stored) equals the two-plan path bit for bit -- the
    transposed conv's MMA, bias and bf16 rounding are the same operations, the
    zero padding of the up tensor is written explicitly.  Sizes with ragged
    pair tiles (240 / 2 = 120 pairs = 8.6 tiles) and the bench's own."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    # (the fused kernel with its staged TMA output stores, the default, and with
    # lane stores: LS_UPF_STAGE=0)
    for h, w in ((128, 240), (1088, 1920)):
        outs = []
        for mode, stage in (("0", "1"), ("1", "1"), ("1", "0")):
            f = tmp_path / f"o{mode}{stage}_{h}.npy"
            env = dict(os.environ, LS_UNET_UPFUSE=mode, LS_UPF_STAGE=stage, H=str(h), W=str(w))
            subprocess.run([sys.executable, os.path.join(root, "scripts", "unet_out.py"), str(f)],
                           env=env, check=True, timeout=300)
            outs.append(np.load(f))
        assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2]), (h, w)
    # a batch of 3 (every layer's item walk crosses images): fused == unfused,
    # and image 0 of the batch == the single-image run of the same input
    outs = []
    for mode in ("0", "1"):
        f = tmp_path / f"b{mode}.npy"
        env = dict(os.environ, LS_UNET_UPFUSE=mode, H="128", W="240", B="3")
        subprocess.run([sys.executable, os.path.join(root, "scripts", "unet_out.py"), str(f)],
                       env=env, check=True, timeout=300)
        outs.append(np.load(f))
    assert outs[0].shape == (3, 128, 240, 3)
    assert np.array_equal(outs[0], outs[1])
    f = tmp_path / "single.npy"  # the first draws of the seeded generator: image 0's input
    subprocess.run([sys.executable, os.path.join(root, "scripts", "unet_out.py"), str(f)],
                   env=dict(os.environ, H="128", W="240", B="1"), check=True, timeout=300)
    assert np.array_equal(np.load(f)[0], outs[1][0])
