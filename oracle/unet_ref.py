"""CPU restatement of the reference U-Net -- TEST INFRASTRUCTURE ONLY.

Follows the reference's float64 engine op by op (FE = /root/reference/pkg/frontend/src):
  conv2d             FE:model/grad64.ts:65-141   NHWC, kernel [kh,kw,ci,co], zero "same" pad
  convTranspose2x2   FE:model/grad64.ts:146-201  kernel [2,2,co,ci], y[2i+dy,2j+dx,o] = b + sum_c x W
  maxPool2           FE:model/grad64.ts:203-238
  batchNorm (infer)  FE:model/grad64.ts:250-313  eps 1e-3 (:247)
  relu / leakyRelu / sigmoid  FE:model/grad64.ts:315-354
  concatC            FE:model/grad64.ts:357-379  [up, skip]
  graph              FE:model/unet.ts:148-184
  input prep         FE:model/weights.ts:90-95 normalizeDepth + FE:bridge.ts:31-53 NHWC pack

Runs in torch on the CPU (float64 = the reference engine, float32 = the tfjs
executor's precision).  U-Net parity is UNPINNED: the reference executors
need node + @tensorflow/tfjs (not installed), so there are no golden vectors;
correctness rests on this restatement plus the reference's relative
properties (shape, [0,1] range, translation covariance, FE:tests/unet.test.ts).
"""

from __future__ import annotations

import numpy as np

BN_EPSILON = 1e-3
DECODER_LEAK = 0.1


def _t(a, dtype, device=None):
    import torch

    if isinstance(a, torch.Tensor):
        return a.to(device=device or a.device, dtype=dtype)
    return torch.as_tensor(np.asarray(a), dtype=dtype, device=device)


def conv2d(x, k, b):
    """x NHWC, k [kh,kw,ci,co] -> NHWC (zero 'same' padding for odd k)."""
    import torch.nn.functional as F

    w = k.permute(3, 2, 0, 1)  # [co, ci, kh, kw]
    y = F.conv2d(x.permute(0, 3, 1, 2), w, b, padding=k.shape[0] // 2)
    return y.permute(0, 2, 3, 1)


def conv_transpose2x2(x, k, b):
    """k [2,2,co,ci] -> torch weight [ci, co, 2, 2]."""
    import torch.nn.functional as F

    w = k.permute(3, 2, 0, 1)
    y = F.conv_transpose2d(x.permute(0, 3, 1, 2), w, b, stride=2)
    return y.permute(0, 2, 3, 1)


def max_pool2(x):
    import torch.nn.functional as F

    return F.max_pool2d(x.permute(0, 3, 1, 2), 2).permute(0, 2, 3, 1)


def batch_norm(x, p, name):
    inv = 1.0 / (p[name + ".moving_var"] + BN_EPSILON).sqrt()
    return (x - p[name + ".moving_mean"]) * inv * p[name + ".gamma"] + p[name + ".beta"]


def forward(cfg, params, x, dtype=None, collect=None, device=None):
    """x: (B,H,W,inChannels) NHWC -> (B,H,W,outChannels) in [0,1].
    ``collect`` (dict) receives intermediate tensors by layer name.  ``device``
    lets the same restatement run as a plain-PyTorch GPU forward (used only to
    measure the bf16 error floor)."""
    import torch

    dtype = dtype or torch.float64
    p = {k: _t(v, dtype, device) for k, v in params.items()}
    x = _t(x, dtype, device)
    h, w = x.shape[1], x.shape[2]
    div = 2 ** cfg.depth
    if h % div or w % div:
        raise ValueError(f"input {w}x{h} not divisible by 2^depth = {div}")

    def keep(name, t):
        if collect is not None:
            collect[name] = t
        return t

    relu = torch.relu
    skips = []
    cur = x
    for s in range(cfg.depth):
        cur = keep(f"enc{s}_1", relu(batch_norm(conv2d(cur, p[f"enc{s}_conv1.kernel"],
                                                       p[f"enc{s}_conv1.bias"]), p, f"enc{s}_bn1")))
        cur = keep(f"enc{s}_2", relu(batch_norm(conv2d(cur, p[f"enc{s}_conv2.kernel"],
                                                       p[f"enc{s}_conv2.bias"]), p, f"enc{s}_bn2")))
        skips.append(cur)
        cur = max_pool2(cur)
    cur = keep("bott_1", relu(batch_norm(conv2d(cur, p["bott_conv1.kernel"], p["bott_conv1.bias"]),
                                         p, "bott_bn1")))
    cur = keep("bott_2", relu(batch_norm(conv2d(cur, p["bott_conv2.kernel"], p["bott_conv2.bias"]),
                                         p, "bott_bn2")))
    leaky = lambda t: torch.where(t > 0, t, DECODER_LEAK * t)  # noqa: E731
    for s in range(cfg.depth - 1, -1, -1):
        cur = keep(f"dec{s}_up", conv_transpose2x2(cur, p[f"dec{s}_up.kernel"], p[f"dec{s}_up.bias"]))
        cur = torch.cat([cur, skips[s]], dim=-1)
        cur = keep(f"dec{s}_1", leaky(conv2d(cur, p[f"dec{s}_conv1.kernel"], p[f"dec{s}_conv1.bias"])))
        cur = keep(f"dec{s}_2", leaky(conv2d(cur, p[f"dec{s}_conv2.kernel"], p[f"dec{s}_conv2.bias"])))
    return torch.sigmoid(conv2d(cur, p["final_conv.kernel"], p["final_conv.bias"]))


def pack_input(rgb, depth, alpha, z_near=0.1, pad_rows_to=16):
    """bridge.ts:31-53 + weights.ts:90-95: NHWC [r,g,b,d',a], d' = zNear/max(d,zNear)
    in f64 stored as f32; zero rows appended to a multiple of 2^depth."""
    h, w = depth.shape
    dn = np.where(depth > 0, (z_near / np.maximum(depth.astype(np.float64), z_near)), 0.0)
    x = np.concatenate([rgb.astype(np.float32), dn.astype(np.float32)[..., None],
                        alpha.astype(np.float32)[..., None]], axis=-1)
    hp = (h + pad_rows_to - 1) // pad_rows_to * pad_rows_to
    out = np.zeros((1, hp, w, 5), np.float32)
    out[0, :h] = x
    return out


class CpuUNet:
    """The CPU U-Net leg of the reference arm: f32 torch (tfjs precision) on
    all host threads, same random-init weights as the device network."""

    def __init__(self, name="default", threads=None, seed=7):
        import torch

        from paper_2502_11618_b200.unet import DEFAULT_CONFIG, REDUCED_CONFIG, init_params

        if threads:
            torch.set_num_threads(threads)
        self.cfg = {"default": DEFAULT_CONFIG, "reduced": REDUCED_CONFIG}[name]
        self.params = init_params(self.cfg, seed)

    def reconstruct(self, rgb, depth, alpha):
        import torch

        x = pack_input(rgb, depth, alpha, self.cfg.depthZNear, 2 ** self.cfg.depth)
        with torch.no_grad():
            y = forward(self.cfg, self.params, x, dtype=torch.float32)
        return y[0, : depth.shape[0]].numpy()


# ---------------------------------------------------------------------------
# Independent scalar restatement of the reference's weight init (checks the
# product's vectorised paper_2502_11618_b200.unet.init_params):
#   mulberry32 + Box-Muller + child streams   FE:rng.ts:1-39
#   FNV-1a layer-name hash                     FE:model/unet.ts:92-99
#   He-normal kernels, zero bias, BN identity  FE:model/unet.ts:58-86, 100-132
# Pure-Python integer arithmetic, one draw at a time exactly as the TS loops.
# ---------------------------------------------------------------------------

def _mul32(a, b):
    return (a * b) % 4294967296


class Mulberry32:
    def __init__(self, seed):
        self.s = seed % 4294967296

    def next(self):
        self.s = (self.s + 0x6D2B79F5) % 4294967296
        t = self.s
        t = _mul32(t ^ (t >> 15), t | 1)
        t = t ^ ((t + _mul32(t ^ (t >> 7), t | 61)) % 4294967296)
        return (t ^ (t >> 14)) / 4294967296.0

    def normal(self):
        import math

        u = 0.0
        while u == 0.0:
            u = self.next()
        v = self.next()
        return math.sqrt(-2.0 * math.log(u)) * math.cos(2.0 * math.pi * v)

    def child(self, tag):
        return Mulberry32(self.s ^ _mul32((tag + 0x9E3779B9) % 4294967296, 0x85EBCA6B))


def fnv1a(name):
    h = 2166136261
    for ch in name:
        h = _mul32(h ^ ord(ch), 16777619)
    return h


def ref_layer_shapes(cfg):
    """(name, kernel shape, fan_in) of every conv in construction order
    (FE:model/unet.ts:100-132)."""
    out = []
    ci = cfg.inChannels
    for s in range(cfg.depth):
        w = cfg.baseWidth * 2 ** s
        out += [(f"enc{s}_conv1", (3, 3, ci, w), 9 * ci), (f"enc{s}_conv2", (3, 3, w, w), 9 * w)]
        ci = w
    bw = cfg.baseWidth * 2 ** cfg.depth
    out += [("bott_conv1", (3, 3, ci, bw), 9 * ci), ("bott_conv2", (3, 3, bw, bw), 9 * bw)]
    cu = bw
    for s in range(cfg.depth - 1, -1, -1):
        w = cfg.baseWidth * 2 ** s
        out += [(f"dec{s}_up", (2, 2, w, cu), 4 * cu), (f"dec{s}_conv1", (3, 3, 2 * w, w), 18 * w),
                (f"dec{s}_conv2", (3, 3, w, w), 9 * w)]
        cu = w
    out.append(("final_conv", (1, 1, cfg.baseWidth, cfg.outChannels), cfg.baseWidth))
    return out


def ref_kernel_values(seed, name, fan_in, count):
    """The first ``count`` He-normal values (flat, row-major) of layer ``name``."""
    import math

    rng = Mulberry32(seed).child(fnv1a(name))
    std = math.sqrt(2.0 / fan_in)
    return np.array([rng.normal() * std for _ in range(count)], np.float64)
