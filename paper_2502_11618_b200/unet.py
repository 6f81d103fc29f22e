"""U-Net RGBDA -> RGB reconstruction on B200 tensor cores.

Architecture, parameter names, initialisation and weights-file format follow
the reference frontend (FE = /root/reference/pkg/frontend/src):
  graph            FE:model/unet.ts:148-184 (encoder conv-BN-ReLU x2 + 2x2 max
                   pool, bottleneck, decoder 2x2 transposed conv + [up, skip]
                   concat + conv-leaky(0.1) x2, 1x1 conv + sigmoid)
  init             FE:model/unet.ts:58-132 (He-normal from mulberry32 child
                   streams seeded by an FNV-1a hash of the layer name; zero
                   bias; BN gamma 1, beta 0, mean 0, var 1)
  BN epsilon       FE:model/grad64.ts:247 (1e-3), inference mode
  weights file     FE:model/weights.ts:24-79 ("lidarsplat-unet-1", base64 LE f32)
  input packing    FE:bridge.ts:31-53 + weights.ts:90-95 (done by the frame
                   kernels, see ls_frame_finish)

Device form: every conv is one implicit-GEMM tcgen05 launch (csrc/unet.cu)
with BatchNorm folded into a per-channel f32 scale/shift applied in the
epilogue; channels are zero-padded to multiples of 16; bf16 activations, f32
accumulation.  A forward pass is 5*depth+2 launches on one stream, planned
once per resolution (TMA descriptors encoded at plan time).
"""

from __future__ import annotations

import base64
import os
import json
import math
from dataclasses import asdict, dataclass

import numpy as np

from . import _lib

BN_EPSILON = 1e-3
DECODER_LEAK = 0.1
FORMAT = "lidarsplat-unet-1"


@dataclass(frozen=True)
class UNetConfig:
    inChannels: int = 5
    outChannels: int = 3
    depth: int = 4
    baseWidth: int = 32
    depthZNear: float = 0.1


DEFAULT_CONFIG = UNetConfig()
REDUCED_CONFIG = UNetConfig(depth=2, baseWidth=8)  # FE:tests/unet.test.ts:9


def stage_width(cfg: UNetConfig, stage: int) -> int:
    return cfg.baseWidth * 2 ** stage


# ---------------------------------------------------------------- init ------
class Rng:
    """mulberry32 + Box-Muller, FE:rng.ts:1-39 (32-bit integer arithmetic)."""

    def __init__(self, seed: int):
        self.state = seed & 0xFFFFFFFF

    def next(self) -> float:
        self.state = (self.state + 0x6D2B79F5) & 0xFFFFFFFF
        t = self.state
        t = _imul(t ^ (t >> 15), t | 1)
        t ^= (t + _imul(t ^ (t >> 7), t | 61)) & 0xFFFFFFFF
        return ((t ^ (t >> 14)) & 0xFFFFFFFF) / 4294967296.0

    def normal(self) -> float:
        u = 0.0
        while u == 0.0:
            u = self.next()
        v = self.next()
        return math.sqrt(-2.0 * math.log(u)) * math.cos(2.0 * math.pi * v)

    def child(self, tag: int) -> "Rng":
        return Rng(self.state ^ _imul((tag + 0x9E3779B9) & 0xFFFFFFFF, 0x85EBCA6B))


def _imul(a: int, b: int) -> int:
    return (a * b) & 0xFFFFFFFF


def _fnv1a(s: str) -> int:
    h = 2166136261
    for ch in s:
        h ^= ord(ch)
        h = _imul(h, 16777619)
    return h


def _uniforms(state: int, n: int) -> np.ndarray:
    """The next n mulberry32 draws of a stream in closed form: the state
    advances by a constant, so every draw is independent given its index."""
    k = np.arange(1, n + 1, dtype=np.uint64)
    t = (np.uint64(state) + k * np.uint64(0x6D2B79F5)) & np.uint64(0xFFFFFFFF)
    m32 = np.uint64(0xFFFFFFFF)
    t = ((t ^ (t >> np.uint64(15))) * (t | np.uint64(1))) & m32
    t = t ^ ((t + (((t ^ (t >> np.uint64(7))) * (t | np.uint64(61))) & m32)) & m32)
    return ((t ^ (t >> np.uint64(14))) & m32).astype(np.float64) / 4294967296.0


def _he(rng: Rng, shape, fan_in: int) -> np.ndarray:
    """He-normal tensor from one child stream (unet.ts:58-63), vectorised;
    falls back to the scalar generator in the 2^-32 case u == 0."""
    std = math.sqrt(2.0 / fan_in)
    n = int(np.prod(shape))
    u = _uniforms(rng.state, 2 * n)
    if (u[0::2] == 0.0).any():
        vals = np.array([rng.normal() for _ in range(n)], np.float64)
    else:
        vals = np.sqrt(-2.0 * np.log(u[0::2])) * np.cos(2.0 * np.pi * u[1::2])
    return (vals * std).reshape(shape)


def init_params(cfg: UNetConfig, seed: int) -> dict:
    """Fresh seeded parameters, tensor names as in the weights file:
    '<layer>.kernel' [kh,kw,ci,co] (transposed: [2,2,co,ci]), '<layer>.bias',
    '<bn>.gamma|beta|moving_mean|moving_var'.  f64 like the reference engine."""
    rng = Rng(seed)
    p = {}

    def conv(name, kh, kw, ci, co):
        p[name + ".kernel"] = _he(rng.child(_fnv1a(name)), (kh, kw, ci, co), kh * kw * ci)
        p[name + ".bias"] = np.zeros(co)

    def up(name, co, ci):
        p[name + ".kernel"] = _he(rng.child(_fnv1a(name)), (2, 2, co, ci), 4 * ci)
        p[name + ".bias"] = np.zeros(co)

    def bn(name, c):
        p[name + ".gamma"], p[name + ".beta"] = np.ones(c), np.zeros(c)
        p[name + ".moving_mean"], p[name + ".moving_var"] = np.zeros(c), np.ones(c)

    ci = cfg.inChannels
    for s in range(cfg.depth):
        w = stage_width(cfg, s)
        conv(f"enc{s}_conv1", 3, 3, ci, w)
        bn(f"enc{s}_bn1", w)
        conv(f"enc{s}_conv2", 3, 3, w, w)
        bn(f"enc{s}_bn2", w)
        ci = w
    bw = stage_width(cfg, cfg.depth)
    conv("bott_conv1", 3, 3, ci, bw)
    bn("bott_bn1", bw)
    conv("bott_conv2", 3, 3, bw, bw)
    bn("bott_bn2", bw)
    cu = bw
    for s in range(cfg.depth - 1, -1, -1):
        w = stage_width(cfg, s)
        up(f"dec{s}_up", w, cu)
        conv(f"dec{s}_conv1", 3, 3, 2 * w, w)
        conv(f"dec{s}_conv2", 3, 3, w, w)
        cu = w
    conv("final_conv", 1, 1, cfg.baseWidth, cfg.outChannels)
    return p


def save_weights(path: str, cfg: UNetConfig, params: dict, seed: int = 0,
                 flavor: str = "untrained", epochs: int = 0) -> None:
    """FE:model/weights.ts:43-56."""
    tensors = {k: {"shape": list(v.shape),
                   "data": base64.b64encode(np.asarray(v, "<f4").tobytes()).decode()}
               for k, v in params.items()}
    meta = {"config": asdict(cfg), "flavor": flavor, "seed": seed, "epochsTrained": epochs,
            "lpipsBackbone": "random-conv-v1"}
    with open(path, "w") as fh:
        json.dump({"format": FORMAT, "meta": meta, "tensors": tensors}, fh)


def load_weights(path: str):
    """FE:model/weights.ts:58-79 -> (config, params, meta)."""
    with open(path) as fh:
        doc = json.load(fh)
    if doc.get("format") != FORMAT:
        raise ValueError(f"unknown weights format {doc.get('format')}")
    meta = doc["meta"]
    cfg = UNetConfig(**meta["config"])
    template = init_params_shapes(cfg)
    params = {}
    for name, shape in template.items():
        entry = doc["tensors"].get(name)
        if entry is None:
            raise ValueError(f"weights file missing tensor {name}")
        arr = np.frombuffer(base64.b64decode(entry["data"]), "<f4").astype(np.float64)
        if arr.size != int(np.prod(shape)):
            raise ValueError(f"weights tensor length {arr.size} != expected {int(np.prod(shape))}")
        params[name] = arr.reshape(shape)
    return cfg, params, meta


def init_params_shapes(cfg: UNetConfig) -> dict:
    shapes = {}
    ci = cfg.inChannels
    for s in range(cfg.depth):
        w = stage_width(cfg, s)
        for name, (a, b) in ((f"enc{s}_conv1", (ci, w)), (f"enc{s}_conv2", (w, w))):
            shapes[name + ".kernel"], shapes[name + ".bias"] = (3, 3, a, b), (b,)
        for k in (1, 2):
            for f in ("gamma", "beta", "moving_mean", "moving_var"):
                shapes[f"enc{s}_bn{k}.{f}"] = (w,)
        ci = w
    bw = stage_width(cfg, cfg.depth)
    for name, (a, b) in (("bott_conv1", (ci, bw)), ("bott_conv2", (bw, bw))):
        shapes[name + ".kernel"], shapes[name + ".bias"] = (3, 3, a, b), (b,)
    for k in (1, 2):
        for f in ("gamma", "beta", "moving_mean", "moving_var"):
            shapes[f"bott_bn{k}.{f}"] = (bw,)
    cu = bw
    for s in range(cfg.depth - 1, -1, -1):
        w = stage_width(cfg, s)
        shapes[f"dec{s}_up.kernel"], shapes[f"dec{s}_up.bias"] = (2, 2, w, cu), (w,)
        shapes[f"dec{s}_conv1.kernel"], shapes[f"dec{s}_conv1.bias"] = (3, 3, 2 * w, w), (w,)
        shapes[f"dec{s}_conv2.kernel"], shapes[f"dec{s}_conv2.bias"] = (3, 3, w, w), (w,)
        cu = w
    shapes["final_conv.kernel"], shapes["final_conv.bias"] = (1, 1, cfg.baseWidth,
                                                              cfg.outChannels), (cfg.outChannels,)
    return shapes


def unet_flops(cfg: UNetConfig, width: int, height: int) -> float:
    """Dense conv FLOPs (2 x MAC) of one forward pass at width x height."""
    px = width * height
    total = 0.0
    ci = cfg.inChannels
    for s in range(cfg.depth):
        w, n = stage_width(cfg, s), px / 4 ** s
        total += 2 * n * 9 * (ci * w + w * w)
        ci = w
    bw, n = stage_width(cfg, cfg.depth), px / 4 ** cfg.depth
    total += 2 * n * 9 * (ci * bw + bw * bw)
    cu = bw
    for s in range(cfg.depth - 1, -1, -1):
        w, n = stage_width(cfg, s), px / 4 ** s
        total += 2 * (n / 4) * 4 * cu * w + 2 * n * 9 * (2 * w * w + w * w)
        cu = w
    total += 2 * px * cfg.baseWidth * cfg.outChannels
    return total


def _pad16(c: int) -> int:
    return max(16, (c + 15) // 16 * 16)


# ------------------------------------------------------------ device net ----
class UNet:
    """Device U-Net; ``forward(x, out)`` enqueues one pass on the current stream.

    x   : bf16 (B, H, W, C) NHWC [r, g, b, d', alpha, 0...], C = in_pad (8) or 16;
          8 channels are read as the first layer's 16-wide K chunk with the
          upper half zero-filled by the TMA, so both give identical outputs
    out : f32  (B, H, W, outChannels), sigmoid output in [0, 1]
    """

    in_pad = 8

    def __init__(self, cfg: UNetConfig, params: dict, device=None):
        import torch

        self.cfg = cfg
        self.params = params
        self.device = device or _lib.device()
        self.divisor = 2 ** cfg.depth
        self.layers = self._prepare()
        self._plans = {}
        self._bufs = {}

    @classmethod
    def from_config(cls, name: str = "default", seed: int = 7, device=None):
        """Fresh untrained weights (FE:model/weights.ts:82-88 freshWeights)."""
        cfg = {"default": DEFAULT_CONFIG, "reduced": REDUCED_CONFIG}[name]
        return cls(cfg, init_params(cfg, seed), device)

    @classmethod
    def from_weights(cls, path: str, device=None):
        cfg, params, _ = load_weights(path)
        return cls(cfg, params, device)

    @property
    def launches(self) -> int:
        # unbanded; see launches_for(h, w, batch).  dec0_up runs inside dec0_conv1
        # (_upfuse) unless LS_UNET_UPFUSE=0
        return 5 * self.cfg.depth + 2 - (1 if _upfuse(1) else 0)

    def launches_for(self, h: int, w: int, batch: int = 1) -> int:
        """Conv launches of one forward at this size (full-resolution row bands
        multiply the 5 full-resolution layers' launches)."""
        nb = _full_res_bands(batch, h, w)
        if nb > 1:
            return 5 * self.cfg.depth + 2 + 5 * (nb - 1)
        return 5 * self.cfg.depth + 2 - (1 if _upfuse(nb) else 0)

    def flops(self, width: int, height: int) -> float:
        return unet_flops(self.cfg, width, height)

    # -- weight preparation: BN fold, channel padding, K-major bf16 ----------
    def _prepare(self):
        import torch

        cfg, P, dev = self.cfg, self.params, self.device
        layers = {}

        def bf16(a):
            return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev).to(torch.bfloat16)

        def f32(a):
            return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev)

        def conv(name, srcs, bn=None):
            k = P[name + ".kernel"]  # [3,3,ci,co]
            co = k.shape[3]
            co_p = _pad16(co)
            ci_p = sum(_pad16(c) for c in srcs)
            # device layout [tap = kx*3+ky][co_p][ci_p] (lidarsplat_unet.h)
            wd = np.zeros((9, co_p, ci_p))
            off_r, off_p = 0, 0
            for c in srcs:
                blk = k[:, :, off_r:off_r + c, :]  # [ky,kx,c,co]
                wd[:, :co, off_p:off_p + c] = blk.transpose(1, 0, 3, 2).reshape(9, co, c)
                off_r += c
                off_p += _pad16(c)
            scale = np.zeros(co_p)
            shift = np.zeros(co_p)
            b = P[name + ".bias"]
            if bn is not None:
                inv = P[bn + ".gamma"] / np.sqrt(P[bn + ".moving_var"] + BN_EPSILON)
                scale[:co] = inv
                shift[:co] = (b - P[bn + ".moving_mean"]) * inv + P[bn + ".beta"]
            else:
                scale[:co] = 1.0
                shift[:co] = b
            layers[name] = dict(w=bf16(wd), scale=f32(scale),
                                shift=f32(shift), cout=co_p)

        def up(name):
            k = P[name + ".kernel"]  # [2,2,co,ci]
            co, ci = k.shape[2], k.shape[3]
            co_p, ci_p = _pad16(co), _pad16(ci)
            wd = np.zeros((4, co_p, ci_p))
            wd[:, :co, :ci] = k.reshape(4, co, ci)
            shift = np.zeros((4, co_p))
            shift[:, :co] = P[name + ".bias"]
            layers[name] = dict(w=bf16(wd.reshape(4 * co_p, ci_p)), scale=f32(np.ones(4 * co_p)),
                                shift=f32(shift.ravel()), cout=co_p)

        ci = cfg.inChannels
        for s in range(cfg.depth):
            w = stage_width(cfg, s)
            conv(f"enc{s}_conv1", [ci], f"enc{s}_bn1")
            conv(f"enc{s}_conv2", [w], f"enc{s}_bn2")
            ci = w
        bw = stage_width(cfg, cfg.depth)
        conv("bott_conv1", [ci], "bott_bn1")
        conv("bott_conv2", [bw], "bott_bn2")
        for s in range(cfg.depth - 1, -1, -1):
            w = stage_width(cfg, s)
            up(f"dec{s}_up")
            conv(f"dec{s}_conv1", [w, w])
            conv(f"dec{s}_conv2", [w])
        fk = P["final_conv.kernel"][0, 0]  # [ci, co]
        hw = np.zeros((cfg.outChannels, _pad16(cfg.baseWidth)))
        hw[:, :cfg.baseWidth] = fk.T
        layers["final_conv"] = dict(w=f32(hw), b=f32(P["final_conv.bias"]))
        return layers

    # -- per-resolution buffers + plans -----------------------------------------
    def _buffers(self, batch, h, w):
        import torch

        # activations are per stream: forwards enqueued on different streams
        # (one renderer per host thread) never share intermediate buffers
        key = (_lib.stream_ptr(), batch, h, w)
        if key in self._bufs:
            return self._bufs[key]
        cfg, dev = self.cfg, self.device
        b = {}
        for s in range(cfg.depth + 1):
            hs, ws = h >> s, w >> s
            c = _pad16(stage_width(cfg, s))
            for name in ("t1", "skip", "d1", "up", "pooled", "d2"):
                b[(name, s)] = torch.empty((batch, hs, ws, c), dtype=torch.bfloat16, device=dev)
        self._bufs[key] = b
        return b

    def _plan(self, x, out):
        import torch

        batch, h, w, cin = x.shape
        if h % self.divisor or w % self.divisor:
            raise ValueError(f"input {w}x{h} not divisible by 2^depth = {self.divisor}")
        key = (_lib.stream_ptr(), x.data_ptr(), out.data_ptr(), batch, h, w)
        if key in self._plans:
            return self._plans[key]
        cfg, L, lib = self.cfg, self.layers, _lib.load()
        B = self._buffers(batch, h, w)
        plans = []
        keep = []

        def mk(src0, c0, src1, c1, hs, ws, layer, act, y=None, pool=None, transposed=False,
               head=None, rows=None):
            st = ctypes.c_int32(0)
            hw, hb, hc, ho = (None, None, 0, None) if head is None else head
            pl = lib.ls_conv_plan_create(
                src0.data_ptr(), c0, None if src1 is None else src1.data_ptr(), c1, batch, hs, ws,
                layer["w"].data_ptr(), 1 if transposed else 3, layer["cout"],
                1 if transposed else 0, layer["scale"].data_ptr(), layer["shift"].data_ptr(), act,
                DECODER_LEAK, _lib.ptr(y), None, _lib.ptr(pool), _lib.ptr(hw), _lib.ptr(hb), hc,
                _lib.ptr(ho), ctypes.byref(st))
            if not pl:
                raise RuntimeError(f"conv plan failed ({st.value})")
            plans.append(pl)
            if rows is not None:
                t = lib.ls_conv_plan_tile_rows(pl)
                hh = hs  # the plan's row grid (input rows for transposed convs)
                lo = max(rows[0] // t * t, 0)
                hi = min(-(-rows[1] // t) * t, hh)
                _lib.check(lib.ls_conv_plan_set_rows(pl, lo, hi), "conv_plan_set_rows")
            return pl

        # Optional full-resolution row bands (LS_UNET_BANDS): a producer layer
        # and its consumer run band by band so the producer's band is still in
        # L2 when the consumer reads it; halo rows are recomputed per band.
        # Off by default (measured slower, see _full_res_bands).
        nb = _full_res_bands(batch, h, w)
        edges = [min(h, (k * h // nb + 15) // 16 * 16) for k in range(nb + 1)]
        edges[-1] = h

        cur, ccur = x, cin
        for s in range(cfg.depth):
            hs, ws = h >> s, w >> s
            c = _pad16(stage_width(cfg, s))
            if s == 0 and nb > 1:
                for b0, b1 in zip(edges[:-1], edges[1:]):
                    mk(cur, ccur, None, 0, hs, ws, L["enc0_conv1"], 1, y=B[("t1", 0)],
                       rows=(b0 - 1, b1 + 1))
                    mk(B[("t1", 0)], c, None, 0, hs, ws, L["enc0_conv2"], 1, y=B[("skip", 0)],
                       pool=B[("pooled", 1)], rows=(b0, b1))
            else:
                mk(cur, ccur, None, 0, hs, ws, L[f"enc{s}_conv1"], 1, y=B[("t1", s)])
                mk(B[("t1", s)], c, None, 0, hs, ws, L[f"enc{s}_conv2"], 1, y=B[("skip", s)],
                   pool=B[("pooled", s + 1)])
            cur, ccur = B[("pooled", s + 1)], c
        d = cfg.depth
        hs, ws, cb = h >> d, w >> d, _pad16(stage_width(cfg, d))
        mk(cur, ccur, None, 0, hs, ws, L["bott_conv1"], 1, y=B[("t1", d)])
        mk(B[("t1", d)], cb, None, 0, hs, ws, L["bott_conv2"], 1, y=B[("d2", d)])
        cur, ccur = B[("d2", d)], cb
        fc = L["final_conv"]
        for s in range(cfg.depth - 1, -1, -1):
            hs, ws = h >> s, w >> s
            c = _pad16(stage_width(cfg, s))
            if s == 0 and nb > 1:
                for b0, b1 in zip(edges[:-1], edges[1:]):
                    # conv2 rows [b0, b1) read conv1 rows b0-1 .. b1 (tile-aligned by
                    # mk), conv1 rows read up rows one further, up rows 2i, 2i+1 come
                    # from input row i of the transposed conv
                    c1r = (max(b0 - 8, 0), min(b1 + 8, h))
                    mk(cur, ccur, None, 0, hs // 2, ws // 2, L["dec0_up"], 0, y=B[("up", 0)],
                       transposed=True, rows=((c1r[0] - 1) // 2, (c1r[1] + 2) // 2))
                    mk(B[("up", 0)], c, B[("skip", 0)], c, hs, ws, L["dec0_conv1"], 2,
                       y=B[("d1", 0)], rows=c1r)
                    mk(B[("d1", 0)], c, None, 0, hs, ws, L["dec0_conv2"], 2,
                       head=(fc["w"], fc["b"], cfg.outChannels, out), rows=(b0, b1))
                continue
            if s == 0 and _upfuse(nb) and c == 32 and ccur == 64:
                # dec0_up computed per tile inside dec0_conv1 (the up tensor is
                # never materialised; results identical)
                st = ctypes.c_int32(0)
                lu, l1 = L["dec0_up"], L["dec0_conv1"]
                pl = lib.ls_conv_plan_create_upfused(
                    cur.data_ptr(), lu["w"].data_ptr(), lu["shift"].data_ptr(),
                    B[("skip", 0)].data_ptr(), batch, hs, ws, l1["w"].data_ptr(),
                    l1["scale"].data_ptr(), l1["shift"].data_ptr(), 2, DECODER_LEAK,
                    B[("d1", 0)].data_ptr(), ctypes.byref(st))
                if not pl:
                    raise RuntimeError(f"fused up/conv plan failed ({st.value})")
                plans.append(pl)
            else:
                mk(cur, ccur, None, 0, hs // 2, ws // 2, L[f"dec{s}_up"], 0, y=B[("up", s)],
                   transposed=True)
                mk(B[("up", s)], c, B[("skip", s)], c, hs, ws, L[f"dec{s}_conv1"], 2,
                   y=B[("d1", s)])
            if s > 0:
                mk(B[("d1", s)], c, None, 0, hs, ws, L[f"dec{s}_conv2"], 2, y=B[("d2", s)])
            else:
                mk(B[("d1", s)], c, None, 0, hs, ws, L[f"dec{s}_conv2"], 2,
                   head=(fc["w"], fc["b"], cfg.outChannels, out))
            cur, ccur = B[("d2", s)], c
        if nb == 1 and os.environ.get("LS_UNET_ALTERNATE", "1") != "0":
            # consecutive layers walk their tiles in opposite directions, so each
            # layer starts on the rows its producer wrote last (still in L2)
            for i, pl in enumerate(plans):
                if i % 2:
                    _lib.check(lib.ls_conv_plan_set_reverse(pl, 1), "conv_plan_set_reverse")
        entry = _Plans(lib, plans)
        self._plans[key] = entry
        return entry

    def forward(self, x, out):
        """Enqueue the whole network on the current stream (no host sync)."""
        self._plan(x, out).launch(_lib.stream_ptr())
        return out


import ctypes  # noqa: E402  (used by the plan helpers above)


def _upfuse(nb: int) -> bool:
    """dec0_up fused into dec0_conv1 (LS_UNET_UPFUSE=0: two launches; row
    bands keep the unfused pair)."""
    return nb == 1 and os.environ.get("LS_UNET_UPFUSE", "1") != "0"


def _full_res_bands(batch: int, h: int, w: int) -> int:
    """Row bands of the full-resolution layers (LS_UNET_BANDS, default 1 = off).
    Measured at 1920x1088 (profiles/README.md): 1 band 0.881 ms, 2 bands 0.897,
    4 bands 0.936, 8 bands 1.027 -- the per-band launch tails and halo
    recompute cost more than the L2 residency of the band saves."""
    import os

    nb = max(1, int(os.environ.get("LS_UNET_BANDS", "1")))
    while nb > 1 and h // nb < 64:  # bands of at least 64 rows
        nb //= 2
    return nb


class _Plans:
    def __init__(self, lib, plans):
        self.lib, self.plans = lib, plans

    def launch(self, stream):
        for pl in self.plans:
            _lib.check(self.lib.ls_conv_plan_launch(pl, stream), "conv_plan_launch")

    def __del__(self):
        try:
            for pl in self.plans:
                self.lib.ls_conv_plan_destroy(pl)
        except Exception:  # noqa: BLE001  (interpreter shutdown)
            pass
