#!/usr/bin/env python3
"""Bridge wire-format fixtures FROM THE REFERENCE ITSELF (build container only).

Imports the reference's pure-Python ``lidarsplat.io.tensor`` and
``lidarsplat.frame`` from /root/reference/pkg/src (no native build needed) and
records, for seeded inputs, the exact bytes its RawTensorFrame.write emits
(RGDA and RGB0), the planes frame_to_tensor builds from an RGBDA frame, and
the frame tensor_to_frame returns (R:io/tensor.py:76-128).

    python tests/golden/make_tensor_golden.py   ->  tests/golden/tensor.npz
"""

import io
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from lidarsplat.frame import FrameRGBDA  # noqa: E402  (the reference's)
from lidarsplat.io.tensor import (MAGIC_RGB, MAGIC_RGBDA, RawTensorFrame,  # noqa: E402
                                  frame_to_tensor, tensor_to_frame)

rng = np.random.default_rng(2502)
out = {}
rgda = rng.random((5, 7, 9)).astype(np.float32)
buf = io.BytesIO()
RawTensorFrame(MAGIC_RGBDA, rgda).write(buf)
out["rgda_planes"], out["rgda_bytes"] = rgda, np.frombuffer(buf.getvalue(), np.uint8)
rgb = rng.random((3, 4, 6)).astype(np.float32)
buf = io.BytesIO()
RawTensorFrame(MAGIC_RGB, rgb).write(buf)
out["rgb_planes"], out["rgb_bytes"] = rgb, np.frombuffer(buf.getvalue(), np.uint8)
h, w = 12, 10
depth = ((rng.random((h, w)) + 0.5) * 5).astype(np.float32)
depth[rng.random((h, w)) < 0.4] = 0.0
alpha = (depth > 0).astype(np.uint8)
frgb = rng.random((h, w, 3)).astype(np.float32) * alpha[..., None]
frame = FrameRGBDA(rgb=frgb, depth=depth, alpha=alpha)
t = frame_to_tensor(frame)
out["frame_rgb"], out["frame_depth"], out["frame_alpha"] = frgb, depth, alpha
out["frame_tensor_planes"] = t.planes
soft = t.planes.copy()
# non-binary alpha plane that still thresholds (> 0.5) to depth > 0
r = rng.random((h, w)).astype(np.float32) * 0.5
soft[4] = np.where(depth > 0, np.float32(0.5) + r + np.float32(1e-3), r)
back = tensor_to_frame(RawTensorFrame(MAGIC_RGBDA, soft))
out["soft_planes"], out["soft_alpha"] = soft, back.alpha
np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "tensor.npz"), **out)
print({k: v.shape for k, v in out.items()})
