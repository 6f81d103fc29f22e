#!/usr/bin/env python3
"""Golden fixtures for the reference API's host helpers, FROM THE REFERENCE.

Runs only in the build container (needs /root/reference; reuses
make_golden.setup_reference's scratch build imported as ``lidarsplat_ref``).
Writes tests/golden/api.json:
  all            the reference package's __all__ (R:__init__.py:36-72)
  bench_schema   R:schemas/bench_report.schema.json (the report contract)
  metrics        psnr / ssim of seeded image pairs (R:metrics.py:27-71)
  augment        sha256 of augment_brightness_contrast outputs on seeded
                 images / masks / params (R:synth.py:154-181)
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)


def metric_cases():
    """(pred, target) pairs shared with tests/test_api_extras.py."""
    rng = np.random.default_rng(2024)
    out = []
    for h, w, ch, noise in [(32, 40, 3, 0.05), (11, 11, 3, 0.2), (64, 48, 1, 0.01),
                            (24, 30, 3, 0.0), (50, 50, 3, 0.5)]:
        t = rng.random((h, w, ch)).astype(np.float32)
        p = np.clip(t + noise * rng.normal(size=t.shape), 0, 1).astype(np.float32)
        out.append((p if ch == 3 else p[:, :, 0], t if ch == 3 else t[:, :, 0]))
    return out


def augment_cases():
    rng = np.random.default_rng(77)
    out = []
    for i, (h, w) in enumerate([(48, 64), (70, 33), (128, 96)]):
        img = rng.random((h, w, 3)).astype(np.float32)
        alpha = (rng.random((h, w)) < 0.6).astype(np.uint8)
        params = dict(seed=1000 + i)
        if i == 1:
            params.update(brightness_delta_range=(0.0, 0.0), contrast_scale_range=(1.0, 1.0))
        if i == 2:
            params.update(group_count_range=(5, 9))
        out.append((img, alpha, params, None if i != 2 else (i, 3)))
    return out


def main():
    from make_golden import setup_reference

    setup_reference()
    import lidarsplat_ref as R
    from lidarsplat_ref.metrics import psnr, ssim
    from lidarsplat_ref.synth import AugmentParams, augment_brightness_contrast

    doc = {"all": list(R.__all__)}
    with open("/root/reference/pkg/src/lidarsplat/schemas/bench_report.schema.json") as fh:
        doc["bench_schema"] = json.load(fh)
    doc["metrics"] = [{"psnr": psnr(p, t), "ssim": ssim(p, t)} for p, t in metric_cases()]
    aug = []
    for img, alpha, params, spawn in augment_cases():
        ss = None if spawn is None else np.random.SeedSequence(entropy=spawn[0],
                                                               spawn_key=(spawn[1],))
        o = augment_brightness_contrast(img, alpha, AugmentParams(**params), ss)
        aug.append(hashlib.sha256(np.ascontiguousarray(o).tobytes()).hexdigest())
    doc["augment"] = aug
    with open(os.path.join(HERE, "api.json"), "w") as fh:
        json.dump(doc, fh, indent=1, sort_keys=True)
        fh.write("\n")
    print("wrote api.json")


if __name__ == "__main__":
    main()
