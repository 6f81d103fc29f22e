"""Shared fixtures.

Scene/camera helpers restate the reference suite's fixtures
(/root/reference/pkg/tests/conftest.py:7-87) so parity tests read like the
reference's own tests.  GPU tests are marked ``gpu``; they FAIL (never skip)
when no CUDA device or library is present, so a silent fallback cannot pass.
"""

from __future__ import annotations

import os
import sys
import types

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: large-scale case")


def look_at(eye, target, up=(0.0, 0.0, 1.0)):
    """world->camera pose with +z toward target (reference conftest.py:7-20)."""
    from paper_2502_11618_b200 import RigidTransform

    eye = np.asarray(eye, np.float64)
    fwd = np.asarray(target, np.float64) - eye
    fwd /= np.linalg.norm(fwd)
    down = -np.asarray(up, np.float64)
    right = np.cross(down, fwd)
    if np.linalg.norm(right) < 1e-9:
        down = np.array([0.0, 1.0, 0.0])
        right = np.cross(down, fwd)
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    rot = np.stack([right, down, fwd])
    return RigidTransform(rot, -(rot @ eye))


def make_camera(eye=(0.0, 0.0, 0.0), target=None, width=64, height=48, fx=50.0, fy=50.0,
                z_near=0.1, z_far=100.0):
    from paper_2502_11618_b200 import CameraModel, RigidTransform

    pose = (RigidTransform(np.eye(3), -np.asarray(eye, np.float64)) if target is None
            else look_at(eye, target))
    return CameraModel(fx=fx, fy=fy, cx=width / 2.0, cy=height / 2.0, width=width,
                       height=height, world_to_camera=pose, z_near=z_near, z_far=z_far)


def random_cloud(rng, n, extent=10.0, offset=0.0):
    from paper_2502_11618_b200 import PointCloud

    pos = (rng.random((n, 3)) * extent + offset).astype(np.float32)
    return PointCloud(pos, rng.integers(0, 256, size=(n, 3), dtype=np.uint8))


def random_view(rng, cloud, **kw):
    lo = cloud.positions.min(axis=0).astype(np.float64)
    hi = cloud.positions.max(axis=0).astype(np.float64)
    radius = float(np.linalg.norm(hi - lo)) / 2 + 1.0
    d = rng.normal(size=3)
    d /= np.linalg.norm(d)
    eye = (lo + hi) / 2 + d * radius * (1.0 + rng.random())
    target = lo + rng.random(3) * (hi - lo)
    return make_camera(**kw).with_pose(look_at(eye, target))


def two_plane_cloud(camera, front=1.0, back=5.0):
    """One point on every pixel-centre ray; checkerboard of front/back depth."""
    from paper_2502_11618_b200 import PointCloud

    w, h = camera.width, camera.height
    us, vs = np.meshgrid(np.arange(w), np.arange(h))
    checker = (us + vs) % 2 == 0
    z = np.where(checker, front, back).astype(np.float64)
    pc = np.stack([(us + 0.5 - camera.cx) / camera.fx * z, (vs + 0.5 - camera.cy) / camera.fy * z,
                   z], axis=-1).reshape(-1, 3)
    pose = camera.world_to_camera
    world = (pc - pose.translation) @ pose.rotation
    cols = np.where(checker.reshape(-1, 1), (200, 60, 60), (60, 60, 200)).astype(np.uint8)
    return PointCloud(world.astype(np.float32), cols), checker


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def golden_camera(d, prefix, unchecked=False):
    """CameraModel rebuilt from a golden fixture (rot, t, intrinsics, size)."""
    from paper_2502_11618_b200 import CameraModel, RigidTransform

    fx, fy, cx, cy, zn, zf = (float(v) for v in d[prefix + "intr"])
    w, h = (int(v) for v in d[prefix + "wh"])
    pose = RigidTransform(d[prefix + "rot"], d[prefix + "t"])
    if unchecked or w % 16 or h % 16:
        return CameraModel.unchecked(fx, fy, cx, cy, w, h, pose, zn, zf)
    return CameraModel(fx, fy, cx, cy, w, h, pose, zn, zf)


def plain_camera(d, prefix):
    """Duck-typed camera for the oracle (no package import)."""
    fx, fy, cx, cy, zn, zf = (float(v) for v in d[prefix + "intr"])
    w, h = (int(v) for v in d[prefix + "wh"])
    pose = types.SimpleNamespace(rotation=d[prefix + "rot"], translation=d[prefix + "t"])
    return types.SimpleNamespace(fx=fx, fy=fy, cx=cx, cy=cy, width=w, height=h, z_near=zn,
                                 z_far=zf, world_to_camera=pose)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import PortKernels

    return PortKernels()


@pytest.fixture(scope="session")
def cuda_ready():
    """Asserts the B200 path is really available (fails, never skips)."""
    import torch

    assert torch.cuda.is_available(), "gpu test run without a CUDA device"
    from paper_2502_11618_b200 import _lib

    _lib.load()
    return True
