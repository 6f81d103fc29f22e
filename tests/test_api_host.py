"""Host-side API contract of the drop-in package (types, validation messages,
backend registry).  CPU only -- no compute is launched."""

import numpy as np
import pytest

import lidarsplat
from lidarsplat import (CameraModel, FilterParams, PointCloud, RenderParams, RigidTransform,
                        build_grid, extract_frustum)
from lidarsplat.errors import CameraError, InvalidCloudError

from conftest import make_camera


def test_backend_registry_is_cuda_only(monkeypatch):
    assert lidarsplat.available_backends() == ["cuda"]
    assert lidarsplat.get_backend().name == "cuda"
    with pytest.raises(ValueError, match="unknown backend"):
        lidarsplat.get_backend("numpy")
    monkeypatch.setenv("LIDARSPLAT_BACKEND", "native")
    with pytest.raises(ValueError, match="not available"):
        lidarsplat.default_backend_name()


def test_camera_rules():
    with pytest.raises(CameraError, match="divisible by 16"):
        CameraModel(1000.0, 1000.0, 960.0, 540.0, 1920, 1080)
    cam = CameraModel.unchecked(1000.0, 1000.0, 960.0, 540.0, 1920, 1080)
    assert (cam.width, cam.height) == (1920, 1080)
    with pytest.raises(CameraError, match="focal"):
        CameraModel(0.0, 1.0, 1.0, 1.0, 16, 16)
    with pytest.raises(CameraError, match="z_near"):
        CameraModel(1.0, 1.0, 1.0, 1.0, 16, 16, z_near=2.0, z_far=1.0)
    with pytest.raises(CameraError, match="orthonormal"):
        RigidTransform(np.ones((3, 3)), np.zeros(3))


def test_cloud_rules():
    with pytest.raises(InvalidCloudError, match="positions must be"):
        PointCloud(np.zeros((0,), np.float32), np.zeros((0,), np.uint8))
    with pytest.raises(InvalidCloudError, match="invalid point"):
        PointCloud(np.array([[0, 0, np.nan]], np.float32), np.zeros((1, 3), np.uint8))
    empty = PointCloud(np.zeros((0, 3), np.float32), np.zeros((0, 3), np.uint8))
    with pytest.raises(InvalidCloudError, match="empty cloud"):
        build_grid(empty, 1.0)
    rng = np.random.default_rng(0)
    far = PointCloud((rng.random((10, 3)) * 1000).astype(np.float32), np.zeros((10, 3), np.uint8))
    with pytest.raises(InvalidCloudError, match="cells exceeds"):
        build_grid(far, 1e-4)


def test_params_rules():
    with pytest.raises(ValueError):
        RenderParams(zbuffer_epsilon_rel=-1)
    with pytest.raises(ValueError):
        FilterParams(levels_n=0)
    with pytest.raises(ValueError):
        FilterParams(edge_threshold=0)
    with pytest.raises(ValueError, match="too small"):
        lidarsplat.build_min_pyramid(np.zeros((4, 4), np.float32), 3)
    with pytest.raises(ValueError, match="ceil-half"):
        lidarsplat.upsample_filter_step(np.ones((3, 3), np.float32), np.ones((4, 4), np.float32),
                                        FilterParams(), True)


def test_frustum_matches_oracle_planes():
    from oracle.oracle import frustum_planes

    cam = make_camera(eye=(1.0, 2.0, -3.0), target=(0.0, 0.0, 5.0))
    assert np.array_equal(extract_frustum(cam).planes, frustum_planes(cam))


def test_cpu_only_host_raises_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from lidarsplat import _lib

    with pytest.raises(_lib.CudaUnavailableError):
        _lib.device()
