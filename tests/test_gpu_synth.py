"""Training-pair synthesis on the B200 vs the reference's
recipes (R:synth.py:77-115) restated over the oracle's frame + filter."""

import numpy as np
import pytest

from conftest import random_cloud, random_view
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu(cuda_ready):
    return cuda_ready


@pytest.mark.parametrize("leaky", [False, True])
def test_pairs_match_reference_recipe(rng, port, leaky):
    from paper_2502_11618_b200 import FilterParams, RenderParams, build_grid
    from paper_2502_11618_b200.synth import make_filtered_pair, make_leaky_pair

    cloud = random_cloud(rng, 120_000, extent=10.0, offset=-5.0)
    cam = random_view(rng, cloud)
    gt = rng.random((cam.height, cam.width, 3)).astype(np.float32)
    fp, rp = FilterParams(), RenderParams()
    grid = build_grid(cloud, 1.0)
    maker = make_leaky_pair if leaky else make_filtered_pair
    pair = maker(cloud, grid, gt, cam, fp, rp, pair_id="p7")
    # the reference recipe over the oracle's (bit-exact) frame and filter
    rgb, depth, alpha, _, _ = O.project(cloud.positions, cloud.colors, np.zeros(1, np.int64),
                                        np.array([cloud.count], np.int64), cam,
                                        rp.zbuffer_epsilon_rel, port)
    frgb, fdepth, falpha, _ = O.depth_filter(rgb, depth, alpha, fp.levels_n, fp.filter_strength,
                                             fp.edge_threshold, port)
    keep = falpha.astype(bool)
    if leaky:
        bg = alpha.astype(bool) & ~keep
        want = np.where(keep[:, :, None], gt, np.where(bg[:, :, None], rgb, np.float32(0)))
        wd, wa = depth, alpha
    else:
        want = np.where(keep[:, :, None], gt, np.float32(0))
        wd, wa = fdepth, falpha
    assert pair.id == "p7" and pair.target is not None and np.array_equal(pair.target, gt)
    assert np.array_equal(pair.input.rgb, want)
    assert np.array_equal(pair.input.depth, wd) and np.array_equal(pair.input.alpha, wa)


def test_gt_shape_checked(rng):
    from paper_2502_11618_b200 import FilterParams, RenderParams, build_grid
    from paper_2502_11618_b200.errors import DatasetError
    from paper_2502_11618_b200.synth import make_filtered_pair

    cloud = random_cloud(rng, 1000)
    cam = random_view(rng, cloud)
    with pytest.raises(DatasetError, match="does not match camera"):
        make_filtered_pair(cloud, build_grid(cloud, 1.0), np.zeros((4, 4, 3), np.float32), cam,
                           FilterParams(), RenderParams())
