"""The in-process bridge on the B200: RGDA requests over a
socket, answered by UNetBridgeModel (device-side packing + tcgen05 U-Net)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu(cuda_ready):
    return cuda_ready


def _frame(rng, h, w):
    from paper_2502_11618_b200 import FrameRGBDA

    depth = ((rng.random((h, w)) + 0.05) * 20).astype(np.float32)
    depth[rng.random((h, w)) < 0.3] = 0.0
    alpha = (depth > 0).astype(np.uint8)
    return FrameRGBDA(rgb=rng.random((h, w, 3)).astype(np.float32) * alpha[..., None],
                      depth=depth, alpha=alpha)


def test_bridge_equals_direct_unet():
    import torch

    from paper_2502_11618_b200.bridge import BridgeServer, UNetBridgeModel, reconstruct
    from paper_2502_11618_b200.unet import UNet

    net = UNet.from_config("reduced", seed=9)
    rng = np.random.default_rng(4)
    fr = _frame(rng, 64, 96)
    with BridgeServer(UNetBridgeModel(net)) as srv:
        got = reconstruct(fr, srv.endpoint)
    # direct: the bridge's packing restated with torch (normalizeDepth in f64)
    dev = torch.device("cuda")
    d = torch.from_numpy(fr.depth).double()
    zn = net.cfg.depthZNear
    dn = torch.where(d > 0, zn / torch.clamp(d, min=zn), torch.zeros_like(d)).float()
    x = torch.zeros((1, 64, 96, net.in_pad), dtype=torch.bfloat16, device=dev)
    x[0, :, :, :3] = torch.from_numpy(fr.rgb).to(dev).bfloat16()
    x[0, :, :, 3] = dn.to(dev).bfloat16()
    x[0, :, :, 4] = torch.from_numpy(fr.alpha.astype(np.float32)).to(dev).bfloat16()
    out = torch.empty((1, 64, 96, 3), dtype=torch.float32, device=dev)
    net.forward(x, out)
    torch.cuda.synchronize()
    assert got.shape == (64, 96, 3) and got.dtype == np.float32
    assert np.array_equal(got, out[0].cpu().numpy())
    assert (got >= 0).all() and (got <= 1).all()


def test_bridge_rejects_indivisible_frame():
    from paper_2502_11618_b200 import BridgeError
    from paper_2502_11618_b200.bridge import BridgeServer, UNetBridgeModel, reconstruct
    from paper_2502_11618_b200.unet import UNet

    net = UNet.from_config("reduced", seed=9)
    with BridgeServer(UNetBridgeModel(net)) as srv:
        with pytest.raises(BridgeError, match="not divisible"):
            reconstruct(_frame(np.random.default_rng(1), 62, 96), srv.endpoint)
