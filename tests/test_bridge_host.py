"""Bridge wire format and client/server plumbing on the CPU (no GPU needed).

Byte-level parity with the reference's RawTensorFrame (fixtures written by the
reference itself: tests/golden/make_tensor_golden.py), the reference suite's
raw-tensor cases (pkg/tests/test_io.py:217-290), and the bridge round trip
of pkg/tests/test_cli.py:280-333 against a passthrough model."""

import io
import os
import socket
import tempfile

import numpy as np
import pytest

from conftest import GOLDEN

from paper_2502_11618_b200 import BridgeError, FrameRGBDA, TensorFormatError
from paper_2502_11618_b200.bridge import BridgeServer, PassthroughModel, reconstruct
from paper_2502_11618_b200.io import (MAGIC_RGB, MAGIC_RGBDA, RawTensorFrame, frame_to_tensor,
                                      read_reply, tensor_to_frame, write_error_frame)


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLDEN, "tensor.npz"))


def _bytes(t):
    buf = io.BytesIO()
    t.write(buf)
    return buf.getvalue()


def test_write_matches_reference_bytes(gold):
    assert _bytes(RawTensorFrame(MAGIC_RGBDA, gold["rgda_planes"])) == gold["rgda_bytes"].tobytes()
    assert _bytes(RawTensorFrame(MAGIC_RGB, gold["rgb_planes"])) == gold["rgb_bytes"].tobytes()


def test_read_reference_bytes(gold):
    t = RawTensorFrame.read(io.BytesIO(gold["rgda_bytes"].tobytes()))
    assert t.magic == MAGIC_RGBDA and np.array_equal(t.planes, gold["rgda_planes"])
    t = RawTensorFrame.read(io.BytesIO(gold["rgb_bytes"].tobytes()))
    assert t.magic == MAGIC_RGB and np.array_equal(t.planes, gold["rgb_planes"])


def test_frame_conversions_match_reference(gold):
    fr = FrameRGBDA(rgb=gold["frame_rgb"], depth=gold["frame_depth"], alpha=gold["frame_alpha"])
    assert np.array_equal(frame_to_tensor(fr).planes, gold["frame_tensor_planes"])
    back = tensor_to_frame(RawTensorFrame(MAGIC_RGBDA, gold["soft_planes"]))
    assert np.array_equal(back.alpha, gold["soft_alpha"])
    assert np.array_equal(back.depth, gold["soft_planes"][3])


def test_roundtrip_bit_exact(rng):
    planes = rng.random((5, 2, 2)).astype(np.float32)
    planes[0, 0, 0] = np.float32(np.nextafter(np.float32(1), np.float32(2)))
    got = RawTensorFrame.read(io.BytesIO(_bytes(RawTensorFrame(MAGIC_RGBDA, planes))))
    assert got.planes.tobytes() == planes.tobytes()


def test_bad_magic_and_channel_count():
    with pytest.raises(TensorFormatError, match="unknown magic"):
        RawTensorFrame.read(io.BytesIO(b"XXXX" + b"\x01\x00\x00\x00" * 3 + b"\x00" * 4))
    with pytest.raises(TensorFormatError, match="implies 5 channels"):
        RawTensorFrame.read(io.BytesIO(b"RGDA" + b"\x01\x00\x00\x00" * 3 + b"\x00" * 4))
    with pytest.raises(TensorFormatError, match="needs 3 channel planes"):
        RawTensorFrame(MAGIC_RGB, np.zeros((5, 2, 2), np.float32))


def test_short_read_and_zero_dims():
    data = _bytes(RawTensorFrame(MAGIC_RGB, np.zeros((3, 4, 4), np.float32)))
    with pytest.raises(TensorFormatError, match="short read"):
        RawTensorFrame.read(io.BytesIO(data[:-3]))
    with pytest.raises(TensorFormatError, match="implausible"):
        RawTensorFrame.read(io.BytesIO(b"RGB0" + (0).to_bytes(4, "little") * 2
                                       + (3).to_bytes(4, "little")))


class _Trickle(io.RawIOBase):
    """A non-seekable stream that hands out a few bytes per read."""

    def __init__(self, data):
        self.data, self.pos = data, 0

    def readable(self):
        return True

    def readinto(self, b):
        n = min(len(b), 7, len(self.data) - self.pos)
        b[:n] = self.data[self.pos:self.pos + n]
        self.pos += n
        return n


def test_streams_without_seeking(rng):
    planes = rng.random((5, 96, 128)).astype(np.float32)
    got = RawTensorFrame.read(_Trickle(_bytes(RawTensorFrame(MAGIC_RGBDA, planes))))
    assert np.array_equal(got.planes, planes)


def test_error_frames():
    buf = io.BytesIO()
    write_error_frame(buf, "model exploded")
    buf.seek(0)
    assert read_reply(buf) == "model exploded"


def _frame(rng, h=8, w=12):
    depth = ((rng.random((h, w)) + 0.5) * 4).astype(np.float32)
    depth[rng.random((h, w)) < 0.3] = 0.0
    alpha = (depth > 0).astype(np.uint8)
    return FrameRGBDA(rgb=rng.random((h, w, 3)).astype(np.float32) * alpha[..., None],
                      depth=depth, alpha=alpha)


def test_bridge_roundtrip_tcp_and_unix(rng):
    fr = _frame(rng)
    with BridgeServer(PassthroughModel()) as srv:
        assert np.array_equal(reconstruct(fr, srv.endpoint), fr.rgb)
        assert np.array_equal(reconstruct(fr, f":{srv.port}"), fr.rgb)
    with tempfile.TemporaryDirectory() as d:
        ep = f"unix:{d}/bridge.sock"
        with BridgeServer(PassthroughModel(), ep):
            assert np.array_equal(reconstruct(fr, ep), fr.rgb)


def test_bridge_serves_several_requests_per_connection(rng):
    frames = [_frame(rng, 4 + i, 6) for i in range(3)]
    with BridgeServer(PassthroughModel()) as srv:
        sock = socket.create_connection(("127.0.0.1", srv.port), timeout=5)
        with sock, sock.makefile("rwb") as stream:
            for fr in frames:
                frame_to_tensor(fr).write(stream)
                reply = read_reply(stream)
                assert reply.magic == MAGIC_RGB
                assert np.array_equal(np.moveaxis(reply.planes, 0, 2), fr.rgb)


class _Failing:
    def reconstruct(self, tensor):
        raise ValueError(f"input {tensor.width}x{tensor.height} not divisible by 2^depth = 16")


class _WrongShape:
    def reconstruct(self, tensor):
        return np.zeros((3, tensor.height + 1, tensor.width), np.float32)


def test_bridge_errors(rng):
    fr = _frame(rng)
    with pytest.raises(BridgeError, match="cannot reach bridge"):
        reconstruct(fr, "127.0.0.1:1", timeout=2)
    with BridgeServer(_Failing()) as srv:
        with pytest.raises(BridgeError, match="not divisible"):
            reconstruct(fr, srv.endpoint)
    with BridgeServer(_WrongShape()) as srv:
        with pytest.raises(BridgeError, match="does not match"):
            reconstruct(fr, srv.endpoint)
    with BridgeServer(PassthroughModel()) as srv:  # an RGB0 request is refused with ERR0
        sock = socket.create_connection(("127.0.0.1", srv.port), timeout=5)
        with sock, sock.makefile("rwb") as stream:
            RawTensorFrame(MAGIC_RGB, np.zeros((3, 2, 2), np.float32)).write(stream)
            assert "expected RGDA" in read_reply(stream)
