"""The neural reconstruction bridge, both ends, with the CUDA U-Net in process.

Client (R:bridge.py:34-56): ``reconstruct(frame, endpoint)`` sends one RGDA
raw tensor frame to a bridge peer and returns its RGB0 reply as (H, W, 3)
float32.  Endpoints: "host:port", ":port" (localhost) or "unix:/path".

Server (the role of FE:src/bridge.ts:64-116, run by node in the reference):
``BridgeServer(model)`` answers RGDA requests on a stream socket, one request
in flight per connection; a request it cannot serve gets an "ERR0" error
frame and the connection is closed.  ``UNetBridgeModel`` is the reference's
UNetBridgeModel (FE:src/bridge.ts:28-53) on the device: the RGDA planes go
to HBM, ``ls_unet_pack_rgbda`` builds the bf16 input (normalizeDepth fused)
and the tcgen05 U-Net runs -- so ``lidarsplat render --bridge``-style callers
work with no node/tfjs process.  ``PassthroughModel`` echoes the rgb planes
(framing tests, FE:src/bridge.ts:56-62).
"""

from __future__ import annotations

import os
import socket
import threading

import numpy as np

from . import _lib
from .errors import BridgeError, TensorFormatError
from .frame import FrameRGBDA
from .io.tensor import (MAGIC_RGB, MAGIC_RGBDA, RawTensorFrame, frame_to_tensor, read_reply,
                        write_error_frame)


# ------------------------------------------------------------------ client --
def _connect(endpoint: str, timeout: float) -> socket.socket:
    try:
        if endpoint.startswith("unix:"):
            sock = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            sock.settimeout(timeout)
            sock.connect(endpoint[len("unix:"):])
            return sock
        host, _, port = endpoint.rpartition(":")
        sock = socket.create_connection((host or "127.0.0.1", int(port)), timeout=timeout)
        sock.settimeout(timeout)
        return sock
    except (OSError, ValueError) as e:
        raise BridgeError(f"cannot reach bridge at {endpoint!r}: {e}") from None


def reconstruct(frame: FrameRGBDA, endpoint: str, timeout: float = 10.0) -> np.ndarray:
    """Round-trip one frame through the bridge; returns (H, W, 3) float32 rgb."""
    request = frame_to_tensor(frame)
    sock = _connect(endpoint, timeout)
    try:
        with sock.makefile("rwb") as stream:
            request.write(stream)
            try:
                reply = read_reply(stream)
            except TensorFormatError as e:
                raise BridgeError(f"bad bridge reply: {e}") from None
    except (OSError, socket.timeout) as e:
        raise BridgeError(f"bridge i/o failed: {e}") from None
    finally:
        sock.close()
    if isinstance(reply, str):
        raise BridgeError(f"bridge error: {reply}")
    if reply.magic != MAGIC_RGB:
        raise BridgeError(f"bridge replied with magic {reply.magic!r}, expected RGB0")
    if reply.planes.shape[1:] != (frame.height, frame.width):
        raise BridgeError(f"bridge reply {reply.planes.shape[1:]} does not match "
                          f"request {(frame.height, frame.width)}")
    return np.ascontiguousarray(np.moveaxis(reply.planes, 0, 2))


# ------------------------------------------------------------------ models --
class PassthroughModel:
    """Echoes the request's rgb planes (framing tests)."""

    def reconstruct(self, tensor: RawTensorFrame) -> np.ndarray:
        return tensor.planes[:3]


class UNetBridgeModel:
    """RGDA tensor -> U-Net RGB planes on the B200 (no host-side packing)."""

    def __init__(self, unet):
        self.unet = unet
        self._bufs = {}
        self._lock = threading.Lock()

    def _buffers(self, h: int, w: int):
        import torch

        key = (h, w)
        if key not in self._bufs:
            dev = self.unet.device
            self._bufs[key] = (
                torch.empty((5, h, w), dtype=torch.float32, device=dev),
                torch.zeros((1, h, w, self.unet.in_pad), dtype=torch.bfloat16, device=dev),
                torch.empty((1, h, w, 3), dtype=torch.float32, device=dev),
                torch.empty((3, h, w), dtype=torch.float32, pin_memory=True),
            )
        return self._bufs[key]

    def reconstruct(self, tensor: RawTensorFrame) -> np.ndarray:
        import torch

        if tensor.magic != MAGIC_RGBDA:
            raise TensorFormatError(f"expected RGDA, got {tensor.magic!r}")
        h, w, div = tensor.height, tensor.width, self.unet.divisor
        if h % div or w % div:  # FE:src/model/tfjsExec.ts:121-125
            raise ValueError(f"input {w}x{h} not divisible by 2^depth = {div}")
        with self._lock, torch.cuda.device(self.unet.device):
            planes, x, out, host = self._buffers(h, w)
            planes.copy_(torch.from_numpy(tensor.planes), non_blocking=False)
            _lib.check(_lib.load().ls_unet_pack_rgbda(
                planes.data_ptr(), h, w, self.unet.in_pad, float(self.unet.cfg.depthZNear),
                x.data_ptr(), _lib.stream_ptr()), "unet_pack_rgbda")
            self.unet.forward(x, out)
            host.copy_(out[0].permute(2, 0, 1))
            return host.numpy().copy()


# ------------------------------------------------------------------ server --
class BridgeServer:
    """Serves RGDA -> RGB0 requests with ``model`` on a TCP or unix socket.

    ``endpoint`` is "host:port" (port 0 picks a free one) or "unix:/path";
    ``start()`` runs the accept loop on a daemon thread, ``close()`` stops it.
    """

    def __init__(self, model, endpoint: str = "127.0.0.1:0"):
        self.model = model
        if endpoint.startswith("unix:"):
            self._path = endpoint[len("unix:"):]
            if os.path.exists(self._path):
                os.unlink(self._path)
            self._sock = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            self._sock.bind(self._path)
            self.endpoint = endpoint
        else:
            self._path = None
            host, _, port = endpoint.rpartition(":")
            self._sock = socket.socket()
            self._sock.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
            self._sock.bind((host or "127.0.0.1", int(port)))
            bound = self._sock.getsockname()
            self.endpoint = f"{bound[0]}:{bound[1]}"
        self._sock.listen(16)
        self._thread = None
        self._closed = False

    @property
    def port(self) -> int | None:
        return None if self._path else int(self.endpoint.rpartition(":")[2])

    def start(self) -> "BridgeServer":
        self._thread = threading.Thread(target=self._accept_loop, daemon=True)
        self._thread.start()
        return self

    def close(self) -> None:
        self._closed = True
        try:
            self._sock.close()
        finally:
            if self._path and os.path.exists(self._path):
                os.unlink(self._path)

    def __enter__(self):
        return self.start()

    def __exit__(self, *exc):
        self.close()

    def _accept_loop(self) -> None:
        while not self._closed:
            try:
                conn, _ = self._sock.accept()
            except OSError:
                return
            threading.Thread(target=self._serve, args=(conn,), daemon=True).start()

    def _serve(self, conn: socket.socket) -> None:
        with conn, conn.makefile("rwb") as stream:
            while True:
                try:
                    request = read_reply(stream)
                except TensorFormatError as e:
                    if "ended after 0 of" in str(e):  # peer closed between requests
                        return
                    write_error_frame(stream, str(e))
                    return
                except OSError:
                    return
                if isinstance(request, str):
                    write_error_frame(stream, f"unexpected error frame: {request}")
                    return
                if request.magic != MAGIC_RGBDA:
                    write_error_frame(stream, f"expected RGDA request, got "
                                              f"{request.magic.decode()}")
                    return
                try:
                    rgb = self.model.reconstruct(request)
                    RawTensorFrame(MAGIC_RGB, rgb).write(stream)
                except Exception as e:  # noqa: BLE001  (any failure becomes an ERR0 reply)
                    try:
                        write_error_frame(stream, str(e))
                    except OSError:
                        pass
                    return
