"""Device plumbing: torch owns memory and streams; libmvb owns the math."""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from ._lib import MvbError, lib


def require_cuda(device=None) -> torch.device:
    """The CUDA device to run on; raises when there is none (no fallback)."""
    if not torch.cuda.is_available():
        raise MvbError("no CUDA device: paper_2508_03065_b200 runs only on a GPU (sm_100a)")
    lib()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise MvbError(f"device {d} is not a CUDA device")
    return d


def ptr(t) -> ctypes.c_void_p:
    if t is None:
        return ctypes.c_void_p(0)
    return ctypes.c_void_p(t.data_ptr())


def stream_handle(device=None) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class _PinnedRing:
    """Persistent pinned staging ring for the planner's small uploads.

    Arrays are copied into the ring and sent with an asynchronous
    stream-ordered copy (no host sync, no per-call cudaHostAlloc, no
    per-call event).  A lap is ~16 MB (hundreds of renders); before the ring
    wraps, the device is synchronised once, so no staged bytes are
    overwritten before their copy ran, whatever stream issued it.
    """

    ALIGN = 256

    def __init__(self, nbytes: int = 16 << 20):
        self.cap = nbytes
        self.buf = None
        self.off = 0

    def put(self, a: np.ndarray, dev) -> torch.Tensor:
        a = np.ascontiguousarray(a)
        n = a.nbytes
        if n > self.cap // 4:  # large arrays: one-off pinned copy (own writable copy)
            return torch.from_numpy(np.array(a, copy=True)).pin_memory().to(dev, non_blocking=True)
        if self.buf is None:
            self.buf = torch.empty(self.cap, dtype=torch.uint8, pin_memory=True)
            self.host = self.buf.numpy()
        if self.off + n > self.cap:
            torch.cuda.synchronize()
            self.off = 0
        self.host[self.off:self.off + n] = a.reshape(-1).view(np.uint8)
        src = self.buf[self.off:self.off + n].view(_TORCH_DTYPE[a.dtype.str[1:]])
        out = src.reshape(a.shape).to(dev, non_blocking=True)
        self.off += -(-max(n, 1) // self.ALIGN) * self.ALIGN
        return out


_TORCH_DTYPE = {"f8": torch.float64, "f4": torch.float32, "i8": torch.int64, "i4": torch.int32,
                "u1": torch.uint8, "b1": torch.bool}
_RING = _PinnedRing()


_PINNED: dict = {}


def pinned_scratch(name: str, n: int, dtype) -> torch.Tensor:
    """Persistent pinned host scratch `name` for small readbacks whose copy
    the caller waits for before the next use.  Pinned (not pageable) so a
    readback on a side stream waits only for that stream -- a pageable
    device->host copy also waits for the legacy default stream -- and
    persistent so no per-call cudaHostAlloc (which synchronises the device)."""
    t = _PINNED.get(name)
    if t is None or t.numel() < n or t.dtype != dtype:
        t = _PINNED[name] = torch.empty(max(n, 1024), dtype=dtype, pin_memory=True)
    return t[:n]


def readback(t: torch.Tensor, name: str) -> np.ndarray:
    """Small device tensor -> numpy through pinned scratch, waiting only for
    the current stream's work up to here."""
    host = pinned_scratch(name, t.numel(), t.dtype)
    host.copy_(t.reshape(-1), non_blocking=True)
    ev = torch.cuda.Event()
    ev.record()
    ev.synchronize()
    return host.numpy().copy().reshape(t.shape)


class StaticUploads:
    """Upload source for CUDA-graph capture: while active (`with`), h2d
    copies host arrays into consecutive slices of one persistent pinned
    buffer that the captured memcpy nodes keep reading at every replay (the
    pinned ring would be overwritten).  `nbytes` must cover the captured
    uploads (size it from a dry run's `used`)."""

    _active = None

    def __init__(self, nbytes: int):
        self.buf = torch.empty(max(int(nbytes), 1024), dtype=torch.uint8, pin_memory=True)
        self.host = self.buf.numpy()
        self.used = 0

    def __enter__(self):
        StaticUploads._active = self
        return self

    def __exit__(self, *exc):
        StaticUploads._active = None

    def put(self, a: np.ndarray, dev) -> torch.Tensor:
        a = np.ascontiguousarray(a)
        n = a.nbytes
        if self.used + n > self.buf.numel():
            raise MvbError("static upload buffer too small for the captured render")
        self.host[self.used:self.used + n] = a.reshape(-1).view(np.uint8)
        src = self.buf[self.used:self.used + n].view(_TORCH_DTYPE[a.dtype.str[1:]])
        self.used += -(-max(n, 1) // 256) * 256
        return src.reshape(a.shape).to(dev, non_blocking=True)


class UploadMeter:
    """Counts the bytes h2d would stage (dry run before a capture)."""

    _active = None

    def __init__(self):
        self.used = 0

    def __enter__(self):
        UploadMeter._active = self
        return self

    def __exit__(self, *exc):
        UploadMeter._active = None


def h2d(a: np.ndarray, dev) -> torch.Tensor:
    """Host array -> device without a host sync (pinned ring staging, or the
    active StaticUploads buffer during a graph capture)."""
    a = np.asarray(a)
    if StaticUploads._active is not None:
        return StaticUploads._active.put(a, dev)
    if UploadMeter._active is not None:
        UploadMeter._active.used += -(-max(a.nbytes, 1) // 256) * 256
    return _RING.put(a, dev)


def to_dev(a, dtype, device) -> torch.Tensor:
    """numpy / torch -> contiguous device tensor of dtype (no copy if already);
    host arrays go through the pinned ring (asynchronous, no host sync)."""
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype).contiguous()
    arr = np.array(np.asarray(a), dtype=torch.empty((), dtype=dtype).numpy().dtype, order="C")
    return h2d(arr, device)


def release_pinned(tags) -> None:
    """Drop the pinned scratch buffers whose names end with one of `tags`."""
    for name in [n for n in _PINNED if any(n.endswith(t) for t in tags)]:
        del _PINNED[name]
