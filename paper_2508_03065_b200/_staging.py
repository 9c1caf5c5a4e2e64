"""Host <-> device staging for the render planner.

parallel_copy  thread-pool numpy copies (host memory bandwidth, not one core)
_BulkStager    persistent pinned slabs: bulk inputs (paths, signals) in one
               asynchronous copy each, no per-call cudaHostAlloc
_PathArena     persistent device buffers for paths staged on the side stream
side_stream    high-priority per-device stream for input staging
d2h            device -> numpy through persistent pinned staging
"""

from __future__ import annotations

import os
import warnings

import numpy as np
import torch

from ._dev import pinned_scratch

_POOL = None


def _copy_pool():
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=max(1, min(8, os.cpu_count() or 1)),
                                   thread_name_prefix="mvb-stage")
    return _POOL


def parallel_copy(pairs, chunk_bytes: int = 4 << 20) -> None:
    """np.copyto(dst, src) for every (dst, src) pair, split into chunks
    along axis 0 and run on a thread pool (numpy releases the GIL for plain
    copies, so host memory bandwidth, not one core, bounds bulk staging)."""
    tasks = []
    total = 0
    for dst, src in pairs:
        n = dst.shape[0] if dst.ndim else 1
        row = max(1, dst.nbytes // max(n, 1))
        step = max(1, chunk_bytes // row)
        for r in range(0, max(n, 1), step):
            tasks.append((dst[r:r + step], src[r:r + step]) if dst.ndim else (dst, src))
        total += dst.nbytes
    if total < (8 << 20) or len(tasks) == 1:
        for d, s_ in tasks:
            np.copyto(d, s_, casting="unsafe")
        return
    pool = _copy_pool()
    nw = pool._max_workers
    groups = [tasks[i::nw] for i in range(nw)]

    def run(group):
        for d, s_ in group:
            np.copyto(d, s_, casting="unsafe")

    for fut in [pool.submit(run, g) for g in groups if g]:
        fut.result()


def _host_tensor(a: np.ndarray) -> torch.Tensor:
    """torch view of a (possibly read-only) host array used only as a copy
    source; torch's warning about non-writable arrays does not apply."""
    with warnings.catch_warnings():
        warnings.filterwarnings("ignore", message="The given NumPy array is not writable")
        return torch.from_numpy(a)


def copy_batch(entries, stream: int, require_pinned: bool) -> np.ndarray:
    """Issue [(dst_ptr, src_ptr, nbytes)] as asynchronous copies on `stream`
    with one libmvb call (mvb_copy_batch); returns which entries were issued
    (with `require_pinned`, sources outside page-locked memory are left to
    the caller)."""
    from . import _lib
    n = len(entries)
    if n == 0:
        return np.zeros(0, bool)
    a = np.asarray(entries, dtype=np.int64).reshape(n, 3)
    dst, src, nb = (np.ascontiguousarray(a[:, k]) for k in range(3))
    issued = np.zeros(n, np.int32)
    _lib.call("mvb_copy_batch", dst.ctypes.data, src.ctypes.data, nb.ctypes.data, n,
              issued.ctypes.data, int(bool(require_pinned)), stream)
    return issued.astype(bool)


def is_pinned(a) -> bool:
    """True for a C-contiguous numpy array in page-locked host memory (e.g.
    a view of a pinned torch tensor, or a Trajectory's positions): such
    parts are sent by DMA straight from the caller's buffer."""
    if not isinstance(a, np.ndarray) or not a.flags.c_contiguous or a.nbytes == 0:
        return False
    try:
        return bool(_host_tensor(a).is_pinned())
    except (TypeError, RuntimeError, ValueError):
        return False


def pinned_copy(a: np.ndarray) -> np.ndarray:
    """A read-only copy of `a` in page-locked host memory (pinned torch
    storage kept alive by the returned array), or a plain copy without a
    GPU -- for inputs uploaded many times (trajectories)."""
    a = np.ascontiguousarray(a)
    if not torch.cuda.is_available():
        out = a.copy()
    else:
        t = torch.empty(a.shape, dtype=_TORCH.get(a.dtype.str[1:], torch.uint8), pin_memory=True)
        out = t.numpy() if a.dtype.str[1:] in _TORCH else t.numpy().view(a.dtype)
        np.copyto(out, a)
    out.flags.writeable = False
    return out


_TORCH = {"f8": torch.float64, "f4": torch.float32, "i8": torch.int64, "i4": torch.int32}


class _BulkStager:
    """Persistent pinned slabs for bulk uploads (paths, signals): parts are
    copied straight into a slab (parallel_copy) and sent with ONE
    asynchronous copy; a slab is reused once the event recorded after its
    copy has completed, so no per-call cudaHostAlloc and no host sync."""

    MAX_SLABS = 4

    def __init__(self):
        self.slabs = []  # [pinned uint8 tensor, event | None]

    def _acquire(self, nbytes: int):
        for sl in self.slabs:
            if sl[0].numel() >= nbytes and (sl[1] is None or sl[1].query()):
                return sl
        cap = 1 << max(20, (max(nbytes, 1) - 1).bit_length())
        sl = [torch.empty(cap, dtype=torch.uint8, pin_memory=True), None]
        self.slabs.append(sl)
        if len(self.slabs) > self.MAX_SLABS:  # drop the smallest idle slab
            idle = [x for x in self.slabs if x is not sl and (x[1] is None or x[1].query())]
            if idle:  # by identity: list.remove compares tensors elementwise
                victim = min(idle, key=lambda x: x[0].numel())
                self.slabs = [x for x in self.slabs if x is not victim]
        return sl

    def upload(self, parts, out: torch.Tensor) -> None:
        """parts: [(row0, host array)] written into rows of `out` (a device
        tensor whose trailing dims match the parts); one H2D copy of the
        covered rows [0, max row)."""
        if not parts:
            return
        np_dt = torch.empty((), dtype=out.dtype).numpy().dtype
        direct = [(r0, p) for r0, p in parts
                  if isinstance(p, np.ndarray) and p.dtype == np_dt and is_pinned(p)]
        if direct:  # page-locked caller buffers: DMA straight from them
            for r0, p in direct:
                n = p.shape[0] if p.ndim else 1
                out[r0:r0 + n].copy_(_host_tensor(p).reshape((n,) + tuple(out.shape[1:])),
                                     non_blocking=True)
            ids = {id(p) for _, p in direct}
            parts = [(r0, p) for r0, p in parts if id(p) not in ids]
            if not parts:
                return
        row_elems = int(np.prod(out.shape[1:])) if out.dim() > 1 else 1
        rows = max(r0 + (p.shape[0] if np.ndim(p) else 1) for r0, p in parts)
        nbytes = rows * row_elems * np_dt.itemsize
        sl = self._acquire(nbytes)
        host = sl[0][:nbytes].numpy().view(np_dt).reshape((rows,) + tuple(out.shape[1:]))
        covered = np.zeros(rows, bool)
        pairs = []
        for r0, p in parts:
            p = np.asarray(p)
            n = p.shape[0]
            pairs.append((host[r0:r0 + n], p.reshape((n,) + tuple(out.shape[1:]))))
            covered[r0:r0 + n] = True
        if not covered.all():
            host[~covered] = 0
        parallel_copy(pairs)
        out[:rows].copy_(sl[0][:nbytes].view(out.dtype).view((rows,) + tuple(out.shape[1:])),
                         non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        sl[1] = ev


_STAGER = _BulkStager()
_SIDE = {}


class _PathArena:
    """Persistent device buffers for the paths of renders staged on the side
    stream (Geometry with inputs_ready).  A buffer is handed out again only
    after the event recorded when its render was fully enqueued has
    completed, so no render overwrites paths a queued kernel still reads;
    buffers are never freed, so no allocator events or cudaMalloc (which can
    stall behind running kernels) sit on the staging path.  At most DEPTH
    buffers: a deeper pipeline waits for the oldest render."""

    DEPTH = 3

    def __init__(self):
        self.bufs = {}  # device -> list of [tensor, event | None]

    def acquire(self, dev, rows: int) -> torch.Tensor:
        lst = self.bufs.setdefault(str(dev), [])
        idle = [b for b in lst if b[1] is None or (b[1] is not False and b[1].query())]
        fits = [b for b in idle if b[0].shape[0] >= rows]
        if fits:
            b = fits[0]
        elif len(lst) < self.DEPTH:
            b = [torch.empty(max(rows, 1 << 16), 3, dtype=torch.float64, device=dev), None]
            lst.append(b)
        else:  # pipeline full: wait for the oldest released render, grow if needed
            released = [x for x in lst if x[1] is not False]
            if not released:  # every buffer held by an unreleased geometry
                return torch.empty(rows, 3, dtype=torch.float64, device=dev)
            b = released[0]
            if b[1] is not None:
                b[1].synchronize()
            if b[0].shape[0] < rows:
                b[0] = torch.empty(rows, 3, dtype=torch.float64, device=dev)
        b[1] = False  # in use until release
        return b[0]

    def release(self, dev, t: torch.Tensor, event) -> None:
        for b in self.bufs.get(str(dev), []):
            if b[0] is t:
                b[1] = event


_ARENA = _PathArena()


def side_stream(dev) -> torch.cuda.Stream:
    """Per-device side stream for input staging that must not queue behind
    the current stream.  Highest priority: its few small kernels (path
    copies, boxes, bandwidth FFT) are scheduled ahead of the pending CTAs of
    a running synthesis instead of after them."""
    key = str(dev)
    if key not in _SIDE:
        _SIDE[key] = torch.cuda.Stream(device=dev, priority=-64)
    return _SIDE[key]


D2H_DIRECT = 1 << 16  # elements: above, d2h returns a pinned block of the caching allocator


def d2h(t: torch.Tensor, dtype=None) -> np.ndarray:
    """Device tensor -> new numpy array (optionally converted to `dtype`).
    Large results: cast on the device, one copy into a pinned block of
    torch's caching host allocator, returned as the array itself (no host
    conversion or copy-out; the block returns to the cache when the array is
    dropped, so steady-state calls allocate no new pinned memory).  Small
    ones: persistent pinned staging + a copy out."""
    if t.numel() >= D2H_DIRECT:
        tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32}.get(
            np.dtype(dtype) if dtype is not None else None, t.dtype)
        src = t.reshape(-1) if tdt == t.dtype else t.reshape(-1).to(tdt)
        host = torch.empty(src.numel(), dtype=tdt, pin_memory=True)
        host.copy_(src, non_blocking=True)
        torch.cuda.current_stream(t.device).synchronize()
        return host.numpy().reshape(tuple(t.shape))
    host = pinned_scratch("d2h_" + str(t.dtype), t.numel(), t.dtype)
    host.copy_(t.reshape(-1), non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    src = host.numpy()
    out = np.empty(t.numel(), dtype=src.dtype if dtype is None else dtype)
    parallel_copy([(out, src)])
    return out.reshape(tuple(t.shape))
