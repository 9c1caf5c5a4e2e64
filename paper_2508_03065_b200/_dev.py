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


def to_dev(a, dtype, device) -> torch.Tensor:
    """numpy / torch -> contiguous device tensor of dtype (no copy if already)."""
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype).contiguous()
    arr = np.array(np.asarray(a), dtype=torch.empty((), dtype=dtype).numpy().dtype, order="C")
    # pinned staging + async copy: no host/stream serialisation
    return torch.from_numpy(arr).pin_memory().to(device, non_blocking=True)
