"""Operator boundary: drop-in for the reference's kernel module.

Reference _kernels.py:21-31 selects numba or numpy once at import and
exposes three hot loops; this module exposes the same three functions with
the same signatures and semantics, executed by libmvb on the GPU with the
reference's fp64 arithmetic order (bit-identical results):

  distance_streams(offset, sign, mic, pos) -> new (S,T)      _kernels.py:65-78
  accumulate_images(out, streams, tau, amp, offset, d0) -> out   :126-136
      (mutates the caller's `out`, numpy or CUDA tensor, like the reference)
  upsample_stream(coarse, table, factor, out_len) -> new (out_len,)  :184-190

Inputs may be numpy arrays (copied to and from the device) or CUDA tensors
(used in place).  `using_numba()` is kept for API parity and is False.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._dev import ptr, require_cuda, stream_handle, to_dev


def using_numba() -> bool:
    return False


def using_cuda() -> bool:
    require_cuda()
    return True


def _is_dev(a) -> bool:
    return isinstance(a, torch.Tensor) and a.is_cuda


def distance_streams(offset, sign, mic, pos):
    dev = require_cuda(offset.device if _is_dev(offset) else None)
    o = to_dev(offset, torch.float64, dev).reshape(-1, 3)
    s = to_dev(sign, torch.float64, dev).reshape(-1, 3)
    m = to_dev(mic, torch.float64, dev).reshape(3)
    p = to_dev(pos, torch.float64, dev).reshape(-1, 3)
    out = torch.empty(o.shape[0], p.shape[0], dtype=torch.float64, device=dev)
    _lib.call("mvb_distance_streams", ptr(o), ptr(s), ptr(m), ptr(p), o.shape[0], p.shape[0],
              ptr(out), stream_handle(dev))
    return out if _is_dev(offset) else out.cpu().numpy()


def accumulate_images(out, streams, tau, amp, offset, d0):
    dev = require_cuda(out.device if _is_dev(out) else None)
    o = out if _is_dev(out) else to_dev(out, torch.float64, dev)
    if o.dtype != torch.float64 or not o.is_contiguous():
        raise ValueError("out must be a contiguous float64 buffer")
    st = to_dev(streams, torch.float64, dev)
    ta = to_dev(tau, torch.float64, dev)
    am = to_dev(amp, torch.float64, dev)
    S = ta.shape[0] if ta.ndim == 2 else 0
    if ta.ndim != 2 or am.shape != ta.shape or ta.shape[1] != o.shape[0]:
        raise ValueError("tau/amp must be (S, len(out))")
    _lib.call("mvb_accumulate_images", ptr(o), o.shape[0], ptr(st), st.shape[0], st.shape[1],
              ptr(ta), ptr(am), S, int(offset), int(d0), stream_handle(dev))
    if not _is_dev(out):
        out[...] = o.cpu().numpy()
    return out


def upsample_stream(coarse, table, factor, out_len):
    dev = require_cuda(coarse.device if _is_dev(coarse) else None)
    c = to_dev(coarse, torch.float64, dev).reshape(-1)
    t = to_dev(table, torch.float64, dev)
    res = torch.empty(int(out_len), dtype=torch.float64, device=dev)
    _lib.call("mvb_upsample_streams", ptr(c), 1, c.shape[0], ptr(t), int(factor), t.shape[1],
              int(out_len), ptr(res), stream_handle(dev))
    return res if _is_dev(coarse) else res.cpu().numpy()


def branch_filter(x, branches):
    """(M+1, len(x)+L-1) branch streams (reference farrow.py:214-229)."""
    dev = require_cuda(x.device if _is_dev(x) else None)
    xv = to_dev(x, torch.float64, dev).reshape(-1)
    b = to_dev(np.asarray(branches, dtype=np.float64) if not _is_dev(branches) else branches,
               torch.float64, dev)
    nb, L = b.shape
    out = torch.empty(nb, xv.shape[0] + L - 1, dtype=torch.float64, device=dev)
    _lib.call("mvb_branch_filter", ptr(xv), xv.shape[0], ptr(b), nb, L, ptr(out), stream_handle(dev))
    return out if _is_dev(x) else out.cpu().numpy()
