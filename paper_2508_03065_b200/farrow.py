"""Fractional-delay filter banks in polynomial (Farrow) form.

The reference realises every time-varying delay with a Farrow bank: M+1
branch FIRs c_k(n) with h(n, mu) = sum_k c_k(n) mu^k, the input convolved
with each branch once and a Horner evaluation per (image, sample)
(reference farrow.py:42-63, 192-229; _kernels.py:107-123; paper Eq. 3-5).
This module keeps that interface:

  FarrowFilter      same fields and validation as reference farrow.py:42-63;
                    reference FarrowFilter objects are accepted anywhere a
                    filter is expected (duck-typed on the same attributes).
  hann_sinc         the configs' L-tap Hann-windowed sinc delay, expressed as
                    a Farrow bank: Chebyshev least-squares fit of
                    h(j, mu) = sinc(t) * 0.5 (1 + cos(2 pi t / L)),
                    t = j - D0 - mu, D0 = (L-1)//2.
                    M = 14 reproduces the exact taps to ~5e-15.
  centered_branches change of basis mu -> (mu - 1/2), used by the fp32 GPU
                    path so that Horner runs on [-1/2, 1/2) (same filter).
  split_delay       D/mu convention of reference farrow.py:192-211.
  branch_filter     the shared branch pass (farrow.py:214-229) on the GPU.
  delay_stream      one time-varying delay (farrow.py:253-274): GPU branch
                    pass + the accumulate operator.
  evaluate, evaluate_power_sum, impulse_response
                    the reference's scalar cross-check helpers
                    (farrow.py:146-149, 232-250): one output sample / one
                    L-tap response, used by tests, never by a render.

Filter *design* by constrained least squares (reference farrow.py:74-136)
is offline setup and out of scope; pass its output here.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache
from math import comb

import numpy as np
import torch


@dataclass(frozen=True)
class FarrowFilter:
    """Immutable branch-filter bank (reference farrow.py:42-63).

    poly_order: M, branch_len: L taps per branch, branches: (M+1, L),
    nominal_delay: D0 = (L-1)//2, passband: fraction of Nyquist.
    """

    poly_order: int
    branch_len: int
    branches: np.ndarray
    nominal_delay: int
    passband: float

    def __post_init__(self):
        b = np.asarray(self.branches, dtype=np.float64)
        if b.shape != (self.poly_order + 1, self.branch_len):
            raise ValueError("branches must have shape (M+1, L)")
        b = b.copy()
        b.flags.writeable = False
        object.__setattr__(self, "branches", b)


@dataclass(frozen=True)
class DelaySplit:
    integer_part: int
    fractional_part: float


def split_delay(total_delay, f) -> DelaySplit:
    """D = floor(total - D0), mu = total - D0 - D in [0, 1)."""
    total = float(total_delay)
    if not np.isfinite(total):
        raise ValueError("delay must be finite")
    if total < f.nominal_delay:
        raise ValueError(f"total delay {total} is below the filter latency {f.nominal_delay}")
    d_int = int(np.floor(total - f.nominal_delay))
    mu = total - f.nominal_delay - d_int
    if mu >= 1.0:
        d_int += 1
        mu = total - f.nominal_delay - d_int
    return DelaySplit(integer_part=d_int, fractional_part=mu)


def hann_sinc_taps(L: int, mu) -> np.ndarray:
    """Exact taps h(j, mu), shape (len(mu), L)."""
    mu = np.atleast_1d(np.asarray(mu, dtype=np.float64))
    d0 = (L - 1) // 2
    t = np.arange(L)[None, :] - d0 - mu[:, None]
    w = np.where(np.abs(t) <= L / 2, 0.5 * (1.0 + np.cos(2.0 * np.pi * t / L)), 0.0)
    return np.sinc(t) * w


def _shift_basis(coef: np.ndarray, shift: float) -> np.ndarray:
    """Coefficients of p(x + shift) given p's monomial coefficients (rows)."""
    M = coef.shape[0] - 1
    out = np.zeros_like(coef)
    for j in range(M + 1):
        for k in range(j + 1):
            out[k] += coef[j] * (comb(j, k) * shift ** (j - k))
    return out


@lru_cache(maxsize=32)
def _hann_sinc_cached(L: int, M: int) -> np.ndarray:
    nodes = 4 * (M + 1)
    k = np.arange(nodes)
    x = 0.5 - 0.5 * np.cos(np.pi * (k + 0.5) / nodes)  # Chebyshev nodes on [0, 1]
    v = 2.0 * x - 1.0
    cheb, *_ = np.linalg.lstsq(np.polynomial.chebyshev.chebvander(v, M),
                               hann_sinc_taps(L, x), rcond=None)
    mono_v = np.zeros((M + 1, L))
    for j in range(L):
        p = np.polynomial.chebyshev.cheb2poly(cheb[:, j])
        mono_v[: p.size, j] = p
    centered = mono_v * (2.0 ** np.arange(M + 1))[:, None]  # v = 2 (mu - 1/2)
    out = _shift_basis(centered, -0.5)  # (mu - 1/2)^k -> mu^k
    out.flags.writeable = False
    return out


def hann_sinc(L: int, M: int = 14) -> FarrowFilter:
    """L-tap Hann-windowed sinc as a degree-M Farrow bank (mu in [0,1))."""
    if L < 2 or M < 1:
        raise ValueError("need L >= 2 and M >= 1")
    return FarrowFilter(poly_order=M, branch_len=L, branches=_hann_sinc_cached(int(L), int(M)),
                        nominal_delay=(L - 1) // 2, passband=1.0)


def centered_branches(branches) -> np.ndarray:
    """Rows c'_k with sum_k c'_k (mu - 1/2)^k == sum_k c_k mu^k."""
    return _shift_basis(np.asarray(branches, dtype=np.float64), 0.5)


def as_filter(f) -> FarrowFilter:
    """Accept this module's FarrowFilter or the reference's (same fields)."""
    if isinstance(f, FarrowFilter):
        return f
    try:
        return FarrowFilter(poly_order=int(f.poly_order), branch_len=int(f.branch_len),
                            branches=np.asarray(f.branches), nominal_delay=int(f.nominal_delay),
                            passband=float(getattr(f, "passband", 1.0)))
    except AttributeError as e:  # pragma: no cover - message only
        raise TypeError("expected a FarrowFilter-like object") from e


def _as_signal(x):
    """1-D finite float64 input (numpy or CUDA tensor), reference
    farrow.py:220-225 errors."""
    if isinstance(x, torch.Tensor):
        a = x.to(torch.float64)
        ok = bool(torch.isfinite(a).all()) if a.numel() else True
    else:
        a = np.asarray(x, dtype=np.float64)
        ok = bool(np.all(np.isfinite(a)))
    if a.ndim != 1:
        raise ValueError("input must be 1-D")
    if not ok:
        raise ValueError("input must be finite")
    if a.shape[0] == 0:
        raise ValueError("input must be nonempty")
    return a


def branch_filter(x, f):
    """(M+1, len(x)+L-1) branch streams: the input convolved with every
    branch once (reference farrow.py:214-229), one libmvb launch.  numpy in
    -> numpy out; a CUDA tensor in -> a CUDA tensor out."""
    from . import kernels
    f = as_filter(f)
    return kernels.branch_filter(_as_signal(x), f.branches)


def evaluate(streams, n, split):
    """One output sample: Horner in mu of the branch streams at n - D
    (reference farrow.py:232-241); 0 outside the streams."""
    v = streams.cpu().numpy() if isinstance(streams, torch.Tensor) else np.asarray(streams)
    idx = n - split.integer_part
    if idx < 0 or idx >= v.shape[1]:
        return 0.0
    mu = split.fractional_part
    acc = v[-1, idx]
    for k in range(v.shape[0] - 2, -1, -1):
        acc = acc * mu + v[k, idx]
    return float(acc)


def evaluate_power_sum(streams, n, split):
    """The same sample as an explicit power sum (reference farrow.py:244-250)."""
    v = streams.cpu().numpy() if isinstance(streams, torch.Tensor) else np.asarray(streams)
    idx = n - split.integer_part
    if idx < 0 or idx >= v.shape[1]:
        return 0.0
    mu = split.fractional_part
    return float(sum(v[k, idx] * mu ** k for k in range(v.shape[0])))


def impulse_response(f, mu):
    """h(n, mu) = sum_k c_k(n) mu^k for one fractional delay (reference
    farrow.py:146-149)."""
    f = as_filter(f)
    return (float(mu) ** np.arange(f.poly_order + 1)) @ f.branches


def delay_stream(x, f, tau):
    """x delayed by the per-output-sample delay tau (samples, all >= D0):
    one GPU branch pass and one accumulate launch (reference
    farrow.py:253-274, same errors).  Output length len(tau)."""
    from . import kernels
    from ._dev import require_cuda, to_dev
    f = as_filter(f)
    t = tau.to(torch.float64) if isinstance(tau, torch.Tensor) else np.asarray(tau, np.float64)
    if t.ndim != 1:
        raise ValueError("tau must be 1-D")
    finite = bool(torch.isfinite(t).all()) if isinstance(t, torch.Tensor) else bool(np.all(np.isfinite(t)))
    if not finite:
        raise ValueError("tau must be finite")
    low = bool((t < f.nominal_delay).any()) if isinstance(t, torch.Tensor) else \
        bool(np.any(t < f.nominal_delay))
    if low:
        raise ValueError("tau below the filter latency; pad the input first")
    on_dev = isinstance(x, torch.Tensor) and x.is_cuda
    dev = require_cuda(x.device if on_dev else None)
    streams = kernels.branch_filter(to_dev(_as_signal(x), torch.float64, dev), f.branches)
    td = to_dev(t, torch.float64, dev).reshape(1, -1).contiguous()
    out = torch.zeros(td.shape[1], dtype=torch.float64, device=dev)
    kernels.accumulate_images(out, streams, td, torch.ones_like(td), 0, f.nominal_delay)
    return out if on_dev else out.cpu().numpy()
