"""Source / receiver paths and the hierarchical track resampling constants.

Trajectory mirrors reference trajectory.py:29-60.  The decimation decision
(trajectory.py:279-298: low-pass only when Nyquist_out < bandwidth <
2 Nyquist_out) is taken on the device with libmvb's own fp64 FFT; the per-factor
Kaiser-windowed-sinc phase table (trajectory.py:235-257) is a cached host
constant like the reference's lru_cache, from which two device constants
are derived:

  * the transposed table (65, N) read by the exact fp64 path, and
  * the degree-8 refit of every table column in u = 2 r / N - 1 that the
    fast path evaluates per sample: exact track on each
    coarse interval to < 1e-9 m at the configs' rates.
"""

from __future__ import annotations

import os

from dataclasses import dataclass
from functools import lru_cache

import numpy as np
import torch

from . import _lib
from ._dev import h2d, pinned_scratch, ptr, require_cuda, stream_handle, to_dev

UPSAMPLE_HALFWIDTH = 32
UPSAMPLE_KAISER_BETA = 7.857
FIT_DEGREE = 8
PIN_BYTES = 1 << 20  # Trajectory positions at least this large live in pinned host memory


@dataclass(frozen=True)
class Trajectory:
    """rate: positions per second; positions (T, 3) metres."""

    rate: float
    positions: np.ndarray

    def __post_init__(self):
        if self.rate <= 0:
            raise ValueError("trajectory rate must be > 0")
        p = np.asarray(self.positions, dtype=np.float64)
        if p.ndim != 2 or p.shape[1] != 3 or p.shape[0] < 1:
            raise ValueError("positions must be a (T, 3) array with T >= 1")
        if not np.all(np.isfinite(p)):
            raise ValueError("positions must be finite")
        if p.nbytes >= PIN_BYTES:
            # large paths are kept page-locked: every render sends them by
            # DMA straight from this copy (no staging memcpy per render)
            from ._staging import pinned_copy
            p = pinned_copy(p)
        else:
            p = p.copy()
        p.flags.writeable = False
        object.__setattr__(self, "positions", p)
        object.__setattr__(self, "rate", float(self.rate))

    def __len__(self):
        return self.positions.shape[0]

    @property
    def duration(self):
        return len(self) / self.rate


@lru_cache(maxsize=16)
def phase_table(factor: int) -> np.ndarray:
    """(factor, 65) Kaiser(7.857)-windowed sinc rows at r/factor - i, each
    normalised to sum 1 (constant input passes exactly)."""
    hw = UPSAMPLE_HALFWIDTH
    offs = np.arange(-hw, hw + 1, dtype=np.float64)
    tab = np.empty((factor, offs.size))
    i0b = np.i0(UPSAMPLE_KAISER_BETA)
    for r in range(factor):
        arg = r / factor - offs
        inside = np.abs(arg) <= hw
        win = np.zeros_like(arg)
        z = np.clip(arg / hw, -1.0, 1.0)
        win[inside] = np.i0(UPSAMPLE_KAISER_BETA * np.sqrt(1.0 - z[inside] ** 2)) / i0b
        row = np.sinc(arg) * win
        tab[r] = row / row.sum()
    tab.flags.writeable = False
    return tab


@lru_cache(maxsize=16)
def phase_fit(factor: int) -> np.ndarray:
    """(FIT_DEGREE+1, 65): table[r, c] ~= sum_p fit[p, c] u^p, u = 2r/N - 1."""
    tab = phase_table(factor)
    u = 2.0 * np.arange(factor) / factor - 1.0
    V = u[:, None] ** np.arange(FIT_DEGREE + 1)[None, :]
    fit, *_ = np.linalg.lstsq(V, tab, rcond=None)
    fit.flags.writeable = False
    return fit


@lru_cache(maxsize=16)
def negative_mass(factor: int) -> float:
    """max over phases of the summed negative weights (overshoot bound)."""
    tab = phase_table(factor)
    return float(np.max(np.sum(np.where(tab < 0, -tab, 0.0), axis=1)))


_DEV_CONST: dict = {}


def device_constants(factor: int, device) -> dict:
    """Transposed table and polynomial refit of `factor` on `device` (cached)."""
    key = (int(factor), str(device))
    c = _DEV_CONST.get(key)
    if c is None:
        c = {
            "tableT": to_dev(np.ascontiguousarray(phase_table(factor).T), torch.float64, device),
            "fit": to_dev(phase_fit(factor), torch.float64, device),
            "negsum": negative_mass(factor),
        }
        _DEV_CONST[key] = c
    return c


# MVB_BW_CUFFT=1: the bandwidth decision through cuFFT (round-1 route), for A/B
# measurements only; the default is libmvb's own FFT
_BW_CUFFT = os.environ.get("MVB_BW_CUFFT") == "1"


def bandwidth_batch(x: torch.Tensor, rate: float, energy_fraction: float = 0.99) -> np.ndarray:
    return bandwidth_batch_async(x, rate, energy_fraction)()


def bandwidth_batch_async(x: torch.Tensor, rate: float, energy_fraction: float = 0.99,
                          slot: str = "bandwidth_index"):
    """bandwidth_batch, split: enqueues the kernels and the readback, returns
    a function that waits for the readback and returns the bandwidths (the
    caller may enqueue more device work before calling it; `finish(False)`
    reads the pinned buffer without waiting -- a render plan's captured
    staging, whose replay the caller waited for).  `slot` names
    the pinned readback buffer (one pending readback per name)."""
    """Per-path smallest frequency holding `energy_fraction` of the
    mean-removed displacement power, max over axes (reference
    trajectory.py:316-339), for x (G, T, 3) on the device -> host (G,).
    One libmvb call (mvb_path_spectrum_index: mean removal, the hand-written
    fp64 FFT, energy index per axis), one small device->host copy.
    Frequencies follow numpy.fft.rfftfreq: k * (1 / (T * (1 / rate)))."""
    G, T, _ = x.shape
    if T < 2 or G == 0:
        return lambda wait=True: np.zeros(G)
    x = x.contiguous()
    st = stream_handle(x.device)
    F = T // 2 + 1
    k = torch.empty(G * 3, dtype=torch.int64, device=x.device)
    if _BW_CUFFT:  # diagnostic A/B only: the round-1 cuFFT route
        scratch = torch.empty(3 * G * _lib.SPEC_PARTS, dtype=torch.float64, device=x.device)
        xc = torch.empty_like(x)
        _lib.call("mvb_center_paths", ptr(x), G, T, ptr(scratch), ptr(xc), st)
        spec = torch.fft.rfft(xc, dim=1).contiguous()
        _lib.call("mvb_spectrum_index", ptr(spec), G, F, float(energy_fraction), ptr(scratch),
                  ptr(k), st)
    else:
        scratch = torch.empty(int(_lib.lib().mvb_path_spectrum_scratch(G, T)),
                              dtype=torch.float64, device=x.device)
        _lib.call("mvb_path_spectrum_index", ptr(x), G, T, float(energy_fraction), ptr(scratch),
                  ptr(k), st)
    host = pinned_scratch(slot, k.numel(), k.dtype)
    host.copy_(k, non_blocking=True)
    done = torch.cuda.Event()
    done.record()

    def finish(wait=True):
        if wait:  # (render plans replay a captured copy and wait themselves)
            done.synchronize()
        kh = host.numpy().copy().reshape(G, 3)
        hz = np.minimum(kh, F - 1) * (1.0 / (T * (1.0 / rate)))
        return np.where(kh < 0, 0.0, hz).max(axis=1)
    return finish


def bandwidth_estimate(traj: Trajectory, energy_fraction: float = 0.99) -> float:
    """Smallest frequency holding `energy_fraction` of the mean-removed
    displacement power, max over the three axes; 0 Hz for a constant or
    single-sample path (reference trajectory.py:316-339, same error)."""
    if not 0.0 < energy_fraction < 1.0:
        raise ValueError("energy_fraction must be in (0, 1)")
    if len(traj) < 2:
        return 0.0
    pos = to_dev(np.asarray(traj.positions, dtype=np.float64), torch.float64, require_cuda())
    return float(bandwidth_batch(pos[None], traj.rate, energy_fraction)[0])


def bandwidth_estimate_dev(pos: torch.Tensor, rate: float, energy_fraction: float = 0.99) -> float:
    return float(bandwidth_batch(pos[None], rate, energy_fraction)[0])


def lowpass_batch(x: torch.Tensor, rate: float, cutoff: float) -> torch.Tensor:
    """Raised-cosine-edged FFT low-pass with odd reflection padding
    (reference trajectory.py:214-232) of x (G, T, 3) on the device: one
    libmvb call (mvb_lowpass_paths, hand-written fp64 FFT)."""
    x = x.to(torch.float64).contiguous()
    G, T, _ = x.shape
    out = torch.empty_like(x)
    scratch = torch.empty(int(_lib.lib().mvb_lowpass_scratch(G, T)), dtype=torch.float64,
                          device=x.device)
    _lib.call("mvb_lowpass_paths", ptr(x), G, T, float(rate), float(cutoff), ptr(scratch),
              ptr(out), stream_handle(x.device))
    return out


def lowpass_columns_dev(x: torch.Tensor, rate: float, cutoff: float) -> torch.Tensor:
    return lowpass_batch(x[None], rate, cutoff)[0].contiguous()


def decimate_batch(x: torch.Tensor, rate: float, factor: int, bw: torch.Tensor | None = None
                   ) -> torch.Tensor:
    """Coarse paths x[:, ::N] of x (G, T, 3), each low-passed first when its
    measured bandwidth lies in (Nyquist_out, 2 Nyquist_out); the low-pass
    runs only for those paths.  `bw` may carry the paths' bandwidths
    (bandwidth_batch, host) when several factors are needed."""
    raw = x[:, ::factor]
    if x.shape[1] < 2 or factor == 1:
        return raw
    nyq = 0.5 * rate / factor
    if bw is None:
        bw = bandwidth_batch(x, rate)
    need = np.nonzero((bw > nyq) & (bw < 2.0 * nyq))[0]  # low-pass only the paths that need it
    if need.size == 0:
        return raw
    if need.size == x.shape[0]:
        return lowpass_batch(x, rate, 0.9 * nyq)[:, ::factor]
    idx = h2d(need.astype(np.int64), x.device)
    out = raw.clone()
    out[idx] = lowpass_batch(x[idx], rate, 0.9 * nyq)[:, ::factor]
    return out


def decimate_dev(pos: torch.Tensor, rate: float, factor: int) -> torch.Tensor:
    """Coarse path pos[::N] (device), low-passed first when the measured
    bandwidth lies in (Nyquist_out, 2 Nyquist_out)."""
    factor = int(factor)
    if factor < 1:
        raise ValueError("decimation factor must be a positive integer")
    if factor == 1:
        return pos
    nyq = 0.5 * rate / factor
    src = pos
    if pos.shape[0] >= 2:
        bw = bandwidth_estimate_dev(pos, rate)
        if nyq < bw < 2.0 * nyq:
            src = lowpass_columns_dev(pos, rate, 0.9 * nyq)
    return src[::factor].contiguous()


def decimate(traj: Trajectory, factor: int) -> Trajectory:
    """Reference-API decimate (trajectory.py:279-298), computed on the GPU."""
    if int(factor) != factor or factor < 1:
        raise ValueError("decimation factor must be a positive integer")
    if factor == 1:
        return traj
    dev = require_cuda()
    p = decimate_dev(to_dev(traj.positions, torch.float64, dev), traj.rate, int(factor))
    return Trajectory(rate=traj.rate / factor, positions=p.cpu().numpy())


def bandlimited_upsample(samples, factor: int, out_len: int) -> np.ndarray:
    """Windowed-sinc interpolation by `factor` (trajectory.py:260-276) on
    the GPU (mvb_upsample_streams); exact on constants, endpoints hold."""
    x = np.asarray(samples, dtype=np.float64)
    if x.ndim != 1 or x.size == 0:
        raise ValueError("samples must be a nonempty 1-D sequence")
    if factor < 1 or int(factor) != factor:
        raise ValueError("factor must be a positive integer")
    factor = int(factor)
    if factor == 1:
        if out_len <= x.size:
            return x[:out_len].copy()
        return np.concatenate([x, np.full(out_len - x.size, x[-1])])
    dev = require_cuda()
    xc = to_dev(x, torch.float64, dev)
    tab = to_dev(phase_table(factor), torch.float64, dev)
    out = torch.empty(out_len, dtype=torch.float64, device=dev)
    _lib.call("mvb_upsample_streams", ptr(xc), 1, x.size, ptr(tab), factor, tab.shape[1], out_len,
              ptr(out), stream_handle(dev))
    return out.cpu().numpy()
