"""Static responses, the splice baseline and the comparison metrics on the GPU.

Mirrors reference reference.py (StaticRIR :22-29, ComparisonReport :32-46,
static_rir :67-100, static_render :103-117, full_rate_moving_oracle
:116-130, splice_baseline :133-187, compare :196-251) with the same
arguments, results and ValueErrors.  The tap placement, the convolution and
the block overlap-add run in libmvb (csrc/static.cu: mvb_static_taps,
mvb_static_gather, mvb_block_convolve, mvb_splice_sum); the metrics use
cuFFT through torch.fft in fp64.  No CPU path: every function needs the
library and a CUDA device.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._dev import ptr, require_cuda, stream_handle, to_dev
from .room import as_mic, image_table
from .synth import full_rate_moving_oracle  # noqa: F401  (reference.py:116-130)
from .trajectory import UPSAMPLE_HALFWIDTH

F64 = torch.float64
I64 = torch.int64


@dataclass(frozen=True)
class StaticRIR:
    """Discrete impulse response of a frozen source/mic/room configuration."""

    rate: float
    taps: np.ndarray
    image_count: int
    max_order: int


@dataclass(frozen=True)
class ComparisonReport:
    """snr_db (band-limited interior SNR, capped at 200), envelope_max_jump,
    inst_freq_track (Hz, smoothed over 10 ms), runtime_counts."""

    snr_db: float
    envelope_max_jump: float
    inst_freq_track: np.ndarray
    runtime_counts: dict = field(default_factory=dict)


def _static_taps(room, sources: np.ndarray, mic, rate: float, max_order: int, c: float,
                 d_min: float):
    """Tap trains of B frozen source positions (B, 3) on the device:
    (taps (B, stride) f64, n_taps (B,) host int64, image count)."""
    if max_order < 0:
        raise ValueError("max_order must be >= 0")
    dev = require_cuda()
    t = image_table(room.dims, room.wall_reflection, int(max_order), dev)
    S = t.count
    B = sources.shape[0]
    src = to_dev(np.ascontiguousarray(sources, dtype=np.float64), F64, dev)
    m = to_dev(as_mic(mic).pos, F64, dev)
    base = torch.empty(B, S, dtype=I64, device=dev)
    tau = torch.empty(B, S, dtype=F64, device=dev)
    ker = torch.empty(B, S, 2 * UPSAMPLE_HALFWIDTH + 1, dtype=F64, device=dev)
    st = stream_handle(dev)
    _lib.call("mvb_static_taps", ptr(t.offset[0]), ptr(t.sign[0]), ptr(t.beta[0]), S, ptr(src), B,
              ptr(m), float(rate), float(c), float(d_min), ptr(base), ptr(tau), ptr(ker), st)
    # n_taps = ceil(max tau) + hw + 2   (reference.py:89)
    n_taps = (torch.ceil(tau.max(dim=1).values).to(I64) + UPSAMPLE_HALFWIDTH + 2)
    n_host = n_taps.cpu().numpy()
    stride = int(n_host.max())
    sb, perm = torch.sort(base, dim=1, stable=True)
    taps = torch.empty(B, stride, dtype=F64, device=dev)
    _lib.call("mvb_static_gather", ptr(sb), ptr(perm), ptr(ker), S, B, ptr(n_taps), stride,
              ptr(taps), st)
    return taps, n_taps, n_host, S


def static_rir(room, source_pos, mic, rate, max_order, c=343.0, d_min=0.05) -> StaticRIR:
    """Tap train of the frozen configuration with fractional (windowed-sinc)
    placement of every image (reference.py:67-100)."""
    source_pos = np.asarray(source_pos, dtype=np.float64)
    if not room.contains(source_pos):
        raise ValueError("source position must be inside the room")
    mic = as_mic(mic)
    mic.require_inside(room)
    taps, _, n_host, S = _static_taps(room, source_pos.reshape(1, 3), mic, rate, max_order, c,
                                      d_min)
    return StaticRIR(rate=float(rate), taps=taps[0, :int(n_host[0])].cpu().numpy(),
                     image_count=int(S), max_order=int(max_order))


def _convolve_dev(x: torch.Tensor, h: torch.Tensor) -> torch.Tensor:
    n, nt = x.numel(), h.numel()
    out = torch.empty(n + nt - 1, dtype=F64, device=x.device)
    nt_dev = torch.tensor([nt], dtype=I64, device=x.device)
    _lib.call("mvb_block_convolve", ptr(x), n, n, 0, 1, 0, ptr(h), ptr(nt_dev), nt, out.numel(),
              ptr(out), out.numel(), stream_handle(x.device))
    return out


def static_render(s, rir, rate=None) -> np.ndarray:
    """Plain convolution with a static impulse response; length
    len(s) + len(taps) - 1 (reference.py:103-117), direct fp64 on the GPU."""
    s = np.asarray(s, dtype=np.float64)
    if rate is not None and rate != rir.rate:
        raise ValueError("sample rate does not match the impulse response")
    taps = np.asarray(rir.taps, dtype=np.float64)
    if s.ndim != 1 or taps.ndim != 1 or s.size == 0 or taps.size == 0:
        raise ValueError("signal and taps must be nonempty 1-D arrays")
    dev = require_cuda()
    return _convolve_dev(to_dev(s, F64, dev), to_dev(taps, F64, dev)).cpu().numpy()


def _block_support(b, n, hop, cf, n_blocks):
    start = b * hop
    stop = min(n, start + hop)
    end = min(n, stop + cf) if (cf > 0 and b < n_blocks - 1) else stop
    return start, end


def splice_baseline(s, traj, room, mic, block_hop, crossfade, cfg) -> np.ndarray:
    """Block-frozen render (reference.py:133-187): the source frozen at each
    block start, one static response per block, blocks windowed (butt-joined
    or linearly cross-faded) and overlap-added.  All blocks' responses are
    built in one launch and all pieces convolved in one launch."""
    s = np.asarray(s, dtype=np.float64)
    if block_hop < 1 or int(block_hop) != block_hop:
        raise ValueError("block_hop must be a positive integer")
    block_hop = int(block_hop)
    crossfade = int(crossfade)
    if crossfade < 0 or crossfade > block_hop:
        raise ValueError("crossfade must lie in [0, block_hop]")
    if traj.rate != cfg.audio_rate:
        raise ValueError("trajectory rate must equal the audio rate")
    n = s.size
    if n == 0:
        raise ValueError("signal must be nonempty")
    n_blocks = max(1, -(-n // block_hop))
    rows = np.minimum(np.arange(n_blocks) * block_hop, len(traj) - 1)
    sources = traj.positions[rows]
    for p in sources:
        if not room.contains(p):
            raise ValueError("source position must be inside the room")
    mic = as_mic(mic)
    mic.require_inside(room)
    taps, n_taps, n_host, _ = _static_taps(room, sources, mic, cfg.audio_rate, cfg.max_order,
                                           cfg.sound_speed, cfg.d_min)
    dev = taps.device
    spans = [(_block_support(b, n, block_hop, crossfade, n_blocks)) for b in range(n_blocks)]
    plen = np.array([hi - lo for lo, hi in spans], dtype=np.int64) + n_host - 1
    max_piece = int(plen.max())
    x = to_dev(s, F64, dev)
    pieces = torch.empty(n_blocks, max_piece, dtype=F64, device=dev)
    st = stream_handle(dev)
    _lib.call("mvb_block_convolve", ptr(x), n, block_hop, crossfade, n_blocks, 1, ptr(taps),
              ptr(n_taps), taps.shape[1], max_piece, ptr(pieces), max_piece, st)
    out_len = n + int(n_host.max()) - 1
    out = torch.empty(out_len, dtype=F64, device=dev)
    _lib.call("mvb_splice_sum", ptr(pieces), max_piece, n, block_hop, crossfade, n_blocks,
              ptr(n_taps), max_piece, ptr(out), out_len, st)
    return out.cpu().numpy()


def _brickwall(x: torch.Tensor, rate: float, cutoff_hz: float) -> torch.Tensor:
    """reference.py:190-194 on the device (cuFFT)."""
    n = x.numel()
    spec = torch.fft.rfft(x)
    freqs = torch.arange(n // 2 + 1, dtype=F64, device=x.device) * (1.0 / (n * (1.0 / rate)))
    spec = torch.where(freqs > cutoff_hz, torch.zeros_like(spec), spec)
    return torch.fft.irfft(spec, n)


def _analytic(x: torch.Tensor) -> torch.Tensor:
    """Analytic signal by the FFT (the scipy.signal.hilbert construction)."""
    n = x.numel()
    h = torch.zeros(n, dtype=F64, device=x.device)
    h[0] = 1.0
    if n % 2 == 0:
        h[n // 2] = 1.0
        h[1:n // 2] = 2.0
    else:
        h[1:(n + 1) // 2] = 2.0
    return torch.fft.ifft(torch.fft.fft(x.to(torch.complex128)) * h)


def _convolve_same(x: torch.Tensor, k: torch.Tensor) -> torch.Tensor:
    """numpy.convolve(x, k, mode="same")."""
    m, K = x.numel(), k.numel()
    full = torch.nn.functional.conv1d(x.view(1, 1, -1), torch.flip(k, [0]).view(1, 1, -1),
                                      padding=K - 1).view(-1)
    n_out = max(m, K)
    off = (min(m, K) - 1) // 2
    return full[off:off + n_out]


def compare(a, b, passband=0.8, rate=16000.0, interior=0.05, runtime_counts=None
            ) -> ComparisonReport:
    """Measure a against reference b (reference.py:196-251): common length,
    band-limited interior SNR (capped at 200 dB), analytic-signal envelope
    jump and 10 ms-smoothed instantaneous frequency of a."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    n = min(a.size, b.size)
    if n < 16:
        raise ValueError("signals too short to compare")
    if not 0.0 < passband <= 1.0:
        raise ValueError("passband must be in (0, 1]")
    if not 0.0 <= interior < 0.5:
        raise ValueError("interior must be in [0, 0.5)")
    dev = require_cuda()
    ad = to_dev(a[:n], F64, dev)
    bd = to_dev(b[:n], F64, dev)
    lo = int(np.floor(interior * n))
    hi = n - lo
    if passband < 1.0:
        a_band = _brickwall(ad, rate, passband * rate / 2.0)
        b_band = _brickwall(bd, rate, passband * rate / 2.0)
    else:
        a_band, b_band = ad, bd
    ref_energy = float(torch.sum(b_band[lo:hi] ** 2))
    if ref_energy <= 0.0:
        raise ValueError("reference has no energy on the interior")
    err_energy = float(torch.sum((a_band[lo:hi] - b_band[lo:hi]) ** 2))
    snr = 200.0 if err_energy == 0.0 else min(200.0, 10.0 * np.log10(ref_energy / err_energy))
    an = _analytic(ad)
    env = torch.abs(an)[lo:hi]
    env_jump = float(torch.max(torch.abs(torch.diff(env)))) if env.numel() > 1 else 0.0
    phase_step = torch.angle(an[1:] * torch.conj(an[:-1]))
    # true division (torch rewrites `tensor / python scalar` as a reciprocal multiply)
    inst = (phase_step * rate) / torch.tensor(2.0 * np.pi, dtype=F64, device=dev)
    smooth = max(1, int(round(0.010 * rate)))
    inst = _convolve_same(inst, torch.full((smooth,), 1.0 / smooth, dtype=F64, device=dev))
    track = inst[lo:max(lo + 1, hi - 1)].cpu().numpy()
    return ComparisonReport(snr_db=float(snr), envelope_max_jump=env_jump, inst_freq_track=track,
                            runtime_counts=dict(runtime_counts or {}))
