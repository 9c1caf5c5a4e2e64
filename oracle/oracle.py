"""CPU oracle for the moving-source path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() (as the checker) and bench.py's
cpu_baseline / ``--impl reference`` leg may import this module.  The product
package (paper_2508_03065_b200) never does, and has no CPU fallback.

The heavy loops are the C restatement in mvb_oracle.c (built by the Makefile
next to this file into _build/libmvb_oracle.so).  The numpy helpers below
restate the small host-side pieces of the reference (all paths relative to
/root/reference/pkg/src/moverb/):

  phase_table          trajectory.py:235-257  (_phase_table)
  bandwidth_estimate   trajectory.py:316-339
  lowpass_columns      trajectory.py:214-232  (_lowpass_columns)
  decimate_positions   trajectory.py:279-298  (decimate)
  hann_sinc_taps       the configs' 32/64-tap Hann-windowed sinc
                       (SURVEY.md 8c-ii, H6 window convention)
  render               synth.py:273-294 + 194-258 for any tier list, fixed or
                       moving receiver, evaluated over a window of samples.

Parity status: pinned.  tests/test_oracle.py checks every function here
against golden vectors produced by the reference itself
(tests/golden/make_golden.py imports /root/reference in the build container).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libmvb_oracle.so")
_lib = None

UPSAMPLE_HALFWIDTH = 32  # trajectory.py:24
UPSAMPLE_KAISER_BETA = 7.857  # trajectory.py:26
BLOCK = 32  # synth.py:36


def build(force: bool = False) -> str:
    """Compile mvb_oracle.c with the committed Makefile (gcc, no GPU)."""
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "mvb_oracle.c"))
    ):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, i32, d = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        P = ctypes.c_void_p
        L.orc_image_count.restype = i64
        L.orc_image_count.argtypes = [ctypes.c_int]
        L.orc_enumerate.restype = i64
        L.orc_enumerate.argtypes = [P, P, ctypes.c_int, P, P, P, P, P, P, P]
        L.orc_distance.restype = None
        L.orc_distance.argtypes = [P, P, P, P, i64, i64, P]
        L.orc_upsample.restype = None
        L.orc_upsample.argtypes = [P, i64, P, i64, i64, i64, P]
        L.orc_accumulate.restype = None
        L.orc_accumulate.argtypes = [P, i64, P, i64, i64, P, P, i64, i64, i64]
        L.orc_branch_filter.restype = None
        L.orc_branch_filter.argtypes = [P, i64, P, i64, i64, P]
        L.orc_render_window.restype = None
        L.orc_render_window.argtypes = [P, i64, i64, P, ctypes.c_int]
        L.orc_tracks_window.restype = None
        L.orc_tracks_window.argtypes = [P, i64, i64, P, ctypes.c_int]
        L.orc_track_max.restype = d
        L.orc_track_max.argtypes = [P, ctypes.c_int]
        L.orc_hann_sinc_gather.restype = None
        L.orc_hann_sinc_gather.argtypes = [P, P, i64, i64, i64, i64, P, ctypes.c_int]
        L.orc_default_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def default_threads() -> int:
    return int(lib().orc_default_threads())


# ---------------------------------------------------------------------------
# image lattice


@dataclass
class Images:
    """Canonical-order image table (room.py:175-187 as_arrays + j/lattice)."""

    j: np.ndarray  # (S,3) int32 signed mirror index
    lattice: np.ndarray  # (S,3) int32
    parity: np.ndarray  # (S,3) int32 0/1
    order: np.ndarray  # (S,) int32
    beta: np.ndarray  # (S,) f64
    offset: np.ndarray  # (S,3) f64
    sign: np.ndarray  # (S,3) f64

    def __len__(self):
        return int(self.order.shape[0])

    def take(self, idx) -> "Images":
        return Images(*(getattr(self, f)[idx] for f in
                        ("j", "lattice", "parity", "order", "beta", "offset", "sign")))


def image_count(max_order: int) -> int:
    return int(lib().orc_image_count(int(max_order)))


def enumerate_images(dims, walls, max_order: int) -> Images:
    dims = _f64(dims).reshape(3)
    walls = _f64(np.broadcast_to(np.asarray(walls, dtype=np.float64), (6,)))
    S = image_count(max_order)
    j = np.empty((S, 3), np.int32)
    lat = np.empty((S, 3), np.int32)
    par = np.empty((S, 3), np.int32)
    order = np.empty(S, np.int32)
    beta = np.empty(S)
    off = np.empty((S, 3))
    sign = np.empty((S, 3))
    n = lib().orc_enumerate(_p(dims), _p(walls), int(max_order), _p(j), _p(lat), _p(par),
                            _p(order), _p(beta), _p(off), _p(sign))
    assert n == S
    return Images(j, lat, par, order, beta, off, sign)


# ---------------------------------------------------------------------------
# kernel trio (_kernels.py)


def distance_streams(offset, sign, mic, pos) -> np.ndarray:
    offset, sign, mic, pos = _f64(offset), _f64(sign), _f64(mic), _f64(pos)
    S, T = offset.shape[0], pos.shape[0]
    out = np.empty((S, T))
    lib().orc_distance(_p(offset), _p(sign), _p(mic), _p(pos), S, T, _p(out))
    return out


def upsample_stream(coarse, table, factor: int, out_len: int) -> np.ndarray:
    coarse, table = _f64(coarse), _f64(table)
    out = np.empty(out_len)
    lib().orc_upsample(_p(coarse), coarse.size, _p(table), int(factor), table.shape[1],
                       int(out_len), _p(out))
    return out


def accumulate_images(out, streams, tau, amp, offset: int, d0: int) -> np.ndarray:
    streams, tau, amp = _f64(streams), _f64(tau), _f64(amp)
    assert out.dtype == np.float64 and out.flags.c_contiguous
    lib().orc_accumulate(_p(out), out.size, _p(streams), streams.shape[0], streams.shape[1],
                         _p(tau), _p(amp), tau.shape[0], int(offset), int(d0))
    return out


def branch_filter(x, branches) -> np.ndarray:
    x, b = _f64(x), _f64(branches)
    nb, L = b.shape
    out = np.empty((nb, x.size + L - 1))
    lib().orc_branch_filter(_p(x), x.size, _p(b), nb, L, _p(out))
    return out


# ---------------------------------------------------------------------------
# trajectory helpers (numpy restatements)


_TABLES: dict = {}


def phase_table(factor: int) -> np.ndarray:
    """Kaiser(beta=7.857, hw=32) windowed sinc, one row per output phase,
    rows normalised to sum 1 (trajectory.py:235-257)."""
    factor = int(factor)
    if factor in _TABLES:
        return _TABLES[factor]
    hw = UPSAMPLE_HALFWIDTH
    taps = np.arange(-hw, hw + 1, dtype=np.float64)
    rows = []
    for r in range(factor):
        x = r / factor - taps
        live = np.abs(x) <= hw
        win = np.zeros_like(x)
        z = np.clip(x / hw, -1.0, 1.0)
        win[live] = np.i0(UPSAMPLE_KAISER_BETA * np.sqrt(1.0 - z[live] ** 2)) / np.i0(
            UPSAMPLE_KAISER_BETA)
        k = np.sinc(x) * win
        rows.append(k / k.sum())
    tab = np.array(rows)
    _TABLES[factor] = tab
    return tab


def bandwidth_estimate(pos, rate: float, energy_fraction: float = 0.99) -> float:
    """Largest per-axis 99%-energy frequency of the mean-removed path."""
    pos = _f64(pos)
    n = pos.shape[0]
    if n < 2:
        return 0.0
    freqs = np.fft.rfftfreq(n, 1.0 / rate)
    worst = 0.0
    for ax in range(3):
        col = pos[:, ax] - pos[:, ax].mean()
        pw = np.abs(np.fft.rfft(col)) ** 2
        tot = pw.sum()
        if tot <= 0:
            continue
        k = int(np.searchsorted(np.cumsum(pw) / tot, energy_fraction))
        worst = max(worst, float(freqs[min(k, freqs.size - 1)]))
    return worst


def lowpass_columns(x, rate: float, cutoff: float) -> np.ndarray:
    """Raised-cosine-edged FFT low-pass with odd-reflection padding."""
    x = _f64(x)
    n = x.shape[0]
    pad = min(n - 1, max(16, n // 4))
    out = np.empty_like(x)
    for ax in range(x.shape[1]):
        c = x[:, ax]
        head = 2 * c[0] - c[pad:0:-1]
        tail = 2 * c[-1] - c[-2:-pad - 2:-1]
        ext = np.concatenate([head, c, tail])
        f = np.fft.rfftfreq(ext.size, 1.0 / rate)
        g = np.ones_like(f)
        lo, hi = 0.8 * cutoff, cutoff
        band = (f > lo) & (f <= hi)
        g[band] = 0.5 * (1 + np.cos(np.pi * (f[band] - lo) / (hi - lo)))
        g[f > hi] = 0.0
        out[:, ax] = np.fft.irfft(np.fft.rfft(ext) * g, ext.size)[pad:pad + n]
    return out


def decimate_positions(pos, rate: float, factor: int) -> np.ndarray:
    """pos[::N], low-passed first only when Nyquist_out < bw < 2 Nyquist_out."""
    pos = _f64(pos)
    factor = int(factor)
    if factor == 1:
        return pos
    nyq = 0.5 * rate / factor
    if pos.shape[0] >= 2:
        bw = bandwidth_estimate(pos, rate)
        if nyq < bw < 2.0 * nyq:
            pos = lowpass_columns(pos, rate, 0.9 * nyq)
    return np.ascontiguousarray(pos[::factor])


# ---------------------------------------------------------------------------
# fractional-delay filter helpers


def hann_sinc_taps(L: int, mu) -> np.ndarray:
    """h(j, mu) = sinc(t) 0.5(1+cos(2 pi t / L)), t = j - (L-1)//2 - mu."""
    mu = np.atleast_1d(np.asarray(mu, dtype=np.float64))
    d0 = (L - 1) // 2
    t = np.arange(L)[None, :] - d0 - mu[:, None]
    w = np.where(np.abs(t) <= L / 2, 0.5 * (1 + np.cos(2 * np.pi * t / L)), 0.0)
    return np.sinc(t) * w


# ---------------------------------------------------------------------------
# render


class _Scene(ctypes.Structure):
    _fields_ = [
        ("S", ctypes.c_int64),
        ("offset", ctypes.c_void_p),
        ("sign", ctypes.c_void_p),
        ("beta", ctypes.c_void_p),
        ("factor", ctypes.c_void_p),
        ("coarse_off", ctypes.c_void_p),
        ("coarse_len", ctypes.c_void_p),
        ("coarse", ctypes.c_void_p),
        ("table_off", ctypes.c_void_p),
        ("tables", ctypes.c_void_p),
        ("ntaps", ctypes.c_int64),
        ("pos", ctypes.c_void_p),
        ("mic", ctypes.c_void_p),
        ("mic_moving", ctypes.c_int32),
        ("T", ctypes.c_int64),
        ("streams", ctypes.c_void_p),
        ("nb", ctypes.c_int64),
        ("ls", ctypes.c_int64),
        ("shift", ctypes.c_int64),
        ("d0", ctypes.c_int64),
        ("rate", ctypes.c_double),
        ("c", ctypes.c_double),
        ("d_min", ctypes.c_double),
    ]


class OracleScene:
    """Everything the reference's render needs, built on the CPU.

    tiers: list of (max_order, N) ascending in max_order; images of order
    <= tiers[0][0] use N0, etc.  The reference's (order_split K, decimation N)
    is tiers=[(K, 1), (max_order, N)] (synth.py:281-287).  mic is (3,) or
    (T,3) for a moving receiver (coarse tiers use mic[::N] likewise).
    """

    def __init__(self, s, pos, mic, dims, walls, max_order, tiers, branches, rate,
                 c=343.0, d_min=0.05, images: Images | None = None):
        self.s = _f64(s)
        self.pos = _f64(pos)
        self.T = self.pos.shape[0]
        mic = _f64(mic)
        self.mic_moving = mic.ndim == 2
        self.mic = mic
        self.rate, self.c, self.d_min = float(rate), float(c), float(d_min)
        br = _f64(branches)
        self.nb, self.L = br.shape
        self.d0 = (self.L - 1) // 2
        self.images = images if images is not None else enumerate_images(dims, walls, max_order)
        S = len(self.images)
        order = self.images.order
        factor = np.empty(S, np.int64)
        assigned = np.zeros(S, bool)
        for mo, N in tiers:
            sel = (order <= mo) & ~assigned
            factor[sel] = int(N)
            assigned |= sel
        if not assigned.all():
            raise ValueError("tiers do not cover every image order")
        self.factor = factor
        # coarse distance rows per decimated image
        coarse_rows, coarse_off, coarse_len = [], np.zeros(S, np.int64), np.ones(S, np.int64)
        tables, table_off = [np.zeros(1)], np.zeros(S, np.int64)
        tab_start = {}
        cur, tcur = 0, 1
        for N in sorted(set(factor.tolist())):
            if N == 1:
                continue
            sel = np.nonzero(factor == N)[0]
            cpos = decimate_positions(self.pos, self.rate, N)
            cmic = decimate_positions(self.mic, self.rate, N) if self.mic_moving else self.mic
            K = cpos.shape[0]
            if self.mic_moving:
                d = np.empty((sel.size, K))
                for r, i in enumerate(sel):
                    off, sg = self.images.offset[i], self.images.sign[i]
                    dx = off[0] + sg[0] * cpos[:, 0] - cmic[:, 0]
                    dy = off[1] + sg[1] * cpos[:, 1] - cmic[:, 1]
                    dz = off[2] + sg[2] * cpos[:, 2] - cmic[:, 2]
                    d[r] = np.sqrt(dx * dx + dy * dy + dz * dz)
            else:
                d = distance_streams(self.images.offset[sel], self.images.sign[sel], self.mic, cpos)
            coarse_rows.append(d.reshape(-1))
            coarse_off[sel] = cur + np.arange(sel.size) * K
            coarse_len[sel] = K
            cur += sel.size * K
            tab = phase_table(N)
            tab_start[N] = tcur
            tables.append(tab.reshape(-1))
            tcur += tab.size
            table_off[sel] = tab_start[N]
        self.coarse = np.concatenate(coarse_rows) if coarse_rows else np.zeros(1)
        self.coarse_off, self.coarse_len = coarse_off, coarse_len
        self.tables = np.concatenate(tables)
        self.table_off = table_off
        self.branches = br
        self.streams = branch_filter(self.s, br)
        self._keep = []

    def _struct(self, images_idx=None) -> _Scene:
        im = self.images
        if images_idx is None:
            arrs = dict(offset=im.offset, sign=im.sign, beta=im.beta, factor=self.factor,
                        coarse_off=self.coarse_off, coarse_len=self.coarse_len,
                        table_off=self.table_off)
        else:
            arrs = dict(offset=im.offset[images_idx], sign=im.sign[images_idx],
                        beta=im.beta[images_idx], factor=self.factor[images_idx],
                        coarse_off=self.coarse_off[images_idx],
                        coarse_len=self.coarse_len[images_idx],
                        table_off=self.table_off[images_idx])
        arrs = {k: np.ascontiguousarray(v) for k, v in arrs.items()}
        self._keep.append(arrs)
        sc = _Scene()
        sc.S = arrs["beta"].shape[0]
        for k in ("offset", "sign", "beta", "factor", "coarse_off", "coarse_len", "table_off"):
            setattr(sc, k, _p(arrs[k]))
        sc.coarse = _p(self.coarse)
        sc.tables = _p(self.tables)
        sc.ntaps = 2 * UPSAMPLE_HALFWIDTH + 1
        sc.pos = _p(self.pos)
        sc.mic = _p(self.mic)
        sc.mic_moving = int(self.mic_moving)
        sc.T = self.T
        sc.streams = _p(self.streams)
        sc.nb, sc.ls = self.streams.shape
        sc.shift = self.L
        sc.d0 = self.d0
        sc.rate, sc.c, sc.d_min = self.rate, self.c, self.d_min
        return sc

    def track_max(self, nthreads: int = 0) -> float:
        """max d over images and t < T (synth.py:201).  Exact: the full
        per-sample scan is restricted to images whose coarse (or exact) range
        can reach the max -- every excluded image is provably below it."""
        S = len(self.images)
        coarse_max = np.empty(S)
        for i in range(S):
            if self.factor[i] == 1:
                coarse_max[i] = np.inf
            else:
                o, k = self.coarse_off[i], self.coarse_len[i]
                coarse_max[i] = self.coarse[o:o + k].max()
        full = np.nonzero(self.factor == 1)[0]
        best = -1.0
        if full.size:
            best = lib().orc_track_max(ctypes.byref(self._struct(full)), nthreads)
        dec = np.nonzero(self.factor != 1)[0]
        if dec.size:
            # phase-0 rows are ~unit impulses, so each coarse max is attained
            # to ~1e-12 m; band-limited reconstruction overshoot of these
            # slowly varying tracks stays far below 1 m, so every image that
            # could hold the max is in `cand` and is scanned exactly
            lo = max(best, coarse_max[dec].max())
            cand = dec[coarse_max[dec] >= lo - 1.0]
            best = max(best, lib().orc_track_max(ctypes.byref(self._struct(cand)), nthreads))
        return best

    def out_len(self, nthreads: int = 0) -> int:
        tau_max = self.rate * self.track_max(nthreads) / self.c
        return self.s.size + int(math.ceil(tau_max)) + self.L  # synth.py:211-212: len(s)

    def render_window(self, n0: int, n1: int, nthreads: int = 0) -> np.ndarray:
        out = np.empty(max(0, n1 - n0))
        sc = self._struct()
        lib().orc_render_window(ctypes.byref(sc), int(n0), int(n1), _p(out), nthreads)
        return out

    def render(self, nthreads: int = 0) -> np.ndarray:
        return self.render_window(0, self.out_len(nthreads), nthreads)

    def tracks_window(self, n0: int, n1: int, nthreads: int = 0) -> np.ndarray:
        """(S, n1 - n0) distance tracks of every image (the reference's
        values: exact per-sample or 65-tap upsampled, hold-extended)."""
        out = np.empty((len(self.images), max(0, n1 - n0)))
        sc = self._struct()
        lib().orc_tracks_window(ctypes.byref(sc), int(n0), int(n1), _p(out), nthreads)
        return out

    def hann_sinc_gather(self, n0: int, n1: int, nthreads: int = 0) -> np.ndarray:
        out = np.empty(max(0, n1 - n0))
        sc = self._struct()
        lib().orc_hann_sinc_gather(ctypes.byref(sc), _p(self.s), self.s.size, self.L,
                                   int(n0), int(n1), _p(out), nthreads)
        return out


# ---------------------------------------------------------------------------
# static responses and the splice baseline (reference.py:49-187)
def sinc_kernels(frac) -> np.ndarray:
    """(n, 65) Kaiser(7.857)-windowed sinc rows at offsets (i - 32) - frac
    (reference.py:49-64), vectorised over frac (n,)."""
    hw = UPSAMPLE_HALFWIDTH
    arg = np.arange(-hw, hw + 1, dtype=np.float64)[None, :] - np.asarray(frac, np.float64)[:, None]
    z = np.clip(arg / hw, -1.0, 1.0)
    win = np.where(np.abs(arg) <= hw, np.i0(7.857 * np.sqrt(np.maximum(0.0, 1.0 - z * z))), 0.0)
    return np.sinc(arg) * (win / np.i0(7.857))


def static_rir_taps(dims, walls, src, mic, rate: float, max_order: int, c: float = 343.0,
                    d_min: float = 0.05) -> np.ndarray:
    """Tap train of a frozen source (reference.py:67-100): every image's
    windowed sinc scaled by beta/(4 pi max(d, d_min)) and added at
    floor(tau) - 32 in canonical image order, clipped to [0, n_taps)."""
    im = enumerate_images(dims, walls, max_order)
    p = im.offset + im.sign * np.asarray(src, np.float64)[None, :]
    d = np.linalg.norm(p - np.asarray(mic, np.float64)[None, :], axis=1)
    tau = rate * d / c
    n_taps = int(np.ceil(tau.max())) + UPSAMPLE_HALFWIDTH + 2
    base = np.floor(tau)
    rows = (im.beta / (4.0 * np.pi * np.maximum(d, d_min)))[:, None] * sinc_kernels(tau - base)
    idx = base.astype(np.int64)[:, None] - UPSAMPLE_HALFWIDTH + np.arange(rows.shape[1])[None, :]
    keep = (idx >= 0) & (idx < n_taps)
    taps = np.zeros(n_taps)
    np.add.at(taps, idx[keep], rows[keep])  # image-major: canonical order per tap
    return taps


def splice_windows(n: int, hop: int, crossfade: int):
    """(start, stop-of-support, window values) of every block
    (reference.py:145-165)."""
    nb = max(1, -(-n // hop))
    out = []
    for b in range(nb):
        start, stop = b * hop, min(n, (b + 1) * hop)
        end = min(n, stop + crossfade) if (crossfade > 0 and b < nb - 1) else stop
        w = np.ones(end - start)
        if crossfade > 0:
            k = np.arange(start, end)
            fade_in = (k < stop) & (k < start + crossfade) & (b > 0)
            w[fade_in] = (k[fade_in] - start + 0.5) / crossfade
            fade_out = k >= stop
            w[fade_out] = np.maximum(0.0, 1.0 - (k[fade_out] - stop + 0.5) / crossfade)
        out.append((start, end, w))
    return out


def splice_baseline(s, pos, dims, walls, mic, rate: float, max_order: int, hop: int,
                    crossfade: int, c: float = 343.0, d_min: float = 0.05) -> np.ndarray:
    """Block-frozen render (reference.py:133-187): source frozen at each
    block start, windowed blocks convolved (direct) with their responses and
    overlap-added in block order."""
    s = np.asarray(s, np.float64)
    pieces = []
    for start, end, w in splice_windows(s.size, hop, crossfade):
        taps = static_rir_taps(dims, walls, pos[min(start, len(pos) - 1)], mic, rate, max_order,
                               c, d_min)
        pieces.append((start, np.convolve(s[start:end] * w, taps), s.size + taps.size - 1))
    out = np.zeros(max(p[2] for p in pieces))
    for start, y, _ in pieces:
        out[start:start + y.size] += y
    return out
