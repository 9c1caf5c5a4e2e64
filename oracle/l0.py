"""L0 CPU baseline: the reference package's OWN code, timed on the host.

TEST / MEASUREMENT INFRASTRUCTURE (like the rest of oracle/): imported only
by bench.py's cpu_baseline / --impl reference legs and tests, never by the
product package.

The reference (`moverb`, /root/reference/pkg) is installed unmodified into
baseline/_ref (`pip install --no-index --no-deps --target
baseline/_ref`), which travels to the GPU box, so its numba kernels run
there.  Two samples, both the reference's code path (BASELINE.md
"CPU baseline plan", pkg/benchmarks/bench_kernels.py:68-88):

  render   the L0 composition of SURVEY 8c on a whole config (c2 by
           default): per tier low_order_distances / high_order_distances(
           decimate(traj, N)), merge_streams, then synthesize(workers =
           nproc) -- tracks + synthesis, timed separately;
  kernel   the reference's synthesize hot loop on the bench workload (c3):
           32-image blocks of _accumulate_numba in a ThreadPoolExecutor of
           nproc workers plus the pairwise block merge (synth.py:223-258),
           over all S images and a mid-signal window of output samples.  The
           window's tau/amp come from the oracle's tracks (bit-identical to
           the reference's) through the reference's formulas (synth.py:218-
           220); the window trick passes tau - n0 so the kernel's (D, mu, idx)
           are the full render's (D' = D - n0, idx' = idx).  Also with the
           reference's default filter design(3, 8, 0.8).
"""

from __future__ import annotations

import os
import sys
import tempfile
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PATH = os.path.join(ROOT, "baseline", "_ref")

_MV = None


def load():
    """The installed reference package (raises ImportError if absent)."""
    global _MV
    if _MV is not None:
        return _MV
    if not os.path.isdir(os.path.join(REF_PATH, "moverb")):
        raise ImportError(f"reference not installed in {REF_PATH}")
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "mvb_l0_numba"))
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    import moverb
    from moverb import _kernels
    if not moverb.using_numba():
        raise ImportError("reference installed but numba is not in use")
    _MV = moverb
    return moverb


def _ref_filter(branches):
    mv = load()
    br = np.asarray(branches, dtype=np.float64)
    M1, L = br.shape
    return mv.FarrowFilter(poly_order=M1 - 1, branch_len=L, branches=br,
                           nominal_delay=(L - 1) // 2, passband=0.8)


def _tier_streams(images, traj, mic, room, tiers):
    from moverb.synth import high_order_distances, low_order_distances, merge_streams
    from moverb.trajectory import decimate
    streams, prev = None, -1
    for mo, N in tiers:
        sel = [sp for sp in images if prev < sp.order <= mo]
        prev = mo
        if not sel:
            continue
        st = low_order_distances(sel, traj, mic, room) if N == 1 else \
            high_order_distances(sel, decimate(traj, N), mic, room, len(traj), N)
        streams = st if streams is None else merge_streams(streams, st)
    return streams


def render_sample(scene, branches, workers: int) -> dict:
    """The reference's whole render of one (fixed-mic) scene: L0
    composition + synthesize(workers).  Returns times, updates, output."""
    mv = load()
    from moverb.room import MicPosition, Room, enumerate_images
    from moverb.synth import SynthesisConfig, synthesize
    from moverb.trajectory import Trajectory
    f = _ref_filter(branches)
    room = Room(dims=scene.dims, wall_reflection=scene.walls)
    t0 = time.perf_counter()
    images = enumerate_images(room, scene.max_order)
    traj = Trajectory(rate=scene.rate, positions=scene.pos)
    streams = _tier_streams(images, traj, MicPosition(pos=scene.mics[0]), room, scene.tiers)
    t1 = time.perf_counter()
    cfg = SynthesisConfig(audio_rate=scene.rate, max_order=scene.max_order, workers=workers)
    y = synthesize(np.asarray(scene.s, dtype=np.float64), streams, f, cfg)
    t2 = time.perf_counter()
    upd = len(images) * y.size
    return {"tracks_s": t1 - t0, "synthesize_s": t2 - t1, "updates": upd, "out": y,
            "value": upd / (t2 - t0), "synthesize_value": upd / (t2 - t1),
            "numba": bool(mv.using_numba()), "workers": workers}


class KernelSample:
    """The reference's block-parallel accumulate over all images of a scene
    and a window of output samples (see the module docstring)."""

    def __init__(self, oracle_scene, branches, n0: int, width: int, threads: int):
        mv = load()
        from moverb import farrow as rfarrow
        o = oracle_scene
        self.n0, self.width = int(n0), int(width)
        d = o.tracks_window(self.n0, self.n0 + self.width, threads)
        beta = o.images.beta
        self.amp = beta[:, None] / (4.0 * np.pi * np.maximum(d, o.d_min))  # synth.py:219-220
        tau = o.rate * d / o.c  # synth.py:218
        del d
        tau -= float(self.n0)  # (D, mu, idx) of the full render (module docstring)
        self.tau_w = tau
        self.f = _ref_filter(branches)
        self.streams = rfarrow.branch_filter(np.asarray(o.s, dtype=np.float64), self.f)
        self.S = tau.shape[0]
        self._k = mv._kernels
        self.run(1, blocks=1)  # numba compile / cache load outside the timing

    def run(self, workers: int, blocks: int | None = None):
        """(window output, seconds): synth.py:223-258 over the window."""
        from moverb.synth import SUMMATION_BLOCK, _pairwise_merge
        f = self.f
        shift = f.branch_len
        nblk = -(-self.S // SUMMATION_BLOCK) if blocks is None else blocks
        spans = [slice(b * SUMMATION_BLOCK, min((b + 1) * SUMMATION_BLOCK, self.S))
                 for b in range(nblk)]

        def block(sl):
            buf = np.zeros(self.width)
            self._k._accumulate_numba(buf, self.streams, self.tau_w[sl], self.amp[sl], shift,
                                      f.nominal_delay)
            return buf

        t = time.perf_counter()
        if workers > 1 and len(spans) > 1:
            with ThreadPoolExecutor(max_workers=workers) as pool:
                bufs = list(pool.map(block, spans))
        else:
            bufs = [block(sl) for sl in spans]
        y = _pairwise_merge(bufs)
        return y, time.perf_counter() - t
