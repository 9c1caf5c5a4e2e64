"""Fused moving-source render engine: plans a batch of jobs on the device
and drives libmvb (include/mvb.h).

A *job* is one output channel of one scene: dry signal s, source path,
receiver (fixed position or path), room, image order and tier table.  The
engine renders any number of jobs with a fixed number of kernel launches:

  Geometry(jobs)                       synth.py:261-288 (prepare_streams)
    paths buffer   every source path, receiver and decimated path (fp64 rows),
                   staged on a side stream when the caller marks its inputs
                   ready; path boxes and the decimation decision
                   (trajectory.py:279-298) are the only host readbacks
    image table    GPU enumeration (room.py:108-143), tier factor per order
    coarse tracks  mvb_coarse_distances (+ bounds) on pos[::N]
    dmax per job   mvb_track_bounds + mvb_track_max: the exact max of the
                   reference's tracks, kept on the device
  render(geometry, signals, filter)    synth.py:194-258 (synthesize)
    capacities     from Geometry.length_bound (host, no wait); the exact
                   reference out_len is written into the device job table
                   by mvb_finalize_lengths and read lazily (RenderResult)
    fast  (fp32):  branch records, interval polynomials, per-job delay sort,
                   mvb_synthesize_f32 over (job, tile, image chunk) CTAs,
                   fixed-order chunk reduction
    exact (fp64):  reference streams + mvb_synthesize_f64 (reference
                   arithmetic and summation order)

Host<->device transfers live in _staging.py.

Sharding (synth.render_jobs): a rank renders a strided subset of every
job's images (Job.image_index) with the batch-wide track maximum supplied by
Geometry's `dmax_hook` (an all-reduce of the per-rank maxima), so every
rank writes the reference's out_len and the partial outputs sum exactly
(parallel.py: one NCCL reduce).
"""

from __future__ import annotations

import ctypes
import functools
import math
import os
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np
import torch

from . import _lib
from ._dev import h2d, pinned_scratch, ptr, require_cuda, stream_handle
from ._staging import _ARENA, _STAGER, copy_batch, d2h, parallel_copy, side_stream  # noqa: F401
from .farrow import as_filter, centered_branches
from .room import image_table
from .trajectory import (bandwidth_batch_async, device_constants, lowpass_batch, negative_mass,
                         phase_fit)

_TRACE = [] if os.environ.get("MVB_TRACE_HOST") else None


def _mark(name: str) -> None:
    """Host-phase timestamps for profiling the planner (env MVB_TRACE_HOST)."""
    if _TRACE is not None:
        import time
        _TRACE.append((name, time.perf_counter()))


SYNTH_U = 16  # steps per lane (mvb_synthesize_f32 u_steps)
TILE = 32 * SYNTH_U  # output samples per CTA
SEG_LEN = int(os.environ.get("MVB_SEG_TILES", "32")) * TILE  # samples per delay-sort segment
SORT_RUN = 2048  # images per independent sort run of time-shard jobs
IMG_COLS, JOB_COLS, WORK_COLS = 12, 19, 4
BOX_WORDS = 16  # mvb_path_bbox record: boxes (12), max steps (2), pad (2)
# fp32 fast-path accuracy envelope: the largest delay excursion (samples) of
# one coarse interval that the fp32 residual of the interval records may
# carry; beyond it the render routes to the exact fp64 engine
# (Geometry.fast_path_ok)
FP32_ENVELOPE = float(os.environ.get("MVB_FP32_ENVELOPE", "48"))
PAD_MARGIN = 64
FOUR_PI = 4.0 * np.pi


@dataclass
class Job:
    s: object  # (Ts,) dry signal (numpy / torch); fp32 selects the fast path
    pos: object  # (T, 3) source path at the audio rate
    mic: object  # (3,) fixed receiver or (T, 3) receiver path
    dims: object
    walls: object
    max_order: int
    tiers: tuple  # ((max_order, N), ...) ascending in max_order
    rate: float
    c: float = 343.0
    d_min: float = 0.05
    image_index: object = None  # optional subset of the canonical image order
    signal_key: object = None  # jobs with equal keys share one dry signal
    path_key: object = None  # jobs with equal keys share one source path
    # time shard (parallel.time_window): render output samples [w0, w1) only
    # (w1 = 0: to the end), zeros elsewhere; the track maximum is then the
    # window's -- a dmax hook must all-reduce it (MAX) for the reference's
    # out_len
    window: tuple = None


def window_fields(T: int, window) -> dict:
    """mvb_job w0, w1, e0, e1 of a job with path length T and output window
    `window` (None: the whole job, all zero).  [e0, e1): path samples whose
    coarse tracks the window needs -- its path range (win_p0 / win_p1 of
    mvb_common.cuh) and the centres of the sort segments its tiles read."""
    if window is None:
        return dict(w0=0, w1=0, e0=0, e1=0)
    w0, w1 = int(window[0]), int(window[1])
    if w0 < 0 or w0 % TILE or (w1 > 0 and (w1 <= w0 or w1 % TILE)):
        raise ValueError(f"window {window}: need 0 <= w0 < w1 (w1 = 0: open), multiples of {TILE}")
    T = int(T)
    p0 = min(w0, T - 1)
    p1 = min(w1, T) if w1 > 0 else T
    last = -(-T // SEG_LEN) - 1
    sa = min(w0 // SEG_LEN, last)
    sb = min((w1 - 1) // SEG_LEN, last) if w1 > 0 else last
    ca = min(sa * SEG_LEN + SEG_LEN // 2, T - 1)
    cb = min(sb * SEG_LEN + SEG_LEN // 2, T - 1)
    return dict(w0=w0, w1=w1, e0=min(p0, ca), e1=max(p1, cb + 1))


def coarse_span(rows: list, N: int) -> int:
    """Largest coarse-sample range [k0, k1) (win_coarse) a factor-N image of
    these job rows computes, + one 64-sample segment of alignment."""
    out = 1
    for r in rows:
        K = -(-int(r["T"]) // N)
        if r.get("e1", 0) <= 0:
            out = max(out, K)
            continue
        k0 = max(int(r["e0"]) // N - 34, 0)
        k1 = min((int(r["e1"]) - 1) // N + 1 + 34, K)
        out = max(out, k1 - k0 + 64)
    return out



def _key(explicit, obj):
    return ("k", explicit) if explicit is not None else ("id", id(obj))


def _as_f64_rows(a) -> object:
    if isinstance(a, torch.Tensor):
        return a.to(torch.float64).reshape(-1, 3)
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64)).reshape(-1, 3)


def _validate_tiers(tiers, max_order):
    if not tiers:
        raise ValueError("tier table is empty")
    prev = -1
    for mo, N in tiers:
        if int(N) != N or N < 1:
            raise ValueError("tier decimation must be a positive integer")
        if mo <= prev:
            raise ValueError("tier max_order must increase")
        prev = mo
    if tiers[-1][0] < max_order:
        raise ValueError("tiers do not cover max_order")


def pack_jobs(rows: list) -> np.ndarray:
    """list of dicts -> (n, 16) int64 array with the mvb_job layout."""
    a = np.zeros((len(rows), JOB_COLS), dtype=np.int64)
    i32 = a[:, 9:12].view(np.int32)
    f64 = a[:, 12:16].view(np.float64)
    for j, r in enumerate(rows):
        a[j, 0:9] = [r["out_off"], r["out_len"], r["part_off"], r["rec_base"], r["ls"],
                     r["img_off"], r["n_img"], r["pos_off"], r["mic_off"]]
        i32[j] = [r["T"], r["mic_moving"], r["L"], r["d0"], r["n_chunks"], r["nb"]]
        f64[j] = [r["rate"], r["c"], r["d_min"], r["kappa"]]
        a[j, 16:19].view(np.int32)[:] = [r.get("img_stride", 0), r.get("rec_rows", 0),
                                          r.get("w0", 0), r.get("w1", 0),
                                          r.get("e0", 0), r.get("e1", 0)]
    return a


@lru_cache(maxsize=64)
def _group_plan(max_order: int, tiers: tuple, sub: tuple | None):
    """Host plan of one enumeration group (pure function of its key):
    canonical source index, factor class and per-class prefix counts of
    every image (the (S, 2+nC) int32 table mvb_build_images reads), the
    classes and their image counts."""
    order_np = np.repeat(np.arange(max_order + 1),
                         [1] + [4 * o * o + 2 for o in range(1, max_order + 1)])
    src = np.arange(order_np.size, dtype=np.int64)
    if sub is not None:
        src = np.asarray(sub, np.int64)
        order_np = order_np[src]
    fac_np = np.ones(order_np.size, np.int64)
    prev = -1
    for mo, N in tiers:
        fac_np[(order_np > prev) & (order_np <= mo)] = N
        prev = mo
    classes = tuple(sorted(set(fac_np.tolist())))
    if len(classes) > _lib.MAX_CLASSES:
        raise ValueError(f"at most {_lib.MAX_CLASSES} distinct decimation factors")
    cidx = np.searchsorted(np.asarray(classes), fac_np)
    onehot = (cidx[:, None] == np.arange(len(classes))[None, :]).astype(np.int32)
    pref = np.cumsum(onehot, axis=0) - onehot  # earlier images per class
    img_tab = np.concatenate([src[:, None], cidx[:, None], pref], axis=1).astype(np.int32)
    img_tab.flags.writeable = False
    return classes, onehot.sum(axis=0), img_tab


@lru_cache(maxsize=16)
def _sm_count(index: int) -> int:
    return torch.cuda.get_device_properties(index).multi_processor_count


_DEV_CACHE: dict = {}


def _cached_dev(key, make):
    """Small read-only device tables reused across renders (bounded).  Not
    filled during a graph capture: a captured upload only runs at replay.
    Users that a graph captures keep their own reference (Geometry._keep)."""
    t = _DEV_CACHE.get(key)
    if t is None:
        from ._dev import StaticUploads
        if StaticUploads._active is not None:
            return make()
        if len(_DEV_CACHE) > 64:
            _DEV_CACHE.clear()
        t = _DEV_CACHE[key] = make()
    return t


class Geometry:
    """Device-side hierarchical tracks of a batch of jobs (prepare stage)."""

    def __init__(self, jobs: list, device=None, inputs_ready=None, dmax_hook=None,
                 paths=None, defer=False, wait=True, bbox=None, on_paths=None,
                 readback_tag: str = ""):
        """`inputs_ready`: optional CUDA event after which every device
        tensor of `jobs` is final.  With it, the paths are staged and their
        bandwidths measured on a side stream that waits only for that event,
        so planning this batch does not queue behind earlier work on the
        current stream (e.g. the previous batch's synthesis).  `dmax_hook`:
        optional callable applied in place to the device tensor of per-job
        track maxima before it is read (image shards: all-reduce MAX).
        `paths`: a caller-owned fp64 (rows, 3) buffer to stage the paths
        into (render plans), `bbox` likewise for the path bounding boxes
        (a plan's graphs read both at every replay); `defer`: stop after the
        staging (bounding boxes,
        decimation decision) -- finish() does the device work.  `wait=False`
        (with defer): enqueue the staging and its two readbacks but do not
        wait for them -- `paths_ready` (an event after the path upload) lets
        device work that needs only the paths start at once, collect() waits
        for the boxes and the decision (render plans replay speculatively).
        `on_paths(event)`: called as soon as that event is recorded, before
        the bandwidth kernels are enqueued (a plan launches its replay
        there, ahead of the host-side issue of the decision pipeline).
        `readback_tag`: suffix of the pinned readback buffers' names -- a
        caller that leaves several stagings pending at once (render plans,
        one per slot) gives each its own buffers."""
        if not jobs:
            raise ValueError("no jobs")
        self.dev = require_cuda(device)
        self.jobs = jobs
        for jb in jobs:
            _validate_tiers(jb.tiers, jb.max_order)
        self.length_slack = 0.0
        self._tag = readback_tag
        host_parts, dev_parts, rows = self._layout_paths()
        self.rows = rows
        _mark("geom.setup")
        self._pending = self._stage_paths(host_parts, dev_parts, rows, inputs_ready, paths, bbox,
                                          on_paths)
        if wait or not defer:
            self.collect()
        _mark("geom.bandwidth")
        if not defer:
            self.finish(dmax_hook)

    def collect(self):
        """Wait for the staging readbacks (path boxes, bandwidth indices)."""
        if self._pending is not None:
            box_ready, box_host, path_groups, finishers = self._pending
            self.bws = [fin() for fin in finishers]
            box_ready.synchronize()
            self.bbox_host = box_host.numpy().copy()
            self.path_groups = path_groups
            self._pending = None
        return self

    def recollect(self, pending) -> "Geometry":
        """Re-read the readbacks of a captured staging (`pending`: the
        `_pending` of the Geometry built during the capture), refilled by a
        replay the caller has waited for (render plans)."""
        _, box_host, path_groups, finishers = pending
        self.bws = [fin(False) for fin in finishers]
        self.bbox_host = box_host.numpy().copy()
        self.path_groups = path_groups
        return self

    def finish(self, dmax_hook=None, fork=None):
        """Device work after the staging: coarse paths, image records, coarse
        tracks, bounds and the exact track maxima (no host waits).  `fork`
        (a stream, render-plan capture only): the exact-maximum chain runs
        there, parallel to what the caller enqueues next (only the exact
        output lengths need it); `join()` merges it back."""
        self._decimate_paths(self.path_groups, self.bws)
        _mark("geom.decimate")
        self._build_images()
        _mark("geom.images")
        self._tracks(dmax_hook, fork)
        _mark("geom.tracks")
        self.eval_count = [int(self.evals[j]) for j in range(len(self.jobs))]

    def lowpass_decision(self) -> tuple:
        """Which (path group, factor) pairs need the anti-alias low-pass
        (trajectory.py:279-298) -- part of a render plan's identity."""
        out = []
        for (T, rate, x, uses), bw in zip(self.path_groups, self.bws):
            for (T2, rate2, N) in sorted(uses):
                if (T2, rate2) == (T, rate) and N > 1:
                    nyq = 0.5 * rate / N
                    out.append(tuple(np.nonzero((bw > nyq) & (bw < 2.0 * nyq))[0].tolist()))
        return tuple(out)

    def _layout_paths(self):
        """Rows of the fp64 paths buffer: every distinct source path first
        (equal-length paths of a batch then form one strided view for the
        decimation decision), the receivers after them, then a slot per
        (job, decimated factor) for the coarse source (and receiver) path."""
        jobs, nJ = self.jobs, len(self.jobs)
        host_parts, dev_parts = [], []
        row = 0
        path_row = {}
        self.T = np.zeros(nJ, np.int64)
        self.pos_off = np.zeros(nJ, np.int64)
        self.mic_off = np.zeros(nJ, np.int64)
        self.moving = np.zeros(nJ, np.int64)
        for j, jb in enumerate(jobs):
            k = _key(jb.path_key, jb.pos)
            if k not in path_row:
                p = _as_f64_rows(jb.pos)
                path_row[k] = (row, p.shape[0])
                (dev_parts if isinstance(p, torch.Tensor) else host_parts).append((row, p))
                row += p.shape[0]
            self.pos_off[j], self.T[j] = path_row[k]
        for j, jb in enumerate(jobs):
            m = _as_f64_rows(jb.mic)
            if m.shape[0] == 1:
                self.moving[j] = 0
            elif m.shape[0] == self.T[j]:
                self.moving[j] = 1
            else:
                raise ValueError("receiver must be a 3-vector or a (T,3) path")
            self.mic_off[j] = row
            (dev_parts if isinstance(m, torch.Tensor) else host_parts).append((row, m))
            row += m.shape[0]
        self.cpath = {}  # (j, N) -> row
        for j, jb in enumerate(jobs):
            for _, N in jb.tiers:
                N = int(N)
                if N > 1 and (j, N) not in self.cpath:
                    self.cpath[(j, N)] = row
                    row += -(-int(self.T[j]) // N) * (1 + int(self.moving[j]))
        return host_parts, dev_parts, max(row, 1)

    def _stage_paths(self, host_parts, dev_parts, rows, inputs_ready, paths=None, bbox=None,
                     on_paths=None):
        """Fill the full-rate rows of the paths buffer, compute every job's
        path bounding boxes and the paths' bandwidths; the two small
        readbacks (boxes, bandwidth indices) are the host's only waits.
        With `inputs_ready` this runs on the high-priority side stream into a
        persistent arena buffer (released by render_jobs), so it does not
        queue behind earlier work on the current stream."""
        dev, nJ = self.dev, len(self.jobs)
        main = torch.cuda.current_stream(dev)
        side = side_stream(dev) if inputs_ready is not None else main
        if side is not main:
            side.wait_event(inputs_ready)
        with torch.cuda.stream(side):
            self._arena = None
            if paths is not None:
                if paths.shape[0] < rows:
                    raise ValueError("paths buffer too small")
                self.paths = paths[:rows]
            elif side is not main:
                self._arena = _ARENA.acquire(dev, rows)
                self.paths = self._arena[:rows]
            else:
                self.paths = torch.empty(rows, 3, dtype=torch.float64, device=dev)
            if host_parts:
                _STAGER.upload(host_parts, self.paths)
            # device-resident paths (render plans' static inputs): one batched
            # call for the contiguous fp64 ones
            batch = []
            for r0, p in dev_parts:
                if p.dtype == torch.float64 and p.is_contiguous() and p.device == dev \
                        and tuple(p.shape[1:]) == (3,):
                    batch.append((self.paths.data_ptr() + 24 * r0, p.data_ptr(), 24 * p.shape[0]))
                else:
                    self.paths[r0:r0 + p.shape[0]].copy_(p)
            if batch:
                copy_batch(batch, side.cuda_stream, require_pinned=False)
            box_rows = h2d(np.stack([self.pos_off, self.T, self.mic_off, self.moving], axis=1), dev)
            # flat: the nJ x BOX_WORDS boxes first, then the 64 partial boxes per job
            if bbox is not None and bbox.numel() >= nJ * 65 * BOX_WORDS:
                self.bbox = bbox
            else:
                self.bbox = torch.empty(nJ * 65 * BOX_WORDS, dtype=torch.float64, device=dev)
            _lib.call("mvb_path_bbox", ptr(box_rows), nJ, ptr(self.paths), ptr(self.bbox),
                      stream_handle(dev))
            box_host = pinned_scratch("bbox" + self._tag, nJ * BOX_WORDS,
                                      torch.float64).view(nJ, BOX_WORDS)
            box_host.copy_(self.bbox[:nJ * BOX_WORDS].view(nJ, BOX_WORDS), non_blocking=True)
            box_ready = torch.cuda.Event()
            box_ready.record()
            self.paths_ready = box_ready  # the paths' full-rate rows are on the device
            if on_paths is not None:
                on_paths(box_ready)
            path_groups, finishers = self._path_bandwidths(main)
        if side is not main:
            main.wait_stream(side)
            self.bbox.record_stream(main)
        return box_ready, box_host, path_groups, finishers

    def join(self) -> None:
        """Order the current stream after the forked exact-maximum chain."""
        if getattr(self, "_fork", None) is not None:
            torch.cuda.current_stream(self.dev).wait_stream(self._fork)
            self._fork = None

    def _tracks(self, dmax_hook, fork=None):
        """Job table, coarse tracks and their bounds, the exact track maximum
        of every job (kept on the device; `dmax_hook` may reduce it across
        ranks in place)."""
        dev, nJ, st = self.dev, len(self.jobs), stream_handle(self.dev)
        self.job_rows = []
        for j, jb in enumerate(self.jobs):
            self.job_rows.append(dict(
                out_off=0, out_len=0, part_off=0, rec_base=0, ls=0,
                img_off=int(self.img_off[j]), n_img=int(self.n_img[j]),
                pos_off=int(self.pos_off[j]), mic_off=int(self.mic_off[j]),
                T=int(self.T[j]), mic_moving=int(self.moving[j]), L=0, d0=0, n_chunks=1, nb=0,
                rate=float(jb.rate), c=float(jb.c), d_min=float(jb.d_min),
                kappa=float(jb.rate) / float(jb.c), **window_fields(self.T[j], jb.window)))
        # kept: the exact-maximum branch (a parallel graph branch in plan
        # captures) still reads it after this function returns
        jobs_dev = self._jobs_dev = h2d(pack_jobs(self.job_rows), dev)
        n_img = self.n_images
        self.coarse = torch.empty(max(self.n_coarse_total, 1), dtype=torch.float64, device=dev)
        lb = torch.zeros(n_img, dtype=torch.float64, device=dev)
        ub = torch.zeros(n_img, dtype=torch.float64, device=dev)
        negsum = max([negative_mass(N) for N in self.factors if N > 1], default=0.0)
        # coarse distances + bounds of the decimated images, one launch per
        # factor (its grid spans that factor's coarse length, no idle chunks)
        for N, sel in self.sel_by_factor.items():
            max_K = coarse_span([self.job_rows[j] for (j, N2) in self.cpath if N2 == N], N)
            _lib.call("mvb_coarse_distances", ptr(self.images), ptr(sel), sel.numel(), max_K,
                      ptr(jobs_dev), ptr(self.paths), negsum, ptr(self.coarse), ptr(lb), ptr(ub),
                      st)
        self._fork = None
        if fork is not None:  # exact-maximum chain as a parallel branch
            fork.wait_stream(torch.cuda.current_stream(dev))
            self._fork = fork
        with torch.cuda.stream(fork if fork is not None else torch.cuda.current_stream(dev)):
            st = stream_handle(dev)
            if self.full_sel.numel():  # bounding-box bounds of the full-rate images
                _lib.call("mvb_track_bounds", ptr(self.images), ptr(self.full_sel),
                          self.full_sel.numel(), ptr(jobs_dev), ptr(self.paths), ptr(self.bbox),
                          ptr(lb), ptr(ub), st)
            scratch = torch.empty(_lib.EXACT_LIST_WORDS + n_img + nJ, dtype=torch.int32,
                                  device=dev)
            dmax = torch.empty(nJ, dtype=torch.float64, device=dev)
            _lib.call("mvb_track_max", ptr(self.images), ptr(jobs_dev), nJ,
                      ptr(self.coarse) if self.dec_sel.numel() else ptr(None), ptr(self.tables),
                      ptr(self.paths), negsum, ptr(lb), ptr(ub), ptr(scratch), ptr(dmax), st)
        if dmax_hook is not None:
            dmax_hook(dmax)
        self.dmax_dev = dmax
        self._bounds = (lb, ub, scratch)  # per-image track bounds, exact-max candidates
        self._dmax = None  # host copy on demand (the render itself never waits for it)

    def release(self) -> None:
        """Hand the staging buffer back (after every kernel reading the paths
        has been enqueued on the current stream); the geometry's tracks may
        not be used afterwards."""
        if getattr(self, "_arena", None) is not None:
            ev = torch.cuda.Event()
            ev.record()
            _ARENA.release(self.dev, self._arena, ev)
            self._arena = None

    @property
    def dmax(self) -> np.ndarray:
        """Per-job exact track maximum (waits for the geometry kernels)."""
        if self._dmax is None:
            self._dmax = self.dmax_dev.cpu().numpy()
        return self._dmax

    # ------------------------------------------------------------------------
    def _path_bandwidths(self, consumer):
        """Paths that need decimation, grouped by (length, rate), and their
        measured bandwidths (trajectory.py:316-339): one batched FFT per
        group and one small device->host copy per group, returned as
        functions that wait for them (collect())."""
        jobs = self.jobs
        groups = {}  # (T, rate) -> {row0: position}
        uses = {}  # (T, rate, N) -> list of (position, destination row)
        for (j, N), dst in self.cpath.items():
            T, rate = int(self.T[j]), float(jobs[j].rate)
            g = groups.setdefault((T, rate), {})
            K = -(-T // N)
            srcs = [(int(self.pos_off[j]), dst)]
            if self.moving[j]:
                srcs.append((int(self.mic_off[j]), dst + K))
            for r0, d in srcs:
                pos = g.setdefault(r0, len(g))
                uses.setdefault((T, rate, N), []).append((pos, d))
        out, bws = [], []
        for (T, rate), rows in groups.items():
            starts = sorted(rows, key=rows.get)
            G = len(starts)
            if all(starts[q] == starts[0] + q * T for q in range(G)):
                x = self.paths[starts[0]:starts[0] + G * T].view(G, T, 3)  # contiguous run
            else:
                x = torch.stack([self.paths[r0:r0 + T] for r0 in starts])  # (G, T, 3)
                x.record_stream(consumer)  # read again by the decimation
            out.append((T, rate, x, uses))
            bws.append(bandwidth_batch_async(x, rate, slot=f"bandwidth_index{len(bws)}{self._tag}"))
        return out, bws

    def _decimate_paths(self, path_groups, bws):
        """Fill the coarse path slots with pos[::N] (and receiver[::N]).  The
        reference's anti-alias decision (low-pass only when Nyquist_out <
        bandwidth < 2 Nyquist_out, trajectory.py:279-298) uses the measured
        bandwidths; the low-pass runs only for the paths it selects; one
        index_copy per (length, factor)."""
        dev = self.dev
        st = stream_handle(dev)
        for (T, rate, x, uses), bw in zip(path_groups, bws):
            for (T2, rate2, N), lst in uses.items():
                if (T2, rate2) != (T, rate):
                    continue
                K = -(-T // N)
                nyq = 0.5 * rate / N
                lp_rows = np.nonzero((bw > nyq) & (bw < 2.0 * nyq))[0] if N > 1 else np.zeros(0)
                pos = np.asarray([p for p, _ in lst], np.int64)
                dst = np.asarray([d for _, d in lst], np.int64)
                raw = ~np.isin(pos, lp_rows)
                if raw.any():  # straight pos[::N] from the full-rate rows (x is (G, T, 3) contiguous)
                    rows = h2d(np.stack([pos[raw] * T, dst[raw]], axis=1), dev)
                    _lib.call("mvb_decimate_rows", ptr(x), ptr(rows), int(raw.sum()), K, N,
                              ptr(self.paths), st)
                if (~raw).any():  # anti-alias low-pass first (trajectory.py:279-298)
                    sel = np.unique(pos[~raw])
                    lp = lowpass_batch(x[h2d(sel.astype(np.int64), dev)], rate, 0.9 * nyq)
                    lp = lp.contiguous()
                    where = np.searchsorted(sel, pos[~raw])
                    rows = h2d(np.stack([where * T, dst[~raw]], axis=1), dev)
                    _lib.call("mvb_decimate_rows", ptr(lp), ptr(rows), int((~raw).sum()), K, N,
                              ptr(self.paths), st)

    def _build_images(self):
        """Image records of every job: rooms enumerated on the device (one
        launch per group of jobs sharing max_order / tiers / subset), then
        one mvb_build_images launch per group writes the records and the
        factor selections straight into their final buffers."""
        jobs, dev = self.jobs, self.dev
        nJ = len(jobs)
        st = stream_handle(dev)
        # factor constants (transposed tables) shared by the batch
        factors = sorted({int(N) for jb in jobs for _, N in jb.tiers if int(N) > 1})
        self.factors = factors
        self.table_off, self.fit_idx = {}, {}
        off = 0
        for q, N in enumerate(factors):
            self.table_off[N] = off
            off += 65 * N
            self.fit_idx[N] = q
        self.tables = _cached_dev(
            ("tables", tuple(factors), str(dev)),
            lambda: torch.cat([device_constants(N, dev)["tableT"].reshape(-1) for N in factors])
            if factors else torch.zeros(1, dtype=torch.float64, device=dev))
        # cached tables this geometry's kernels read: owned here too, so a
        # captured graph's pointers stay valid if the bounded cache drops them
        self._keep = [self.tables]
        groups = {}
        for j, jb in enumerate(jobs):
            sub = None if jb.image_index is None else tuple(np.asarray(jb.image_index).tolist())
            key = (int(jb.max_order), tuple((int(a), int(b)) for a, b in jb.tiers), sub)
            groups.setdefault(key, []).append(j)
        self.img_off = np.zeros(nJ, np.int64)
        self.n_img = np.zeros(nJ, np.int64)
        self.evals = np.zeros(nJ, np.int64)
        # pass 1 (host): classes, per-image prefix counts, sizes
        plans = []
        img_base = coarse_base = n_full = n_dec = 0
        n_cls = {N: 0 for N in factors}
        for (max_order, tiers, sub), members in groups.items():
            classes, counts, img_tab = _group_plan(max_order, tiers, sub)
            S = img_tab.shape[0]
            G = len(members)
            Tj = self.T[members].astype(np.int64)
            Kc = np.array([[-(-int(T) // N) if N > 1 else 0 for N in classes] for T in Tj],
                          np.int64).reshape(G, len(classes))
            per_job = (Kc * counts[None, :]).sum(axis=1)
            kbase = coarse_base + np.concatenate([[0], np.cumsum(per_job)[:-1]]).astype(np.int64)
            ct = _lib.ClassTable()
            ct.n = len(classes)
            for q, N in enumerate(classes):
                ct.factor[q] = int(N)
                ct.fit[q] = self.fit_idx.get(int(N), 0)
                ct.count[q] = int(counts[q])
                ct.table[q] = self.table_off.get(int(N), 0)
                if N > 1:
                    ct.sel_off[q] = n_cls[int(N)]
                    n_cls[int(N)] += G * int(counts[q])
            full_cnt = sum(int(counts[q]) for q, N in enumerate(classes) if N == 1)
            plans.append(dict(key=(max_order, tiers, sub), max_order=max_order, members=members,
                              S=S, img_tab=img_tab, classes=classes, kbase=kbase, ct=ct,
                              img_base=img_base, full_off=n_full, dec_off=n_dec,
                              per_job=per_job, counts=counts))
            for g, j in enumerate(members):
                self.img_off[j] = img_base + g * S
                self.n_img[j] = S
                T = int(self.T[j])
                self.evals[j] = int(sum(int(counts[q]) * (T if N == 1 else -(-T // int(N)))
                                        for q, N in enumerate(classes)))
            img_base += G * S
            coarse_base += int(per_job.sum())
            n_full += G * full_cnt
            n_dec += G * (S - full_cnt)
        # class selections: one region per factor, groups in order inside it
        cls_base, acc = {}, 0
        for N in factors:
            cls_base[N] = acc
            acc += n_cls[N]
        i32 = dict(dtype=torch.int32, device=dev)
        self.images = torch.empty(max(img_base, 1), IMG_COLS, dtype=torch.int64, device=dev)
        self.full_sel = torch.empty(n_full, **i32)
        self.dec_sel = torch.empty(n_dec, **i32)
        class_sel = torch.empty(max(acc, 1), **i32)
        # pass 2 (device): enumerate each group's rooms, build its records
        for pl in plans:
            members = pl["members"]
            room_key, rooms, member_room = {}, [], []
            for j in members:
                d = np.asarray(jobs[j].dims, dtype=np.float64).reshape(3)
                w = np.asarray(jobs[j].walls, dtype=np.float64)
                w = np.full(6, float(w)) if w.ndim == 0 else w.reshape(6)
                k = (d.tobytes(), w.tobytes())
                if k not in room_key:
                    room_key[k] = len(rooms)
                    rooms.append((d, w))
                member_room.append(room_key[k])
            # the lattice depends on the rooms and the order only: cached across
            # renders (a render plan's graphs then skip the enumeration)
            tab = _cached_dev(("image_table", tuple(room_key), pl["max_order"], str(dev)),
                              lambda: image_table(np.stack([r[0] for r in rooms]),
                                                  np.stack([r[1] for r in rooms]),
                                                  pl["max_order"], dev))
            self._keep.append(tab)
            ct, classes, S = pl["ct"], pl["classes"], pl["S"]
            for q, N in enumerate(classes):
                if N > 1:
                    ct.sel_off[q] += cls_base[int(N)]

            cp = np.asarray([[self.cpath.get((j, int(N)), 0) for N in classes] for j in members],
                            np.int64).reshape(len(members), len(classes))
            job_tab = np.concatenate([np.asarray(member_room, np.int64)[:, None],
                                      self.T[members].astype(np.int64)[:, None],
                                      np.asarray(members, np.int64)[:, None], pl["kbase"][:, None], cp],
                                     axis=1)
            img_dev = _cached_dev(("img_tab", pl["key"], str(dev)),
                                  lambda: h2d(pl["img_tab"], dev))  # (S, 2 + nC) int32 (mvb.h)
            self._keep.append(img_dev)
            job_dev = h2d(np.ascontiguousarray(job_tab), dev)
            _lib.call("mvb_build_images", ptr(tab.offset), ptr(tab.sign), ptr(tab.beta), tab.count,
                      ptr(img_dev), S, ptr(job_dev), len(members), ctypes.byref(ct), pl["img_base"],
                      ptr(self.images), ptr(self.full_sel), pl["full_off"], ptr(self.dec_sel),
                      pl["dec_off"], ptr(class_sel), st)
        self.n_images = img_base
        self.n_coarse_total = coarse_base
        # record groups (prepare_render, RECORD_BUDGET): a uniform batch --
        # one structure group, jobs in order -- lays each job's coarse
        # samples / interval records and its slice of every factor's
        # selection out contiguously, so consecutive jobs can have their
        # records computed into a shared buffer group by group
        self.rec_layout = None
        if len(plans) == 1 and plans[0]["members"] == list(range(nJ)):
            pl = plans[0]
            sel = {}  # factor N: (offset of job 0's slice in sel_by_factor[N], images per job)
            dec = [int(N) for N in pl["classes"] if N > 1]
            if len(dec) == len(set(dec)):  # one class per factor: one slice per job
                for q, N in enumerate(pl["classes"]):
                    if N > 1:
                        sel[int(N)] = (int(pl["ct"].sel_off[q]) - cls_base[int(N)],
                                       int(pl["counts"][q]))
                self.rec_layout = dict(kbase=np.asarray(pl["kbase"], np.int64),
                                       per_job=np.asarray(pl["per_job"], np.int64), sel=sel)
        self.sel_by_factor = {N: class_sel[cls_base[N]:cls_base[N] + n_cls[N]] for N in factors
                              if n_cls[N]}
        if self.full_sel.numel() > 65535:
            raise ValueError("more than 65535 full-rate images in one batch")

    # ------------------------------------------------------------------------
    def length_bound(self, j: int) -> int:
        """Upper bound of ceil(rate * dmax_j / c) from the image lattice extent
        and the path / receiver bounding boxes, known on the host without
        waiting for the tracks.  Image coordinate along axis a:
        2 l_a L_a + s_a p_a with |2 l_a L_a| <= (|j_a| + 1) L_a and
        sum |j_a| <= max_order, so the distance is at most
        max_a sqrt(((K+1) L_a + P_a + M_a)^2 + sum_{b != a} (L_b + P_b + M_b)^2)
        (P, M: largest source / receiver coordinate magnitudes); widened by
        the upsampler's overshoot (negative tap mass) and a 2% + 1 cm margin
        for the anti-alias low-pass, times (1 + length_slack) (render plans
        reserve headroom so nearby data reuse a capture).
        mvb_finalize_lengths checks it."""
        jb = self.jobs[j]
        box = self.bbox_host[j]
        P = np.maximum(np.abs(box[0:3]), np.abs(box[3:6]))
        M = np.maximum(np.abs(box[6:9]), np.abs(box[9:12]))
        dims = np.asarray(jb.dims, dtype=np.float64).reshape(3)
        K = int(jb.max_order)
        base = dims + P + M
        ext = (K + 1) * dims + P + M
        d2 = max(ext[a] ** 2 + sum(base[b] ** 2 for b in range(3) if b != a) for a in range(3))
        neg = max([negative_mass(int(N)) for _, N in jb.tiers if int(N) > 1], default=0.0)
        d_ub = (1.02 * math.sqrt(d2) * (1.0 + neg) + 0.01) * (1.0 + self.length_slack)
        return int(math.ceil(float(jb.rate) * d_ub / float(jb.c)))

    def interval_excursion(self) -> np.ndarray:
        """Per job: an upper bound (samples) of the delay excursion over one
        coarse interval of its largest decimation factor N, kappa * (largest
        source step + largest receiver step) * N (triangle inequality: an
        image path moves like the source).  The fast path carries the delay
        inside an interval as an fp32 residual around the fp64 anchor, so
        its rounding grows with this span."""
        out = np.zeros(len(self.jobs))
        for j, jb in enumerate(self.jobs):
            n_max = max((int(N) for _, N in jb.tiers if int(N) > 1), default=0)
            if n_max:
                step = float(self.bbox_host[j, 12])
                if self.moving[j]:
                    step += float(self.bbox_host[j, 13])
                out[j] = float(jb.rate) / float(jb.c) * step * n_max
        return out

    @property
    def fast_path_ok(self) -> bool:
        """Every job inside the fp32 fast path's envelope (FP32_ENVELOPE)."""
        return bool(np.all(self.interval_excursion() <= FP32_ENVELOPE))

    def tau_max(self, j: int) -> float:
        jb = self.jobs[j]
        return float(jb.rate) * float(self.dmax[j]) / float(jb.c)


# ----------------------------------------------------------------------------
# filter banks


_BANKS: dict = {}


def fast_bank(filt) -> tuple:
    f = as_filter(filt)
    key = (f.branches.shape, f.branches.tobytes())
    if key not in _BANKS:
        _BANKS[key] = _fast_bank(f)
    return _BANKS[key]


def _fast_bank(filt) -> tuple:
    """Centred fp32-path Farrow bank: (coeffs (M1, L) fp64, M1, nb).  Banks
    above degree 7 are reduced to degree 7 when that changes no tap by more
    than 5e-7 of the largest tap (below fp32 resolution of the path)."""
    f = as_filter(filt)
    cb = centered_branches(f.branches)
    M1 = cb.shape[0]
    if M1 > 8:
        mu = 0.5 - 0.5 * np.cos(np.pi * (np.arange(256) + 0.5) / 256)
        u = mu - 0.5
        h = (u[:, None] ** np.arange(M1)[None, :]) @ cb
        V = np.polynomial.chebyshev.chebvander(2 * u, 7)
        ch, *_ = np.linalg.lstsq(V, h, rcond=None)
        red = np.zeros((8, cb.shape[1]))
        for j in range(cb.shape[1]):
            p = np.polynomial.chebyshev.cheb2poly(ch[:, j])
            red[:p.size, j] = p * (2.0 ** np.arange(p.size))
        uu = np.linspace(-0.5, 0.5, 2001)
        ex = (uu[:, None] ** np.arange(M1)[None, :]) @ cb
        ap = (uu[:, None] ** np.arange(8)[None, :]) @ red
        if np.max(np.abs(ex - ap)) <= 5e-7 * np.max(np.abs(ex)):
            cb, M1 = red, 8
    nb = 4 if M1 <= 4 else 8 if M1 <= 8 else 12 if M1 <= 12 else 16
    if M1 > 16:
        raise ValueError("fast path supports Farrow degree <= 15")
    return cb, M1, nb


# ----------------------------------------------------------------------------
# render stage


def _events(timing):
    """Timing event before the synthesis launch.  `external` events keep
    their timestamps when recorded inside a CUDA-graph capture (render
    plans), so every replay re-times the kernel."""
    if timing is None:
        return None
    e = torch.cuda.Event(enable_timing=True, external=True)
    e.record()
    return e


def _events_end(timing, e0):
    if timing is not None:
        e1 = torch.cuda.Event(enable_timing=True, external=True)
        e1.record()
        timing.append((e0, e1))


class RenderResult:
    """Output of a batch render.  `out` is the flat output (fp32 fast / fp64
    exact) with job j at offsets[j], capacity[j] samples reserved (zeros
    past its length).  The exact lengths are computed on the device
    (mvb_finalize_lengths); `lengths`, `updates` and `job()` wait for them
    on first use, so a render can be queued without a host round trip.
    A render plan's result is produced on the plan's own streams: `done` is
    its completion event and `stream` the stream that produced it; `job()`,
    `host()` and `lengths` order the current stream after it (wait()), code
    that reads `out` directly calls wait() first.  A plan's speculative
    replay is validated on first use of the result (`_validate`, see
    plan.RenderPlan.run): reading any field settles it, and a replay the
    staging readbacks invalidate is redone before the field is returned."""

    def __init__(self, out, offsets, capacity, n_images, launches, lengths_dev, err_dev,
                 done=None, stream=None, validate=None):
        self._out = out
        self._offsets = offsets
        self._capacity = capacity
        self._n_images = n_images
        self.launches = launches
        self._lengths = None
        self._devs = (lengths_dev, err_dev)  # read on first use (no per-render pinned buffers)
        self._done = done
        self.stream = stream
        self._validate = validate

    def _settle(self) -> None:
        v = self._validate
        if v is not None:
            self._validate = None
            v(self)

    def _redo(self, r: "RenderResult", done) -> None:
        """Replace the fields by those of `r` (a re-captured plan slot)."""
        self._out, self._offsets, self._capacity = r._out, r._offsets, r._capacity
        self._n_images, self._devs, self._done, self._lengths = r._n_images, r._devs, done, None

    out = property(lambda self: (self._settle(), self._out)[1])
    offsets = property(lambda self: (self._settle(), self._offsets)[1])
    capacity = property(lambda self: (self._settle(), self._capacity)[1])
    n_images = property(lambda self: (self._settle(), self._n_images)[1])
    _dev = property(lambda self: (self._settle(), self._devs)[1])

    @property
    def done(self):
        self._settle()
        return self._done

    @done.setter
    def done(self, ev):
        self._settle()
        self._done = ev

    @property
    def precision(self) -> str:
        """Engine that rendered it: "fp32" fast or "fp64" exact."""
        return "fp64" if self.out.dtype == torch.float64 else "fp32"

    def wait(self) -> "RenderResult":
        """Order the current stream after the render (no host wait)."""
        done = self.done
        if done is not None:
            torch.cuda.current_stream(self._out.device).wait_event(done)
        return self

    @property
    def lengths(self) -> np.ndarray:
        """Per-job out_len (synth.py:211-212)."""
        if self._lengths is None:
            self.wait()
            lengths_dev, err_dev = self._dev
            h = torch.cat([lengths_dev, err_dev.to(torch.int64)]).cpu().numpy()
            if h[-1]:
                raise _lib.MvbError("output length exceeded its planned bound "
                                    f"(lengths {h[:-1].tolist()}, capacity {self.capacity.tolist()})")
            self._lengths = h[:-1].copy()
        return self._lengths

    @property
    def updates(self) -> int:
        """image x output-sample updates computed."""
        return int(np.sum(self.lengths * self.n_images))

    @staticmethod
    def concat(parts: list) -> "RenderResult":
        """One result for consecutive sub-batches (outputs concatenated)."""
        for p in parts:
            p.wait()
        shift = np.concatenate([[0], np.cumsum([p.out.numel() for p in parts])[:-1]])
        return RenderResult(torch.cat([p.out for p in parts]),
                            np.concatenate([p.offsets + d for p, d in zip(parts, shift)]),
                            np.concatenate([p.capacity for p in parts]),
                            np.concatenate([p.n_images for p in parts]),
                            sum(p.launches for p in parts),
                            torch.cat([p._dev[0] for p in parts]),
                            torch.stack([p._dev[1] for p in parts]).amax(dim=0))

    def job(self, j: int) -> torch.Tensor:
        return self.out[self.offsets[j]:self.offsets[j] + self.lengths[j]]

    def host(self) -> np.ndarray:
        """The flat output as numpy (pinned D2H, waits for the render)."""
        self.wait()
        return d2h(self.out)


CHUNK_MIN_IMAGES = int(os.environ.get("MVB_CHUNK_MIN_IMAGES", "320"))
CHUNK_WAVES = float(os.environ.get("MVB_CHUNK_WAVES", "18"))  # target waves of 3 CTAs / SM
# batches with few tiles (c2: 131) need many chunks per tile to fill the GPU;
# there smaller chunks win (c2 synthesis 0.335 -> 0.233 ms at 160), while a
# W = 8 image shard of c3 (1050 tiles, 1440 images) is 1.5% faster at 320
SMALL_GRID_TILES, SMALL_GRID_CHUNK_MIN = 512, 160


def _chunking(n_imgs, tiles, sm_count):
    """Image chunks per (job, tile): enough CTAs for ~18 waves of 3 CTAs/SM
    (a partial last wave then costs little), chunks of >= CHUNK_MIN_IMAGES
    images (a CTA's staging prologue and reduction epilogue amortise over
    them; image shards with ~1.4k images per job were 2% slower at 128)."""
    total_tiles = int(sum(tiles))
    want = int(CHUNK_WAVES * 3 * sm_count)
    if total_tiles >= want:
        return [1] * len(n_imgs)
    cmin = SMALL_GRID_CHUNK_MIN if total_tiles < SMALL_GRID_TILES else CHUNK_MIN_IMAGES
    out = []
    for S, t in zip(n_imgs, tiles):
        per = max(1, math.ceil(want / max(total_tiles, 1)))
        per = min(per, max(1, S // cmin))
        out.append(per)
    return out


def render(geom: Geometry, signals: list, filt, precision: str = "fp32",
           signal_keys=None, timing: list | None = None) -> RenderResult:
    """Synthesize every job of `geom` (signals[j] is job j's dry signal).
    `timing`, if a list, receives (start, end) CUDA events recorded on the
    launch stream around the synthesis kernel."""
    return prepare_render(geom, signals, filt, precision, signal_keys).launch(timing)


class PreparedRender:
    """A render up to its synthesis launch: the host plan is done and the
    device work that does not need the exact track maxima (interval
    records, delay sort, branch records, output buffers) is enqueued.
    `launch()` enqueues the rest -- exact output lengths from the (possibly
    cross-rank reduced) maxima, synthesis, partial-sum reduction -- so a
    render plan can capture the two halves into separate graphs and replay
    them on different streams."""

    def __init__(self, launch_fn, launches0):
        self._launch = launch_fn
        self._launches0 = launches0

    def launch(self, timing: list | None = None) -> RenderResult:
        res = self._launch(timing)
        res.launches = _lib.launch_count() - self._launches0
        return res


def prepare_render(geom: Geometry, signals: list, filt, precision: str = "fp32",
                   signal_keys=None, fork=None) -> PreparedRender:
    """First half of render() (see PreparedRender).  `fork`: two extra
    streams (render plans, during graph capture): the delay sort and the
    branch records then run as parallel branches next to the interval
    records (they depend on the coarse tracks / the signal only), joined
    before the function returns, so the captured graph's critical path is
    the longest of the three instead of their sum."""
    dev = geom.dev
    st = stream_handle(dev)
    jobs = geom.jobs
    nJ = len(jobs)
    f = as_filter(filt)
    L, d0 = int(f.branch_len), int(f.nominal_delay)
    if precision not in ("fp32", "fp64"):
        raise ValueError("precision must be 'fp32' or 'fp64'")
    if precision == "fp32" and not geom.fast_path_ok:
        # delay excursions beyond the fp32 residual's envelope (sources or
        # receivers moving at hundreds of m/s under a large decimation):
        # the exact fp64 engine renders the batch instead
        precision = "fp64"
    if precision == "fp64" and any(jb.window is not None for jb in jobs):
        raise ValueError("time-shard windows need the fp32 fast path (the exact engine runs "
                         "replicas only; fast sources beyond the fp32 envelope cannot be sharded)")
    sm_count = _sm_count(dev.index if dev.index is not None else torch.cuda.current_device())
    # signals: dedupe, upload
    keys = signal_keys or [_key(jobs[j].signal_key, signals[j]) for j in range(nJ)]
    uniq = {}
    for j in range(nJ):
        uniq.setdefault(keys[j], []).append(j)
    dt = torch.float32 if precision == "fp32" else torch.float64
    sig_dev, sig_len = {}, {}
    host_sigs, n_host = [], 0
    for k, members in uniq.items():
        s = signals[members[0]]
        if isinstance(s, torch.Tensor):
            t = s.to(dev, dt).reshape(-1).contiguous()
            sig_dev[k], sig_len[k] = t, t.numel()
        else:
            a = np.asarray(s).reshape(-1)
            host_sigs.append((k, n_host, a))
            sig_len[k] = a.size
            n_host += a.size
        if sig_len[k] == 0:
            raise ValueError("input must be a nonempty 1-D signal")
    if host_sigs:  # all host signals: one bulk upload, device views per key
        sig_all = torch.empty(n_host, dtype=dt, device=dev)
        _STAGER.upload([(r0, a) for _, r0, a in host_sigs], sig_all)
        for k, r0, a in host_sigs:
            sig_dev[k] = sig_all[r0:r0 + a.size]
    base_rows = [dict(r, L=L, d0=d0) for r in geom.job_rows]
    launches0 = _lib.launch_count()

    def finish_rows():
        """Capacities from the host-side bound of every output length (no
        wait for the geometry kernels); the exact lengths are written into
        the device job table by mvb_finalize_lengths (finalize)."""
        out_len = np.zeros(nJ, np.int64)
        tau_bound = np.zeros(nJ, np.int64)
        for j in range(nJ):
            tau_bound[j] = geom.length_bound(j)
            out_len[j] = sig_len[keys[j]] + tau_bound[j] + L
        offsets = np.concatenate([[0], np.cumsum(out_len)[:-1]]).astype(np.int64)
        rows = [dict(r) for r in base_rows]
        for j in range(nJ):
            rows[j].update(out_off=int(offsets[j]), out_len=int(out_len[j]),
                           ls=int(sig_len[keys[j]] + L - 1))
        return out_len, tau_bound, offsets, rows

    def finalize(jobs_dev, st):
        geom.join()  # the exact maxima (a parallel branch in plan captures)
        lengths = torch.empty(nJ, dtype=torch.int64, device=dev)
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.call("mvb_finalize_lengths", ptr(jobs_dev), nJ, ptr(geom.dmax_dev), ptr(lengths),
                  ptr(err), st)
        return lengths, err

    if precision == "fp64":
        nb = int(f.poly_order) + 1
        br = h2d(np.asarray(f.branches, dtype=np.float64), dev)
        base, bases = 0, {}
        for k in uniq:
            bases[k] = base
            base += nb * (sig_len[k] + L - 1)
        streams = torch.empty(base, dtype=torch.float64, device=dev)
        for k in uniq:
            _lib.call("mvb_branch_filter", ptr(sig_dev[k]), sig_len[k], ptr(br), nb, L,
                      ptr(streams[bases[k]:]), st)
        out_len, _, offsets, rows = finish_rows()
        for j in range(nJ):
            rows[j].update(rec_base=bases[keys[j]], nb=nb)
        jobs_dev = h2d(pack_jobs(rows), dev)
        out = torch.zeros(int(out_len.sum()), dtype=torch.float64, device=dev)

        def launch64(timing):
            st = stream_handle(dev)
            lengths, err = finalize(jobs_dev, st)
            ev = _events(timing)
            _lib.call("mvb_synthesize_f64_ex", ptr(jobs_dev), nJ, int(out_len.max()),
                      ptr(geom.images), ptr(geom.coarse), ptr(geom.tables), ptr(streams),
                      ptr(geom.paths), ptr(out), int(geom.n_img.max()), st)
            _events_end(timing, ev)
            return RenderResult(out, offsets, out_len, geom.n_img.copy(), 0, lengths, err)
        return PreparedRender(launch64, launches0)

    # ---------------------------------------------------------------- fast --
    _mark("render.signals")
    cb, M1, nb = fast_bank(f)
    pre_dev = h2d(pack_jobs(base_rows), dev)
    out_len, tau_bound, offsets, rows = finish_rows()
    concat = sig_all if host_sigs and len(host_sigs) == len(uniq) else None
    # record groups: batches whose interval records exceed RECORD_BUDGET get
    # them computed group by group into two alternating buffers, inside the
    # synthesis launch (launch32), instead of all up front
    groups = _record_groups(geom) if FD_GATHER != "table" else None
    rec_bufs = None
    if groups:
        lay = geom.rec_layout
        most = max(int(lay["kbase"][b - 1] + lay["per_job"][b - 1] - lay["kbase"][a])
                   for a, b in groups)
        rec_bufs = [torch.empty(most * 12, dtype=torch.float32, device=dev)
                    for _ in range(min(2, len(groups)))]
    main = torch.cuda.current_stream(dev)
    if fork is not None:
        forked = torch.cuda.Event()
        forked.record(main)
        for fs in fork:  # every branch stream joins the capture (unused ones too)
            fs.wait_event(forked)
        with torch.cuda.stream(fork[0]):
            images_sorted, n_seg, max_seg, max_img, keyed = _delay_sort(geom, pre_dev,
                                                                 stream_handle(dev))
        with torch.cuda.stream(fork[1]):
            rec, rec_start = _branch_records(uniq, sig_dev, sig_len, tau_bound, L, cb, M1, nb, dev,
                                             stream_handle(dev), concat)
        coef = None if groups else _interval_records(geom, pre_dev, st, fork=fork[2:])
        for fs in fork:
            main.wait_stream(fs)
    else:
        coef = None if groups else _interval_records(geom, pre_dev, st)
        _mark("render.coeffs_keys")
        images_sorted, n_seg, max_seg, max_img, keyed = _delay_sort(geom, pre_dev, st)
        _mark("render.sorted")
        rec, rec_start = _branch_records(uniq, sig_dev, sig_len, tau_bound, L, cb, M1, nb, dev, st,
                                         concat)
    _mark("render.plan_lengths")
    table = None
    if FD_GATHER == "table":  # literal per-fraction table, not the product
        rec, table = _table_records(uniq, sig_dev, sig_len, rec_start, rec.numel() // (
            4 if nb == 4 else 8 * -(-nb // 8)), f, dev, st, concat)
    rec_rows = rec.numel() // (1 if table is not None else (4 if nb == 4 else 8 * -(-nb // 8)))
    for j in range(nJ):
        rows[j].update(rec_base=rec_start[keys[j]], nb=nb, img_off=j * max_seg * max_img,
                       img_stride=max_img, rec_rows=rec_rows)
    work, part_rows = _work_list(geom.n_img, out_len, n_seg, sm_count, rows, geom.jobs)
    work_at = np.searchsorted(work[:, 0], np.arange(nJ + 1), side="left")  # job j: [at[j], at[j+1])
    _mark("render.records_plan")
    jobs_dev = h2d(pack_jobs(rows), dev)
    work_dev = h2d(work, dev)
    out = torch.zeros(int(out_len.sum()), dtype=torch.float32, device=dev)
    part = torch.empty(max(part_rows, 1), dtype=torch.float32, device=dev)
    _mark("render.work_upload")

    def synth(w0, w1, coef_p, st):
        # work items [w0, w1) with the interval records at coef_p
        wp = work_dev.data_ptr() + 32 * int(w0)
        if keyed is not None and TEX_GATHER and nb == 8:
            _lib.call("mvb_synthesize_f32_tex", ptr(jobs_dev), wp, int(w1 - w0),
                      ptr(images_sorted), ptr(keyed[0]), keyed[1], SEG_LEN,
                      max(geom.factors, default=1), ptr(geom.bbox), coef_p, ptr(rec), rec.numel(),
                      ptr(geom.paths), ptr(out), ptr(part), nb, TEX_GATHER, st)
        elif keyed is not None:
            _lib.call("mvb_synthesize_f32_ranged", ptr(jobs_dev), wp, int(w1 - w0),
                      ptr(images_sorted), ptr(keyed[0]), keyed[1], SEG_LEN,
                      max(geom.factors, default=1), ptr(geom.bbox), coef_p, ptr(rec),
                      ptr(geom.paths), ptr(out), ptr(part), nb, SYNTH_U, st)
        else:
            _lib.call("mvb_synthesize_f32", ptr(jobs_dev), wp, int(w1 - w0),
                      ptr(images_sorted), coef_p, ptr(rec), ptr(geom.paths), ptr(out),
                      ptr(part), nb, SYNTH_U, st)

    def launch32(timing):
        st = stream_handle(dev)
        lengths, err = finalize(jobs_dev, st)
        ev = _events(timing)
        if table is not None:
            _lib.call("mvb_synthesize_f32_table", ptr(jobs_dev), ptr(work_dev), len(work),
                      ptr(images_sorted), ptr(coef), ptr(rec), ptr(geom.paths), ptr(out),
                      ptr(part), ptr(table), L, st)
        elif groups:
            _grouped_synthesis(geom, pre_dev, groups, rec_bufs, work_dev, work_at,
                               lambda w0, w1, coef_p, s: synth(w0, w1, coef_p, s))
        else:
            synth(0, len(work), coef.data_ptr(), st)
        _events_end(timing, ev)
        if part_rows:
            _lib.call("mvb_reduce_partials_f32", ptr(jobs_dev), nJ, int(out_len.max()),
                      ptr(part), ptr(out), st)
        _mark("render.synth_launched")
        return RenderResult(out, offsets, out_len, geom.n_img.astype(np.int64), 0, lengths, err)
    return PreparedRender(launch32, launches0)


# Interval-record budget of one render (bytes).  Grouping bounds the
# footprint but costs time: c4 (32 GB of records) with 2 GB groups ran 99 ms
# per step against 90.5 ungrouped (a group's records and the previous
# group's synthesis share the SMs under different shared-memory carveouts;
# a high-priority records stream: 121 ms).  So the default only groups what
# would not fit comfortably: a quarter of the device memory (45 GB on a
# B200); MVB_RECORD_BUDGET_GB sets it (2: c4's plan slot holds 4 GB of
# records instead of 32).
RECORD_BUDGET = float(os.environ["MVB_RECORD_BUDGET_GB"]) * 2 ** 30 \
    if os.environ.get("MVB_RECORD_BUDGET_GB") else None


def _record_budget(dev) -> float:
    if RECORD_BUDGET is not None:
        return RECORD_BUDGET
    return 0.25 * torch.cuda.get_device_properties(dev).total_memory


def _record_groups(geom):
    """Consecutive job ranges [j0, j1) whose interval records (48 B per
    coarse interval) fit RECORD_BUDGET each, cut at equal record counts; None
    when the whole batch fits (or its layout is not uniform:
    Geometry.rec_layout).  With a 2 GB budget c4's 32 GB of records run
    as 16 groups in two alternating 2 GB buffers."""
    lay = geom.rec_layout
    total = 48 * int(geom.n_coarse_total)
    nJ = len(geom.jobs)
    budget = _record_budget(geom.dev)
    if lay is None or total <= budget or nJ < 2:
        return None
    n = min(nJ, -(-total // int(budget)))
    cum = np.concatenate([[0], np.cumsum(lay["per_job"])])
    cuts = np.searchsorted(cum, cum[-1] * np.arange(n + 1) / n, side="left")
    cuts[0], cuts[-1] = 0, nJ
    cuts = np.unique(np.clip(cuts, 0, nJ))
    return [(int(a), int(b)) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]


def _group_streams(dev):
    key = ("groups", str(dev))
    if key not in _GROUP_STREAMS:
        # equal priorities (a high-priority records stream measured 121 ms
        # per c4 step against 99: MVB_GROUP_REC_PRIORITY=-1)
        _GROUP_STREAMS[key] = (torch.cuda.Stream(device=dev, priority=GROUP_REC_PRIORITY),
                               torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev))
    return _GROUP_STREAMS[key]


_GROUP_STREAMS = {}
GROUP_REC_PRIORITY = int(os.environ.get("MVB_GROUP_REC_PRIORITY", "0"))


def _grouped_synthesis(geom, pre_dev, groups, bufs, work_dev, work_at, synth) -> None:
    """Interval records and synthesis group by group: the records of group
    g go to bufs[g % 2] (image coef offsets rebased by the group's first
    coarse sample) on one stream, its synthesis (work items of its jobs) on
    another; group g + 2 reuses the buffer once group g's synthesis is done,
    so group g + 1's records overlap group g's synthesis.  Forks from and
    joins the current stream (legal inside a graph capture)."""
    dev = geom.dev
    lay = geom.rec_layout
    main = torch.cuda.current_stream(dev)
    sa, *sbs = _group_streams(dev)  # records; synthesis on alternating streams
    start = torch.cuda.Event()       # (group g + 1's CTAs fill group g's tail)
    start.record(main)
    for x in (sa, *sbs):
        x.wait_event(start)
    windowed = any(jb.window is not None for jb in geom.jobs)
    done = []
    for g, (j0, j1) in enumerate(groups):
        coef_p = bufs[g % len(bufs)].data_ptr() - 48 * int(lay["kbase"][j0])
        with torch.cuda.stream(sa):
            if g >= len(bufs):
                sa.wait_event(done[g - len(bufs)])
            for N, sel in geom.sel_by_factor.items():
                off, cnt = lay["sel"][N]
                part = sel[off + j0 * cnt: off + j1 * cnt]
                fit = np.ascontiguousarray(phase_fit(N), dtype=np.float64)
                max_K = coarse_span(geom.job_rows[j0:j1], N)
                _lib.call("mvb_track_coeffs_windowed" if windowed else "mvb_track_coeffs",
                          ptr(geom.images), ptr(part), part.numel(), max_K, ptr(pre_dev),
                          ptr(geom.coarse), fit.ctypes.data_as(ctypes.c_void_p), coef_p,
                          stream_handle(dev))
            ready = torch.cuda.Event()
            ready.record(sa)
        sb = sbs[g % 2]
        with torch.cuda.stream(sb):
            sb.wait_event(ready)
            synth(work_at[j0], work_at[j1], coef_p, stream_handle(dev))
            ev = torch.cuda.Event()
            ev.record(sb)
            done.append(ev)
    for x in (sa, *sbs):
        main.wait_stream(x)


def _interval_records(geom, pre_dev, st, fork=()) -> torch.Tensor:
    """Fast-path interval records (mvb_coef32, 12 floats) of every decimated
    image, one mvb_track_coeffs launch per decimation factor; with `fork`
    streams (graph capture) the factors after the first run as parallel
    branches (the caller joins them)."""
    dev = geom.dev
    coef = torch.empty(max(geom.n_coarse_total, 1) * 12, dtype=torch.float32, device=dev)
    windowed = any(jb.window is not None for jb in geom.jobs)
    main = torch.cuda.current_stream(dev)
    start = torch.cuda.Event()
    start.record(main)  # fork point: before the first factor's launch
    for q, (N, sel) in enumerate(geom.sel_by_factor.items()):
        fit = np.ascontiguousarray(phase_fit(N), dtype=np.float64)
        max_K = coarse_span(geom.job_rows, N)
        fs = fork[(q - 1) % len(fork)] if q and fork else main
        if fs is not main:
            fs.wait_event(start)
        with torch.cuda.stream(fs):
            _lib.call("mvb_track_coeffs_windowed" if windowed else "mvb_track_coeffs",
                      ptr(geom.images), ptr(sel), sel.numel(), max_K,
                      ptr(pre_dev), ptr(geom.coarse), fit.ctypes.data_as(ctypes.c_void_p),
                      ptr(coef), stream_handle(dev))
    return coef


def _delay_sort(geom, pre_dev, st):
    """Image records of every job sorted by delay per SEG_LEN-sample time
    segment (L1 locality of the gathers) into the (job, segment, max_img)
    layout: mvb_delay_sort (one block radix sort per segment) up to
    DELAY_SORT_MAX images per job; beyond, keys by mvb_sort_keys, one
    batched argsort (padding keys +inf sort last, padded slots repeat an own
    image) and mvb_gather_images."""
    dev, nJ = geom.dev, len(geom.jobs)
    n_seg = [-(-int(geom.T[j]) // SEG_LEN) for j in range(nJ)]
    max_seg, max_img = max(n_seg), int(geom.n_img.max())
    windowed = any(jb.window is not None for jb in geom.jobs)
    if max_img <= _lib.DELAY_SORT_MAX or windowed:
        # fused keys + block radix sort + gather, one launch.  Time-shard
        # jobs (image table in delay-band order, parallel.band_order) sort
        # in independent runs of SORT_RUN images: a few segments per rank,
        # each one 16k-key block sort, would be a ~140 us chain at W = 8
        images_sorted = torch.empty(nJ * max_seg * max_img, IMG_COLS, dtype=torch.int64,
                                    device=dev)
        key_bits = max(1, min(32, max(int(geom.length_bound(j)) for j in range(nJ)).bit_length()))
        run_len = SORT_RUN if windowed else max(max_img, 1)
        if ACTIVE_RANGES:
            # the sorted keys let each synthesis tile skip the images that
            # read only zero pads there (mvb_synthesize_f32_ranged)
            keys = torch.empty(nJ * max_seg * max_img, dtype=torch.int32, device=dev)
            _lib.call("mvb_delay_sort_keyed", ptr(geom.images), ptr(pre_dev), nJ, max_img,
                      max_seg, SEG_LEN, ptr(geom.paths), ptr(geom.coarse), key_bits, run_len,
                      ptr(images_sorted), ptr(keys), st)
            return images_sorted, n_seg, max_seg, max_img, (keys, run_len)
        if windowed:
            _lib.call("mvb_delay_sort_runs", ptr(geom.images), ptr(pre_dev), nJ, max_img, max_seg,
                      SEG_LEN, ptr(geom.paths), ptr(geom.coarse), key_bits, SORT_RUN,
                      ptr(images_sorted), st)
        else:
            _lib.call("mvb_delay_sort", ptr(geom.images), ptr(pre_dev), nJ, max_img, max_seg,
                      SEG_LEN, ptr(geom.paths), ptr(geom.coarse), key_bits, ptr(images_sorted), st)
        return images_sorted, n_seg, max_seg, max_img, None
    key = torch.full((nJ, max_seg, max_img), float("inf"), dtype=torch.float64, device=dev)
    _lib.call("mvb_sort_keys", ptr(geom.images), ptr(pre_dev), nJ, max_img, max_seg, SEG_LEN,
              ptr(geom.paths), ptr(geom.coarse), ptr(key), st)
    order = torch.argsort(key, dim=2)
    base = h2d(geom.img_off, dev)[:, None, None]
    nimg_dev = h2d(geom.n_img, dev)[:, None, None]
    gidx = (base + torch.minimum(order, nimg_dev - 1)).reshape(-1)
    images_sorted = torch.empty(gidx.numel(), IMG_COLS, dtype=torch.int64, device=dev)
    _lib.call("mvb_gather_images", ptr(geom.images), ptr(gidx), gidx.numel(), ptr(images_sorted), st)
    return images_sorted, n_seg, max_seg, max_img, None


def _branch_records(uniq, sig_dev, sig_len, tau_bound, L, cb, M1, nb, dev, st, concatenated=None):
    """Zero-padded fp32 branch records of every distinct signal (mvb.h
    layout) in one launch.  A signal's region is [front pad | len + L - 1
    rows | back pad] with the front pad covering the largest delay bound of
    the jobs using it, so every gather row is in range.  Returns the record
    buffer and, per signal key, the global row of its sample 0."""
    rec_rows, start, zlo, zhi = 0, {}, {}, {}
    for k, members in uniq.items():
        front = int(max(tau_bound[j] for j in members)) + L + PAD_MARGIN
        back = front + TILE + PAD_MARGIN
        zlo[k] = rec_rows
        start[k] = rec_rows + front
        rec_rows += front + sig_len[k] + L - 1 + back
        zhi[k] = rec_rows
    if rec_rows + int(max(sig_len.values())) + int(max(tau_bound)) + 2 * L >= 2**31 - 0x4B400000:
        raise ValueError("batch too large for 32-bit record rows; split it")
    row_floats = 4 if nb == 4 else 8 * -(-nb // 8)  # mvb.h record layout
    # no zero fill: the records kernel writes every signal's pads as zeros
    rec = torch.empty(rec_rows * row_floats, dtype=torch.float32, device=dev)
    ukeys = list(uniq)
    lens = np.asarray([sig_len[k] for k in ukeys], np.int64)
    if len(ukeys) == 1:
        x_all = sig_dev[ukeys[0]]
    elif concatenated is not None:
        x_all = concatenated  # host signals were uploaded back to back in key order
    else:
        x_all = torch.cat([sig_dev[k] for k in ukeys])
    sig_tab = h2d(np.stack([np.concatenate([[0], np.cumsum(lens)[:-1]]), lens,
                            np.asarray([start[k] for k in ukeys], np.int64),
                            np.asarray([zlo[k] for k in ukeys], np.int64),
                            np.asarray([zhi[k] for k in ukeys], np.int64)]), dev)
    cb_dev = h2d(np.ascontiguousarray(cb), dev)
    max_rows = max(zhi[k] - zlo[k] for k in ukeys)
    _lib.call("mvb_branch_records_f32", ptr(x_all), ptr(sig_tab[0]), ptr(sig_tab[1]),
              ptr(sig_tab[2]), ptr(sig_tab[3]), ptr(sig_tab[4]), len(ukeys), int(max_rows),
              ptr(cb_dev), M1, L, nb, ptr(rec), st)
    return rec, start


TAB_P = 512  # mvb.h MVB_TAB_P
# MVB_FD_GATHER=table: the fast synthesis gathers through the literal
# per-fraction table instead of the Farrow records (measurement only)
FD_GATHER = os.environ.get("MVB_FD_GATHER", "farrow")
# per-tile active image ranges from the sorted keys (mvb_synthesize_f32_ranged);
# MVB_ACTIVE_RANGES=0: every tile walks its whole chunk (A/B)
ACTIVE_RANGES = os.environ.get("MVB_ACTIVE_RANGES", "1") != "0"
# measurement variant: gathers through the texture pipe (1: all, 2: odd steps)
TEX_GATHER = int(os.environ.get("MVB_TEX_GATHER", "0"))


def fraction_table(filt) -> np.ndarray:
    """(TAB_P + 1, L) fp32 taps h_j(p / TAB_P) = sum_k c_k[j] (p / TAB_P)^k of
    the filter's Farrow bank (farrow.py:42-63 basis), evaluated in fp64."""
    f = as_filter(filt)
    mu = np.arange(TAB_P + 1, dtype=np.float64) / TAB_P
    powers = mu[:, None] ** np.arange(f.branches.shape[0])[None, :]
    return np.ascontiguousarray(powers @ np.asarray(f.branches, dtype=np.float64),
                                dtype=np.float32)


def _table_records(uniq, sig_dev, sig_len, start, rec_rows, filt, dev, st, concatenated=None):
    """The table A/B's inputs: the zero-padded signal plane (one float per
    branch-record row, same row numbering) and the fraction table."""
    ukeys = list(uniq)
    lens = np.asarray([sig_len[k] for k in ukeys], np.int64)
    if len(ukeys) == 1:
        x_all = sig_dev[ukeys[0]]
    elif concatenated is not None:
        x_all = concatenated
    else:
        x_all = torch.cat([sig_dev[k] for k in ukeys])
    sig_tab = h2d(np.stack([np.concatenate([[0], np.cumsum(lens)[:-1]]), lens,
                            np.asarray([start[k] for k in ukeys], np.int64)]), dev)
    xp = torch.zeros(rec_rows, dtype=torch.float32, device=dev)
    _lib.call("mvb_signal_plane_f32", ptr(x_all), ptr(sig_tab[0]), ptr(sig_tab[1]), ptr(sig_tab[2]),
              len(ukeys), int(lens.max()), ptr(xp), st)
    return xp, h2d(fraction_table(filt), dev)


# Work-item order (MVB_WORK_ORDER; measured same box, synthesis ms, chunk-major
# / cost-descending / tile-major / tiles by total cost with their chunks
# adjacent): c3 8.20 / 8.06 / 8.03 / 7.83, c5 21.87 / 21.66 / 21.59 / 21.62,
# c2 0.244 / 0.384 / 0.367 / 0.380 -- small grids (c2: 131 tiles x 11 chunks,
# 3.2 waves) keep chunk-major order (an image's consecutive tiles share their
# interval-record lines), larger ones take order 3.  -1 = this rule.
WORK_ORDER = int(os.environ.get("MVB_WORK_ORDER", "-1"))


def _delay_estimates(jb) -> np.ndarray:
    """Sorted structural delay estimates (samples) of a job's images:
    kappa * |j * dims| (the image of the room centre), cached per structure."""
    return _delay_est(_est_key(jb))[0]


def _cost_prefix(jb) -> np.ndarray:
    """Prefix sums (length S + 1) of the per-image synthesis cost weights
    in the sorted-delay order of _delay_estimates: a full-rate image (fp64
    distance per sample) ~3 decimated ones; a decimated image pays its
    interval records' broadcast on top of the 8.75-wavefront gather,
    1 + (6 wavefronts x 32 / N) / 8.75 -- N = 16 about twice N = 256."""
    return _delay_est(_est_key(jb))[1]


def _est_key(jb):
    return (np.asarray(jb.dims, np.float64).tobytes(), int(jb.max_order),
            None if jb.image_index is None else np.asarray(jb.image_index, np.int64).tobytes(),
            float(jb.rate) / float(jb.c), tuple((int(a), int(b)) for a, b in jb.tiers))


@functools.lru_cache(maxsize=64)
def _delay_est(key) -> tuple:
    from . import parallel
    dims_b, max_order, images_b, kappa, tiers = key
    j, order = parallel.canonical_lattice(max_order)
    if images_b is not None:
        sel = np.frombuffer(images_b, dtype=np.int64)
        j, order = j[sel], order[sel]
    tau = kappa * np.linalg.norm(j * np.frombuffer(dims_b, np.float64)[None, :], axis=1)
    N = np.ones(order.size)
    prev = -1
    for mo, f in tiers:
        N[(order > prev) & (order <= mo)] = f
        prev = mo
    w = np.where(N == 1, 3.0, 1.0 + (6.0 * 32.0 / np.maximum(N, 1)) / 8.75)
    idx = np.argsort(tau, kind="stable")
    return tau[idx], np.concatenate([[0.0], np.cumsum(w[idx])])


def _work_list(n_img, out_len, n_seg, sm_count, rows, jobs=None):
    """mvb_work items (job, tile, image range, chunk, sort segment) of every
    job, image ranges split into chunks (_chunking); chunked jobs get
    partial-output rows (rows[j]['n_chunks'], ['part_off'] are set).  A
    time-shard job (rows[j] w0 / w1) gets the tiles of its window only.
    With `jobs`, each job's items are ordered by their estimated cost --
    the chunk's images whose structural delay estimate puts a row inside
    the signal over the tile (the synthesis visits only those, §5.6 of
    DESIGN.md) -- most expensive first: the CTAs dispatched last, which
    set the kernel's tail, are the cheap front / tail tiles.  Jobs stay
    contiguous (record groups slice the list by job)."""
    nJ = len(rows)
    first = [int(rows[j].get("w0", 0)) // TILE for j in range(nJ)]
    end = [-(-int(out_len[j]) // TILE) for j in range(nJ)]
    end = [min(e, int(rows[j]["w1"]) // TILE) if rows[j].get("w1", 0) > 0 else e
           for j, e in enumerate(end)]
    tiles = [max(e - a, 0) for a, e in zip(first, end)]
    chunks = _chunking([int(v) for v in n_img], tiles, sm_count)
    part_rows, blocks = 0, []
    for j in range(nJ):
        nc = chunks[j] if n_img[j] > 0 else 1
        rows[j]["n_chunks"] = nc
        if nc > 1:
            rows[j]["part_off"] = part_rows
            part_rows += nc * int(out_len[j])
        span = int(n_img[j])
        cs = np.arange(nc)
        blk = np.zeros((nc, tiles[j], 8), dtype=np.int32)
        blk[:, :, 0] = j
        tj = np.arange(first[j], first[j] + tiles[j])
        blk[:, :, 1] = tj[None, :]
        blk[:, :, 2] = ((span * cs) // nc)[:, None]
        blk[:, :, 3] = ((span * (cs + 1)) // nc)[:, None]
        blk[:, :, 4] = cs[:, None]
        blk[:, :, 5] = np.minimum(tj * TILE // SEG_LEN, n_seg[j] - 1)[None, :]
        blk = blk.reshape(-1, 8)
        order = WORK_ORDER if WORK_ORDER >= 0 else \
            (0 if sum(tiles) < SMALL_GRID_TILES else 3)
        if order and jobs is not None and len(blk) > 1:
            tau, W = _delay_estimates(jobs[j]), _cost_prefix(jobs[j])
            ls = int(rows[j]["ls"])
            n0 = blk[:, 1].astype(np.float64) * TILE
            b, e = blk[:, 2], blk[:, 3]
            # weighted images of [b, e) (sorted-delay positions) with
            # n0 - ls < tau <= n0 + TILE, plus a little per image visited
            lo = np.clip(np.searchsorted(tau, n0 - ls, side="right"), b, e)
            hi = np.clip(np.searchsorted(tau, n0 + TILE, side="right"), b, e)
            cost = (W[hi] - W[lo]) + 0.05 * (e - b)
            if order == 1:
                blk = blk[np.argsort(-cost, kind="stable")]
            elif order == 2:  # tile-major (the chunks of a tile adjacent)
                blk = blk[np.lexsort((blk[:, 4], blk[:, 1]))]
            elif order == 3:  # tiles by their total cost, chunks of a tile adjacent
                tc = np.bincount(blk[:, 1] - blk[:, 1].min(), weights=cost)
                blk = blk[np.lexsort((blk[:, 4], blk[:, 1], -tc[blk[:, 1] - blk[:, 1].min()]))]
            elif order == 4:  # chunk-major, each chunk's tiles by cost
                blk = blk[np.lexsort((-cost, blk[:, 4]))]
            elif order == 5:  # chunks by total cost (most first), chunk-major
                cc = np.bincount(blk[:, 4], weights=cost)
                blk = blk[np.lexsort((blk[:, 1], blk[:, 4], -cc[blk[:, 4]]))]
        blocks.append(blk)
    work = np.concatenate(blocks)
    if len(work) == 0:  # every window past its job's length bound: one idle item
        work = np.zeros((1, 8), np.int32)
        work[0, 1] = end[0]  # n0 >= out_len: the CTA returns at once
    return work, part_rows
