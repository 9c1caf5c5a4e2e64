"""CUDA-graph render plans: repeated renders of one job structure.

A plan fixes the structure of a batch -- per job the path length, signal
length, receiver kind, room, image order, tier table, filter and precision --
and captures every kernel of a render into CUDA graphs: the staging (path
copies, bounding boxes, bandwidth indices and their two small readbacks),
the geometry and the synthesis.  Each `run` copies the new inputs into the
plan's static buffers and replays the graphs, which recompute all
data-dependent work (boxes, bandwidths, coarse tracks, bounds, exact maxima,
interval records, delay sort, branch records, output lengths, synthesis).
Only the host planning is amortised.  The replay is speculative: the host
decisions a capture is valid for (low-pass decision, fp32 envelope, output
capacities) are re-checked from the replayed readbacks on first use of the
result (RenderResult._settle), and when the new data changed them the run
is staged again, the slot captured again and replayed.

Each slot holds two graphs: the geometry graph (tracks, maxima, records,
sort, branch records -- short, mostly latency-bound kernels) replays on a
high-priority stream, the synthesis graph (exact lengths, synthesis,
partial sums) on the plan's synthesis stream.  Run k+1's geometry therefore
executes while run k's synthesis still occupies the GPU: its CTAs are
dispatched ahead of the synthesis' pending ones, so the geometry chain
leaves the critical path and back-to-back renders approach the synthesis
time alone.  Image shards reduce the track maxima across ranks between the
two graphs (eager collective on the geometry stream, never captured).

Two slots alternate; a slot is reused only after its previous replay
finished.  The RenderResult of a run references the slot's static output,
valid until that slot runs again (two runs later); it is produced on the
synthesis stream (`res.done`, `res.stream`; `res.job()` / `res.host()`
order the caller after it, `join()` orders the current stream after every
pending run).  A run orders its input copies after the caller's current
stream, so inputs written there before run() are seen.
"""

from __future__ import annotations

from dataclasses import replace

import os
import weakref

import numpy as np
import torch

from . import _lib, engine
from ._dev import StaticUploads, UploadMeter, release_pinned, require_cuda
from ._staging import _STAGER, copy_batch, side_stream

_NP_DTYPE = {torch.float64: np.dtype(np.float64), torch.float32: np.dtype(np.float32)}
from .farrow import as_filter


def _dims(a):
    return tuple(int(v) for v in a.shape) if hasattr(a, "shape") else tuple(np.shape(a))


def structure_key(jobs, filt, precision) -> tuple:
    """What a plan is valid for (data excluded, room constants included)."""
    f = as_filter(filt)
    key = [precision, id(f.branches) if isinstance(f.branches, torch.Tensor) else
           np.asarray(f.branches).tobytes(), f.branch_len, f.nominal_delay]
    # which jobs share a path / signal (first-occurrence index), not identities
    share_p, share_s = {}, {}
    for jb in jobs:
        share_p.setdefault(engine._key(jb.path_key, jb.pos), len(share_p))
        share_s.setdefault(engine._key(jb.signal_key, jb.s), len(share_s))
    for jb in jobs:
        key.append((_dims(jb.pos), _dims(jb.s), _dims(jb.mic),
                    np.asarray(jb.dims, np.float64).tobytes(),
                    np.asarray(jb.walls, np.float64).tobytes(), int(jb.max_order),
                    tuple((int(a), int(b)) for a, b in jb.tiers), float(jb.rate), float(jb.c),
                    float(jb.d_min),
                    None if jb.image_index is None else np.asarray(jb.image_index).tobytes(),
                    None if jb.window is None else tuple(int(v) for v in jb.window),
                    share_p[engine._key(jb.path_key, jb.pos)],
                    share_s[engine._key(jb.signal_key, jb.s)]))
    return tuple(key)


_STREAMS: dict = {}


def plan_streams(dev) -> tuple:
    """(geometry, synthesis) streams of the render plans on `dev`, shared
    by every plan on the device.  Both at the default priority: the next
    run's geometry then fills the drain of the running synthesis (FIFO
    dispatch); a high-priority geometry stream (MVB_GEO_PRIO) interleaves
    its CTAs into the synthesis and was measured slower."""
    key = str(dev)
    if key not in _STREAMS:
        _STREAMS[key] = (torch.cuda.Stream(device=dev, priority=int(os.environ.get("MVB_GEO_PRIO", "0"))),
                         torch.cuda.Stream(device=dev, priority=0))
    return _STREAMS[key]


_FORK: dict = {}


def fork_streams(dev) -> list:
    """Capture-only streams for the parallel branches of a geometry graph
    (delay sort, branch records, the second factor's interval records, the
    exact maxima); the captured graph records the fork / join, not the
    streams."""
    key = str(dev)
    if key not in _FORK:
        _FORK[key] = [torch.cuda.Stream(device=dev) for _ in range(4)]
    return _FORK[key]


class _Slot:
    def __init__(self):
        self.graph = None
        self.done = None
        self.decision = None
        self.capacity = None
        self.timing = []  # (start, end) events of the captured synthesis launch
        self.run_index = None  # run whose replay last used the slot
        self.pending = None  # result of an unvalidated speculative replay
        self.tag = f"@slot{id(self)}"  # its own pinned readback buffers (validation is deferred)


class RenderPlan:
    """Captured render of `jobs`' structure (see the module docstring)."""

    DEPTH = int(os.environ.get("MVB_PLAN_DEPTH", "2"))  # slots (diagnostic knob)

    def __init__(self, jobs, f, precision: str = "fp32", device=None, shard=None, dmax_hook=None):
        """`shard=(rank, world[, "images" | "time"])`: render the image
        shard / output window of `rank` of every job (parallel.shard_jobs,
        as synth.render_jobs) with `dmax_hook`
        (default: all-reduce MAX over the process group) applied to the
        track maxima between the geometry graph and the synthesis graph --
        the collective itself is issued eagerly on the geometry stream,
        never captured."""
        if precision not in ("fp32", "fp64"):
            raise ValueError("precision must be 'fp32' or 'fp64'")
        if shard is not None and int(shard[1]) > 1:
            from . import parallel
            if precision == "fp64":
                raise ValueError("the exact fp64 engine runs replicas only")
            rank, world = int(shard[0]), int(shard[1])
            jobs = parallel.shard_jobs(jobs, rank, world, parallel.shard_kind(shard))
            if dmax_hook is None:
                dmax_hook = parallel.allreduce_max
        self.shard = shard
        self.dmax_hook = dmax_hook
        self.dev = require_cuda(device)
        self.geo_stream, self.syn_stream = plan_streams(self.dev)
        self.fork_streams = fork_streams(self.dev)
        self.f = as_filter(f)
        self.precision = precision
        self.template = list(jobs)
        self.key = structure_key(jobs, f, precision)
        self.slots = []
        dt = torch.float32 if precision == "fp32" else torch.float64
        for _ in range(self.DEPTH):
            slot = _Slot()
            static_pos, static_sig = {}, {}
            slot.jobs = []
            for jb in jobs:
                pk, sk = engine._key(jb.path_key, jb.pos), engine._key(jb.signal_key, jb.s)
                if pk not in static_pos:
                    static_pos[pk] = torch.empty(_dims(jb.pos), dtype=torch.float64, device=self.dev)
                if sk not in static_sig:
                    static_sig[sk] = torch.empty(int(np.prod(_dims(jb.s))), dtype=dt, device=self.dev)
                mic = torch.empty(_dims(jb.mic), dtype=torch.float64, device=self.dev)
                slot.jobs.append(replace(jb, pos=static_pos[pk], s=static_sig[sk], mic=mic,
                                         path_key=("plan", pk), signal_key=("plan", sk)))
            slot.paths = slot.bbox = None
            self.slots.append(slot)
        weakref.finalize(self, release_pinned, [sl.tag for sl in self.slots])
        self.k = 0
        self.captures = 0
        self.misses = 0  # speculative replays redone after a decision / capacity change
        self.kernel_ms = {}  # run index -> synthesis kernel time of that replay

    # ------------------------------------------------------------------
    def _load(self, slot, jobs):
        """Copy the inputs of `jobs` into the slot's static tensors (on the
        current stream)."""
        seen = set()
        direct, rest = [], []
        for jb, sj in zip(jobs, slot.jobs):
            for src, dst in ((jb.pos, sj.pos), (jb.s, sj.s), (jb.mic, sj.mic)):
                if id(dst) in seen:
                    continue
                seen.add(id(dst))
                if isinstance(src, torch.Tensor):
                    dst.copy_(src.reshape(dst.shape), non_blocking=True)
                elif isinstance(src, np.ndarray) and src.flags.c_contiguous and \
                        src.dtype == _NP_DTYPE[dst.dtype] and src.size == dst.numel():
                    direct.append((dst, src))
                else:
                    rest.append((dst, src))
        # page-locked caller arrays: one batched libmvb call issues every DMA
        # (a batch of 256 scenes has 768 inputs); the others are staged
        if direct:
            issued = copy_batch([(d.data_ptr(), a.ctypes.data, a.nbytes) for d, a in direct],
                                torch.cuda.current_stream(self.dev).cuda_stream,
                                require_pinned=True)
            rest += [pair for pair, ok in zip(direct, issued) if not ok]
        for dst, src in rest:
            a = np.asarray(src).reshape(dst.shape[0], -1) if dst.dim() > 1 else \
                np.asarray(src).reshape(-1)
            _STAGER.upload([(0, a)], dst)

    def _stage(self, slot, ready):
        """Stage the slot's static inputs into its static paths buffer on the
        current stream (after event `ready`, if given) and wait for the
        readbacks (eager: first run of a slot, a miss)."""
        if ready is not None:
            torch.cuda.current_stream(self.dev).wait_event(ready)
        if slot.paths is None:  # first staging allocates the slot's paths / box buffers
            geom = engine.Geometry(slot.jobs, device=self.dev, defer=True, readback_tag=slot.tag)
            slot.paths, slot.bbox = geom.paths, geom.bbox
            return geom
        return engine.Geometry(slot.jobs, device=self.dev, paths=slot.paths, defer=True,
                               bbox=slot.bbox, readback_tag=slot.tag)

    SLACK = 0.1  # output capacity headroom of a capture (fraction of the length bound)

    def _prepare(self, slot, geom, fork=None):
        """Geometry and the render's first half (see engine.PreparedRender);
        `fork` (capture only): four streams for the parallel branches -- delay
        sort, branch records, further factors' interval records, exact
        maxima -- all joined before the geometry graph ends."""
        geom.length_slack = self.SLACK
        geom.finish(fork=None if fork is None else fork[3])  # exact maxima: own branch
        prep = engine.prepare_render(geom, [sj.s for sj in slot.jobs], self.f,
                                     precision=self.precision,
                                     signal_keys=[engine._key(sj.signal_key, sj.s)
                                                  for sj in slot.jobs],
                                     fork=None if fork is None else fork[:3])
        geom.join()  # every branch ends inside the geometry graph
        return prep

    def _collect(self, slot):
        """Record the synthesis time of the slot's finished replay."""
        if slot.run_index is not None and slot.timing:
            a, b = slot.timing[-1]
            self.kernel_ms[slot.run_index] = a.elapsed_time(b)
            slot.run_index = None

    def settle(self) -> None:
        """Validate every pending speculative replay (run())."""
        for slot in self.slots:
            if slot.pending is not None:
                slot.pending._settle()

    def flush_timing(self) -> dict:
        """Wait for every slot and collect the pending kernel timings."""
        self.settle()
        for slot in self.slots:
            if slot.done is not None:
                slot.done.synchronize()
            self._collect(slot)
        return self.kernel_ms

    def join(self) -> None:
        """Order the current stream after every pending run (no host wait
        beyond the validation of pending speculative replays)."""
        self.settle()
        cur = torch.cuda.current_stream(self.dev)
        for slot in self.slots:
            if slot.done is not None:
                cur.wait_event(slot.done)

    def _capture(self, slot, geom):
        """Dry run (populates caches, sizes the static uploads), re-stage,
        capture the geometry graph on the geometry stream and the synthesis
        graph on the synthesis stream; both are then replayed for this run."""
        with UploadMeter() as meter:
            prep = self._prepare(slot, geom)
            if self.dmax_hook is not None:
                self.dmax_hook(geom.dmax_dev)
            prep.launch()
        torch.cuda.synchronize(self.dev)
        geom = self._stage(slot, None)
        uploads = StaticUploads(int(meter.used * 1.25) + (64 << 10))
        g_geo, g_syn = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        slot.timing = []
        launches0 = _lib.launch_count()
        fork = self.fork_streams if os.environ.get("MVB_PLAN_FORK", "1") != "0" else None
        with uploads, torch.cuda.graph(g_geo, stream=self.geo_stream):
            prep = self._prepare(slot, geom, fork=fork)
        with uploads, torch.cuda.graph(g_syn, stream=self.syn_stream):
            res = prep.launch(slot.timing)
        slot.graphs = [g_geo, g_syn]
        slot.geom = geom  # owns the cached tables the graphs read
        slot.dmax = geom.dmax_dev
        slot.graph_launches = _lib.launch_count() - launches0  # kernels replayed per run
        slot.graph, slot.result, slot.uploads = g_geo, res, uploads
        slot.decision = self._decision(geom)
        slot.capacity = np.asarray([geom.length_bound(j) for j in range(len(slot.jobs))])  # slacked
        self._capture_staging(slot)
        self.captures += 1

    def _decision(self, geom) -> tuple:
        """Data-dependent choices a captured slot is valid for: the low-pass
        decision and whether the fp32 fast path's envelope holds (else the
        capture renders on the exact engine, engine.prepare_render)."""
        ok = self.precision == "fp64" or geom.fast_path_ok
        if not ok and self.shard is not None and int(self.shard[1]) > 1:
            raise ValueError("delay excursions beyond the fp32 envelope: image shards need the "
                             "fp32 fast path (render replicas on the exact engine instead)")
        return (geom.lowpass_decision(), ok)

    def _replay(self, slot, after):
        """Replay the slot's graphs on the plan streams after event `after`."""
        geo, syn = self.geo_stream, self.syn_stream
        geo.wait_event(after)
        with torch.cuda.stream(geo):
            slot.graphs[0].replay()
            if self.dmax_hook is not None:
                self.dmax_hook(slot.dmax)
            geo_done = torch.cuda.Event()
            geo_done.record()
        syn.wait_event(geo_done)
        with torch.cuda.stream(syn):
            slot.graphs[1].replay()
            slot.done = torch.cuda.Event()
            slot.done.record()

    def reduce(self, res: engine.RenderResult, group=None, root: int = 0) -> engine.RenderResult:
        """Image shards: sum the ranks' partial outputs of `res` (this plan's
        latest run) into `root` (parallel.reduce_to_root), on the synthesis
        stream after the render.  The slot's completion event is re-recorded
        after the collective, so `res.wait()` / `host()` / `join()` and the
        slot's next reuse (its geometry graph zero-fills the same static
        output) are all ordered after the reduction, not only the render."""
        from . import parallel
        slot = self.slots[(self.k - 1) % self.DEPTH]
        if res.done is not slot.done:
            raise ValueError("reduce() takes the result of the plan's latest run")
        with torch.cuda.stream(self.syn_stream):
            self.syn_stream.wait_event(slot.done)
            parallel.reduce_to_root(res.out, group=group, root=root)
            ev = torch.cuda.Event()
            ev.record()
        slot.done = res.done = ev
        return res

    def run(self, jobs) -> engine.RenderResult:
        """Render `jobs` (same structure as the plan's template)."""
        if self.shard is not None and int(self.shard[1]) > 1:
            from . import parallel
            rank, world = int(self.shard[0]), int(self.shard[1])
            jobs = parallel.shard_jobs(jobs, rank, world, parallel.shard_kind(self.shard))
        if structure_key(jobs, self.f, self.precision) != self.key:
            raise ValueError("jobs do not match the plan's structure")
        slot = self.slots[self.k % self.DEPTH]
        self.k += 1
        if slot.pending is not None:
            slot.pending._settle()  # the slot's previous run (two runs ago)
        if slot.done is not None:
            slot.done.synchronize()  # its previous replay finished
        self._collect(slot)
        cur = torch.cuda.current_stream(self.dev)
        entry = torch.cuda.Event()
        entry.record(cur)  # inputs the caller wrote on its stream
        side = side_stream(self.dev)
        spec = slot.graph is not None
        with torch.cuda.stream(side):
            side.wait_event(entry)
            self._load(slot, jobs)
            ready = torch.cuda.Event()
            ready.record()
            if spec:  # captured staging, part 1: paths and boxes
                slot.stage[0].replay()
                paths_ev = torch.cuda.Event()
                paths_ev.record()
        slot.run_index = self.k - 1
        if not spec:  # first run of the slot: stage eagerly, capture, replay
            self._redo(slot, self._stage(slot, ready), side)
            return self._result(slot)
        # speculative replay: a captured slot is valid while the low-pass
        # decision, the fp32 envelope and the output capacities hold.  The
        # graphs replay as soon as the paths are on the device; the staging
        # readbacks (boxes, bandwidth indices: captured part 2) are checked
        # later -- on first use of the result, at the slot's next run, or
        # join() / flush_timing() -- and the run is re-captured and replayed
        # only if they changed.  Image shards check at once (their ranks
        # must take the same branch before the next collective).
        self._replay(slot, paths_ev)
        with torch.cuda.stream(side):
            if slot.stage[1] is not None:
                slot.stage[1].replay()
            staged = torch.cuda.Event()
            staged.record()
        res = self._result(slot, lambda res: self._check(slot, staged, res))
        slot.pending = res
        if self.shard is not None and int(self.shard[1]) > 1:
            res._settle()
        return res

    def _result(self, slot, validate=None) -> engine.RenderResult:
        r = slot.result
        return engine.RenderResult(r._out, r._offsets, r._capacity, r._n_images,
                                   slot.stage_launches + slot.graph_launches, *r._devs,
                                   done=slot.done, stream=self.syn_stream, validate=validate)

    def _valid(self, slot, geom) -> bool:
        """The staging readbacks of `geom` (collected) fit the slot's capture."""
        bound = np.asarray([geom.length_bound(j) for j in range(len(slot.jobs))])
        return self._decision(geom) == slot.decision and not np.any(bound > slot.capacity)

    def _redo(self, slot, geom, side) -> None:
        """(Re-)capture the slot for the staged run (`geom`) and replay it."""
        cur = torch.cuda.current_stream(self.dev)
        cur.wait_stream(side)
        self._capture(slot, geom)
        staged_ev = torch.cuda.Event()
        staged_ev.record(cur)  # _stage ordered the current stream after the staging
        self._replay(slot, staged_ev)

    def _check(self, slot, staged, res) -> None:
        """Deferred validation of a speculative replay (RenderResult._settle):
        wait for the replayed staging, re-read its readbacks; on a changed
        decision / capacity the run is staged again eagerly from the slot's
        static inputs (still this run's: the slot's next run validates
        first), re-captured and replayed, and `res` takes the new fields."""
        if slot.pending is res:
            slot.pending = None
        staged.synchronize()
        geom = slot.stage_geom.recollect(slot.stage_pending)
        if not self._valid(slot, geom):
            self.misses += 1
            slot.done.synchronize()  # the speculative replay
            self._redo(slot, self._stage(slot, None), side_stream(self.dev))
            res._redo(slot.result, slot.done)

    def _capture_staging(self, slot) -> None:
        """Capture the slot's staging -- path copies into the paths buffer,
        bounding boxes, bandwidth indices and their readbacks into the
        slot's pinned buffers -- as two graphs on the side stream: part 1
        ends after the boxes (the geometry graph needs only paths and
        boxes), part 2 measures the bandwidths.  A run replays both instead
        of re-issuing the staging's host calls (c1 / c2 runs were host-bound
        at ~0.6 ms by them)."""
        side = side_stream(self.dev)
        torch.cuda.synchronize(self.dev)
        g = [torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()]
        live = [g[0]]

        decimated = any(int(N) > 1 for jb in slot.jobs for _, N in jb.tiers)

        def split(_ev):  # the boxes are read back: part 2 (bandwidths) starts
            live.pop().capture_end()
            if decimated:  # (full-rate plans measure no bandwidth)
                g[1].capture_begin(pool=g[0].pool())
                live.append(g[1])

        uploads = StaticUploads(64 * len(slot.jobs) + (64 << 10))
        launches0 = _lib.launch_count()
        with uploads, torch.cuda.stream(side):
            g[0].capture_begin()
            try:
                geom = engine.Geometry(slot.jobs, device=self.dev, paths=slot.paths,
                                       bbox=slot.bbox, defer=True, wait=False, on_paths=split,
                                       readback_tag=slot.tag)
            finally:
                while live:
                    live.pop().capture_end()
        if geom.paths.data_ptr() != slot.paths.data_ptr():
            raise _lib.MvbError("render plan: staging captured into another paths buffer")
        slot.stage, slot.stage_uploads = (g if decimated else [g[0], None]), uploads
        slot.stage_geom, slot.stage_pending = geom, geom._pending
        slot.stage_launches = _lib.launch_count() - launches0
