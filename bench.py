#!/usr/bin/env python
"""Benchmark of the moving-source synthesis hot path (BASELINE.json metric:
image x output-sample updates per second; real-time factor alongside).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
    python bench.py --impl reference ...   # CPU oracle port on the host cores
    torchrun --nproc-per-node N bench.py --gpus N ...

A step is one complete render of the workload from device-resident inputs:
GPU image enumeration, decimation decisions, coarse tracks, exact out_len,
branch records, interval polynomials, delay sort and the fused synthesis
(+ the NCCL reduce of image shards for N > 1).  `value` = all updates
processed by all ranks / max-over-ranks device time.  `e2e` = the same
metric through the public API `render(s, traj, room, mic, f, cfg)` with host
numpy buffers (H2D of s/path/mic and D2H of the output inside the timing).
Default workload: c3 (20x15x8 m hall, order 20, 10 s at 48 kHz, 11521
images, 64-tap Hann-sinc) -- the largest single-scene config.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-plan", action="store_true",
                    help="render each step directly instead of replaying a RenderPlan graph")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU work of the cpu_baseline / reference sample")
    ap.add_argument("--no-l0", action="store_true",
                    help="skip the reference-code (baseline/_ref, numba) CPU samples")
    ap.add_argument("--no-per-config", action="store_true",
                    help="headline config only (no per_config block)")
    ap.add_argument("--per-config-steps", type=int, default=10,
                    help="timed steps of each per_config entry (capped by --steps)")
    ap.add_argument("--profile", action="store_true",
                    help="ncu mode: warmup+steps renders only, no probes/e2e/cpu")
    return ap.parse_args()


METRIC = "image x output-sample updates/sec"


def workload_note(name):
    from paper_2508_03065_b200 import workloads
    w = workloads.WORKLOADS[name]
    return w


# ----------------------------------------------------------------------------
# clocks


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms from before
    the warm-up (nvidia-smi's start-up must not overlap the timed steps);
    each sample is timestamped and the summary keeps the samples taken
    during the timed window (widened to the nearest samples when the window
    is shorter than the sampling period)."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.file, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        """Stop sampling and parse the samples (timestamp, sm, max, reasons)."""
        import datetime
        self.rows = []
        if self.proc is None:
            return
        time.sleep(0.15)
        self.proc.terminate()
        self.proc.wait()
        self.file.flush()
        self.file.seek(0)
        for line in self.file.read().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                self.rows.append((ts, float(f[2]), float(f[3]), f[6:10]))
            except ValueError:
                continue
        os.unlink(self.file.name)

    def window(self, t0=None, t1=None):
        """Summary of the samples within [t0, t1] (host wall-clock seconds);
        call after stop()."""
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = self.rows
        sel = rows
        if t0 is not None and rows:
            inside = [r for r in rows if t0 <= r[0] <= t1]
            if not inside:  # window shorter than the period: nearest samples around it
                before = [r for r in rows if r[0] < t0][-1:]
                after = [r for r in rows if r[0] > t1][:1]
                inside = before + after
            sel = inside
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in sel:
            for n, v in zip(names, r[3]):
                if v.lower() in ("active", "1"):
                    reasons.add(n)
        sm = [r[1] for r in sel]
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": sel[-1][2] if sel else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------
# workload


def parallel_mode(name):
    from paper_2508_03065_b200 import parallel
    return parallel.shard_mode(name, 2)


def build_workload(name, rank, world):
    """Scenes, the jobs this rank renders, and the sharding mode."""
    from paper_2508_03065_b200 import parallel, workloads
    from paper_2508_03065_b200.room import image_count
    scenes = workloads.make_scenes(name)
    mode = parallel.shard_mode(name, world)
    if mode == "single":
        return scenes, scenes, None, "single"
    if mode == "images":
        return scenes, scenes, (rank, world), f"image-shard x{world} + NCCL reduce"
    if mode == "scenes":
        # LPT by update count ~ images x (T + max delay of the room's reach)
        cost = [image_count(sc.max_order) * len(sc.mics) *
                (sc.T + sc.max_order * float(np.max(sc.dims)) * sc.rate / 343.0) for sc in scenes]
        mine = [scenes[i] for i in parallel.lpt_assign(cost, world)[rank]]
        return scenes, mine, None, f"scene-shard x{world} LPT (no collective)"
    if mode == "channels":
        import dataclasses
        mine = [dataclasses.replace(sc, mics=[sc.mics[i] for i in
                                              parallel.channel_shard(len(sc.mics), rank, world)])
                for sc in scenes]
        return scenes, [sc for sc in mine if sc.mics], None, \
            f"channel-shard x{world} (no collective)"
    return scenes, scenes, None, f"replicas x{world}"


def device_jobs(scenes, dev):
    """engine.Job list with every input already resident on the device."""
    import torch
    from paper_2508_03065_b200 import engine
    jobs = []
    for q, sc in enumerate(scenes):
        s = torch.from_numpy(np.ascontiguousarray(sc.s)).to(dev)
        pos = torch.from_numpy(np.ascontiguousarray(sc.pos)).to(dev)
        for ch, m in enumerate(sc.mics):
            mic = torch.from_numpy(np.ascontiguousarray(m, dtype=np.float64)).to(dev)
            jobs.append(engine.Job(s=s, pos=pos, mic=mic, dims=sc.dims, walls=sc.walls,
                                   max_order=sc.max_order, tiers=sc.tiers, rate=sc.rate,
                                   signal_key=("s", q), path_key=("p", q)))
    return jobs


# ----------------------------------------------------------------------------
# CPU oracle sample


_ORACLE_CACHE = {}


def cpu_sample(name, target_s, nthreads):
    """Time the oracle port on a bounded slice of the workload: all images of
    the first scene/channel, output samples [n0, n0 + W) with W calibrated to
    ~target_s seconds.  Returns (updates/s, description, threads)."""
    from oracle import oracle as orc
    from paper_2508_03065_b200 import hann_sinc, workloads
    if name not in _ORACLE_CACHE:
        sc = workloads.make_scenes(name, n_scenes=1 if name == "c4" else None,
                                   n_channels=1 if name == "c5" else None)[0]
        f = hann_sinc(sc.fd_taps, 14)
        _ORACLE_CACHE[name] = (sc, orc.OracleScene(sc.s, sc.pos, sc.mics[0], sc.dims, sc.walls,
                                                   sc.max_order, sc.tiers, f.branches, sc.rate))
    sc, o = _ORACLE_CACHE[name]
    S = len(o.images)
    n0 = sc.T // 2
    w = 256
    for _ in range(2):  # calibrate the slice to ~target_s of CPU work
        t = time.perf_counter()
        o.render_window(n0, n0 + w, nthreads)
        dt = max(time.perf_counter() - t, 1e-6)
        w = int(max(256, min(sc.T // 2, w * min(target_s / dt, 64.0))))
    t = time.perf_counter()
    o.render_window(n0, n0 + w, nthreads)
    dt = time.perf_counter() - t
    desc = (f"{name} scene 0 ch 0: all {S} images x output samples [{n0}, {n0 + w}) "
            f"(oracle C port, Farrow M=14 Hann-sinc L={sc.fd_taps}, per-sample 65-tap tracks)")
    return S * w / dt, desc, nthreads, S * w, dt


def l0_samples(name, nthreads, target_s=6.0):
    """The reference's OWN code (baseline/_ref, numba asserted; oracle/l0.py):
    kernel-only block-parallel accumulate on the bench workload (all images,
    a mid-signal window, tau/amp from the oracle's bit-identical tracks),
    the same with the reference's default filter design(3, 8, 0.8), and the
    whole L0 render (tracks + synthesize) of a 1 s c2 scene."""
    try:
        from oracle import l0
        l0.load()
    except Exception as e:  # noqa: BLE001 -- reported, not fatal
        return {"unavailable": f"{type(e).__name__}: {e}"}
    from oracle import oracle as orc
    from paper_2508_03065_b200 import hann_sinc, workloads
    cpu_sample(name, 0.2, nthreads)  # builds the cached oracle scene
    sc, o = _ORACLE_CACHE[name]
    out = {"kind": "reference (moverb from baseline/_ref, numba)", "threads": nthreads}
    # the reference's default filter design(3, 8, 0.8), exported from the reference itself
    g = np.load(os.path.join(ROOT, "tests", "golden", "kernels.npz"))
    for key, branches in (("kernel", o.branches), ("kernel_design_3_8_0.8", g["design_3_8_08"])):
        # window sized to ~target_s / 2 of work from a 512-sample probe, capped
        # so the (S, w) fp64 tau / amp arrays stay within ~3 GB
        ks = l0.KernelSample(o, branches, sc.T // 2, 512, nthreads)
        _, dt = ks.run(nthreads)
        cap = max(512, int(3e9 / (24 * ks.S)))
        w = int(min(cap, sc.T // 2, 512 * target_s / 2 / max(dt, 1e-4)))
        ks = l0.KernelSample(o, branches, sc.T // 2, w, nthreads)
        _, dt = ks.run(nthreads)
        out[key] = {"value": ks.S * w / dt, "unit": "updates/s", "seconds": dt,
                    "sample": f"{name}: all {ks.S} images x output samples [{sc.T // 2}, "
                              f"{sc.T // 2 + w}), _accumulate_numba in 32-image blocks on "
                              f"{nthreads} threads + pairwise merge ({branches.shape[0]} branches, "
                              f"{branches.shape[1]} taps)"}
    sc2 = workloads.make_scenes("c2", duration=1.0)[0]
    r = l0.render_sample(sc2, hann_sinc(sc2.fd_taps, 14).branches, nthreads)
    out["render"] = {"value": r["value"], "unit": "updates/s", "tracks_s": r["tracks_s"],
                     "synthesize_s": r["synthesize_s"], "synthesize_value": r["synthesize_value"],
                     "sample": "c2 scene, 1 s of dry signal, whole render: per-tier "
                               "low/high_order_distances(decimate) + merge_streams + "
                               f"synthesize(workers={nthreads}) (SURVEY 8c L0 composition)"}
    return out


# ----------------------------------------------------------------------------


def measured_peaks(dev):
    """FP32 FFMA / FP64 DFMA TFLOP/s and L1-hit load GB/s on this GPU (CUDA
    events, best of 3)."""
    import torch
    from paper_2508_03065_b200 import _lib
    from paper_2508_03065_b200._dev import ptr, stream_handle
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    sink = torch.zeros(sms * 64, dtype=torch.float64, device=dev)
    buf = torch.randn(64 * 16 * 1024 // 4, dtype=torch.float32, device=dev)
    st = stream_handle(dev)
    out = {}
    for name, blocks, iters, work in (
            ("ffma", sms * 8, 4000, lambda b, it: b * 256 * it * 128 * 2),
            ("dfma", sms * 8, 500, lambda b, it: b * 256 * it * 128 * 2),
            ("l1", sms * 8, 4000, lambda b, it: b * 256 * it * 4 * 16)):
        best = 0.0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if name == "ffma":
                _lib.call("mvb_peak_ffma", blocks, iters, ptr(sink), st)
            elif name == "dfma":
                _lib.call("mvb_peak_dfma", blocks, iters, ptr(sink), st)
            else:
                _lib.call("mvb_peak_l1", blocks, iters, ptr(buf), ptr(sink), st)
            e1.record()
            torch.cuda.synchronize()
            best = max(best, work(blocks, iters) / (e0.elapsed_time(e1) * 1e-3))
        out[name] = best
    return {"ffma_tf": out["ffma"] / 1e12, "dfma_tf": out["dfma"] / 1e12, "l1_gbs": out["l1"] / 1e9}


def load_traffic(name):
    """DRAM bytes per synthesis launch from the committed ncu --set full
    summary of this config (profiles/ncu_synth_<name>.json), or None."""
    p = os.path.join(ROOT, "profiles", f"ncu_synth_{name}.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except (OSError, ValueError):
            return None
    return None


class Ctx:
    """Per-process distributed plumbing of a bench run."""

    def __init__(self):
        import torch
        import torch.distributed as dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        local = int(os.environ.get("LOCAL_RANK", "0"))
        # NCCL over NVLink; MVB_DIST_BACKEND=gloo rehearses the multi-rank
        # path on fewer GPUs than ranks (collectives staged through host
        # memory, no kernel waits on another rank)
        self.backend = os.environ.get("MVB_DIST_BACKEND", "nccl")
        if self.backend != "nccl":
            local %= torch.cuda.device_count()
        self.local = local
        torch.cuda.set_device(local)
        self.dev = torch.device("cuda", local)
        if self.world > 1:
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=self.dev)
            else:
                dist.init_process_group(self.backend)

    def barrier(self):
        import torch.distributed as dist
        if self.world > 1:
            if self.backend == "nccl":
                dist.barrier(device_ids=[self.local])
            else:
                dist.barrier()

    def allreduce(self, t, op):
        """Timing / count reductions (outside the timed brackets)."""
        import torch.distributed as dist
        if self.world == 1:
            return t
        if self.backend == "nccl":
            dist.all_reduce(t, op=op)
            return t
        h = t.cpu()
        dist.all_reduce(h, op=op)
        return h.to(t.device)


def measure(ctx, name, steps, warmup, peaks, args, precision=None, with_e2e=True):
    """One config: K timed render steps (value, kernel time, roofline) and
    the end-to-end public-API number.  Returns (line dict, clock window)."""
    import gc

    import torch
    import torch.distributed as dist
    from paper_2508_03065_b200 import (Room, SynthesisConfig, Trajectory, hann_sinc, parallel,
                                       render, workloads)
    from paper_2508_03065_b200.synth import render_jobs, release_plans

    world, rank, dev = ctx.world, ctx.rank, ctx.dev
    w = workloads.WORKLOADS[name]
    scenes, mine, shard, mode = build_workload(name, rank, world)
    f = hann_sinc(w.fd_taps, 14)
    jobs = device_jobs(mine, dev)
    timing = []
    if precision is None:
        precision = "fp64" if w.dtype == "f64" else "fp32"  # c1 is an fp64 config
    if precision == "fp64" and shard is not None:  # the exact engine runs replicas only
        shard, mode = None, f"replicas x{world} (exact engine)"
        scenes, mine = scenes, scenes

    # the device inputs are final from here on: planning of step k+1 may
    # overlap step k's kernels (render_jobs inputs_ready)
    inputs_ready = torch.cuda.Event()
    inputs_ready.record()

    # repeated renders of one structure replay captured CUDA graphs
    # (plan.RenderPlan: inputs re-staged and every kernel re-run each step;
    # image shards all-reduce the track maxima eagerly between two graphs)
    plan = None
    if not args.no_plan:
        from paper_2508_03065_b200.plan import RenderPlan
        plan = RenderPlan(jobs, f, precision=precision, shard=shard)

    def step(record=False):
        if plan is not None:
            res = plan.run(jobs)
            if shard is not None:  # on the plan's synthesis stream, after the render
                plan.reduce(res)
            return res
        tl = timing if record else None
        res = render_jobs(jobs, f, precision=precision, shard=shard, timing=tl,
                          inputs_ready=inputs_ready)
        if shard is not None:
            parallel.reduce_to_root(res.out)
        return res

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(warmup):
        res = step()
    torch.cuda.synchronize()
    ctx.barrier()
    if args.profile:
        for _ in range(steps):
            step()
        torch.cuda.synchronize()
        return None, None
    launches = 0
    timing.clear()
    # K steps back to back, bracketed once by barrier + synchronize; an L2
    # flush (256 MiB write) is queued before every step and stays inside the
    # timed region (conservative)
    torch.cuda.synchronize()
    ctx.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    first_run = plan.k if plan is not None else 0
    wall0 = time.time()
    e0.record()
    results = []
    for k in range(steps):
        flush.fill_(float(k))
        res = step(record=True)
        results.append(res)  # lengths / update counts are read after the bracket
        launches += res.launches
    if plan is not None:
        plan.join()  # the plan renders on its own streams: order e1 after them
    e1.record()
    torch.cuda.synchronize()
    ctx.barrier()
    wall1 = time.time()
    total_ms = e0.elapsed_time(e1)
    updates = sum(r.updates for r in results)
    if plan is not None:  # synthesis time of every timed replay
        km = plan.flush_timing()
        kern_ms = [km[i] for i in range(first_run, first_run + steps) if i in km]
    else:
        kern_ms = [a.elapsed_time(b) for a, b in timing]
    rendered = sorted({r.precision for r in results})
    t = torch.tensor([total_ms, float(updates), sum(kern_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        tmax = ctx.allreduce(t.clone(), dist.ReduceOp.MAX)
        tsum = ctx.allreduce(t.clone(), dist.ReduceOp.SUM)
        # every rank's updates count: image shards and scene shards split the
        # work, replicas each do all of it (value = N x one replica)
        total_ms_all, updates_all = float(tmax[0]), float(tsum[1])
    else:
        total_ms_all, updates_all = total_ms, float(updates)
    value = updates_all / (total_ms_all * 1e-3)
    ms_step = total_ms_all / steps
    audio_s = sum(sc.T / sc.rate * len(sc.mics) for sc in scenes)
    if mode.startswith("replicas") and world > 1:
        audio_s *= world
    rtf = audio_s * steps / (total_ms_all * 1e-3)

    # ---- end to end through the public API with host buffers ----------------
    # the value loop's plan (its two graph pools) is released first: batch
    # configs hold tens of GB of interval records per slot (c4: 32 GB)
    _ = res.lengths, res.updates  # what the roofline reads later
    results.clear()
    used_plan = plan is not None
    plan = None
    gc.collect()
    torch.cuda.empty_cache()
    def plan_e2e():
        # batch / multi-rank: the public API for repeated renders of one
        # structure (RenderPlan) fed from host arrays in pinned memory --
        # H2D of every signal / path / receiver, the render (+ reduce to
        # rank 0) and the D2H of the output inside every timed step
        from dataclasses import replace as _replace

        from paper_2508_03065_b200.plan import RenderPlan
        from paper_2508_03065_b200.synth import scene_jobs

        def pinned(a):
            a = np.ascontiguousarray(a)
            t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
            out = t.numpy()
            np.copyto(out, a)
            return out

        host_jobs = [_replace(jb, s=pinned(jb.s), pos=pinned(jb.pos), mic=pinned(jb.mic))
                     for jb in scene_jobs(mine)]
        # shared paths / signals stay shared (one pinned copy per key)
        by_key = {}
        for j, jb in enumerate(host_jobs):
            pk, sk = jb.path_key, jb.signal_key
            if pk is not None:
                host_jobs[j] = _replace(host_jobs[j], pos=by_key.setdefault(("p", pk), jb.pos))
            if sk is not None:
                host_jobs[j] = _replace(host_jobs[j], s=by_key.setdefault(("s", sk), jb.s))
        plan_e = RenderPlan(host_jobs, f, precision=precision, shard=shard)
        tt = 0.0
        upd = 0
        h2d = sum(sc.s.nbytes + sc.pos.nbytes + sum(np.asarray(m).nbytes for m in sc.mics)
                  for sc in mine)
        d2h = 0
        for _ in range(max(4, warmup)):  # captures both slots, then replays
            r = plan_e.run(host_jobs)
            if shard is not None:
                plan_e.reduce(r)
            if shard is None or rank == 0:
                r.host()
        # (a) one render per timed step, synchronous (host staging, H2D,
        # render, D2H back to back)
        for _ in range(steps):
            torch.cuda.synchronize()
            ctx.barrier()
            t0 = time.perf_counter()
            r = plan_e.run(host_jobs)
            if shard is not None:
                plan_e.reduce(r)
            out_h = r.host() if (shard is None or rank == 0) else None
            torch.cuda.synchronize()
            ctx.barrier()
            tt += time.perf_counter() - t0
            upd += r.updates
            d2h = 0 if out_h is None else out_h.nbytes
        # (b) pipelined: run(k + 1) is issued before host(k), so step k+1's
        # host staging and H2D overlap step k's device work; every step
        # still copies its inputs in and its output out inside the bracket
        torch.cuda.synchronize()
        ctx.barrier()
        t0 = time.perf_counter()
        prev, upd_p = None, 0

        def collect(res_k):
            # the step's D2H (root) and its update count, before the
            # slot is reused two runs later
            if shard is None or rank == 0:
                res_k.host()
            return res_k.updates

        for _ in range(steps):
            r = plan_e.run(host_jobs)
            if shard is not None:
                plan_e.reduce(r)
            if prev is not None:
                upd_p += collect(prev)
            prev = r
        upd_p += collect(prev)
        plan_e.join()
        torch.cuda.synchronize()
        ctx.barrier()
        tp = time.perf_counter() - t0
        del plan_e, r, prev
        gc.collect()
        torch.cuda.empty_cache()
        tt_t = torch.tensor([tt, float(upd), tp, float(upd_p)], dtype=torch.float64, device=dev)
        if world > 1:
            tmax = ctx.allreduce(tt_t.clone(), dist.ReduceOp.MAX)
            tsum = ctx.allreduce(tt_t.clone(), dist.ReduceOp.SUM)
            tt, upd, tp, upd_p = float(tmax[0]), float(tsum[1]), float(tmax[2]), float(tsum[3])
        e2e_p = {"value": upd_p / tp, "unit": "updates/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h),
               "api": "paper_2508_03065_b200.RenderPlan.run (repeated renders of one "
                      "structure) + RenderResult.host(), pipelined: run(k+1) is issued "
                      "before host(k)",
               "sync_value": upd / tt,
               "sync": "the same with run + host back to back per step (no overlap)",
               "inputs": "pinned host memory, copied to the device inside every timed step"}
        return e2e_p

    e2e = None
    if with_e2e and not args.no_e2e:
        if world == 1 and len(scenes) == 1 and len(scenes[0].mics) == 1:
            sc = scenes[0]
            room = Room(dims=sc.dims, wall_reflection=sc.walls)
            traj = Trajectory(rate=sc.rate, positions=sc.pos)
            cfg = SynthesisConfig(audio_rate=sc.rate, max_order=sc.max_order, tiers=sc.tiers,
                                  precision=precision)
            # inputs in pinned host memory (the e2e contract): the dry signal in a
            # page-locked buffer, the path in the Trajectory's own pinned copy
            sx = torch.empty(sc.s.shape, dtype=torch.from_numpy(np.asarray(sc.s)).dtype,
                             pin_memory=True).numpy()
            np.copyto(sx, sc.s)
            # warm: render() caches a plan on a repeat, captures one slot per call
            # and replays speculatively from the next call on (one-time costs)
            for _ in range(max(5, warmup)):
                y = render(sx, traj, room, sc.mics[0], f, cfg)
            tt = 0.0
            calls = []
            for _ in range(steps):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                y = render(sx, traj, room, sc.mics[0], f, cfg)
                torch.cuda.synchronize()
                calls.append(time.perf_counter() - t0)
                tt += calls[-1]
            release_plans()
            e2e_upd = res.updates * steps
            h2d = sx.nbytes + traj.positions.nbytes + np.asarray(sc.mics[0]).nbytes
            e2e = {"value": e2e_upd / tt, "unit": "updates/s", "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": int(y.nbytes), "api": "paper_2508_03065_b200.render",
                   "inputs": "pinned host memory (signal buffer; Trajectory positions are held "
                             "page-locked), copied to the device inside every timed call; "
                             "output returned as float64 numpy (8 B per sample)",
                   "ms_per_call": [round(c * 1e3, 3) for c in calls]}
            # the same render through RenderPlan from the same host buffers,
            # pipelined (repeated renders of one structure: dataset generation)
            pe = plan_e2e()
            e2e["plan_pipelined"] = {k: pe[k] for k in ("value", "sync_value", "api")}
        else:
            e2e = plan_e2e()

    # ---- roofline of the dominant kernel (fused synthesis) --------------------
    kern_avg_ms = float(np.mean(kern_ms)) if kern_ms else float("nan")
    # the metric counts S x out_len updates per job (the reference's loop);
    # only S x (len(s) + L - 1) of them can be non-zero (an image's delayed
    # copy of the signal is that long), and the fast synthesis skips (image,
    # tile) pairs whose gathers read only zero pads -- its roofline counts the
    # non-zero updates one launch must compute; the exact engine evaluates
    # every (image, sample) pair like the reference
    metric_upd = res.updates  # one synthesis launch per step
    exact = res.precision == "fp64"
    upd_per_launch = int(sum(int(res.n_images[j]) * (int(res.lengths[j]) if exact else
                                                     min(int(res.lengths[j]),
                                                         int(jobs[j].s.numel()) + w.fd_taps - 1))
                             for j in range(len(res.lengths))))
    flops = upd_per_launch * w.fd_taps * 2.0  # taps x FMA (north_star roofline)
    achieved = flops / (kern_avg_ms * 1e-3) / 1e12
    traffic = None if exact else load_traffic(name)
    # the other leg of the north_star roofline: algorithmic HBM bytes of a
    # render (dry signal + trajectory in, output out) at the
    # measured HBM bandwidth -- the slower leg (FMA) is the bound
    out_bytes = 8 if exact else 4
    alg_bytes = sum(sc.s.itemsize * sc.T + 24 * sc.T * (1 + (np.ndim(sc.mics[0]) > 1) * len(sc.mics))
                    for sc in mine) + out_bytes * int(np.sum(res.lengths))
    hbm_gbs = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 7700.0
    hbm_leg = {"algorithmic_bytes": int(alg_bytes),
               "achieved_gbs": alg_bytes / (kern_avg_ms * 1e-3) / 1e9, "peak_gbs": hbm_gbs,
               "frac": alg_bytes / (kern_avg_ms * 1e-3) / 1e9 / hbm_gbs,
               "measured_dram_gbs": None if traffic is None else
               traffic.get("dram_bytes_per_launch") / (kern_avg_ms * 1e-3) / 1e9}
    if exact:
        peak, kernel, bound = peaks["dfma_tf"], "k_synth_f64 (mvb_synthesize_f64)", "fp64"
        # executed: per (image, sample) the reference's 65-tap upsample
        # (decimated tiers; 65 DMUL + 65 DADD) and the M+1-term Horner
        executed = {"algorithm": "exact fp64 engine: per (image, sample) 65-tap Kaiser upsample "
                                 "(decimated tiers) or exact distance, tau, gain, floor split, "
                                 "15-term Horner, reference summation order",
                    "note": "fp64 DMUL/DADD issue separately (no FMA contraction, bit-identity)"}
        peak_source = "measured on this GPU by bench.py (mvb_peak_dfma, best of 3)"
    else:
        peak, kernel, bound = peaks["ffma_tf"], "k_synth_f32 (mvb_synthesize_f32)", "fp32"
        executed = {
            "algorithm": "Farrow (paper Eq. 5): 32 B record gather + 8 FMA Horner per update",
            "l1_bytes_per_update": 32,
            "achieved_l1_gbs": upd_per_launch * 32 / (kern_avg_ms * 1e-3) / 1e9,
            "peak_l1_gbs": peaks["l1_gbs"],
            "frac_l1": upd_per_launch * 32 / (kern_avg_ms * 1e-3) / 1e9 / peaks["l1_gbs"],
            # the binding pipe's utilisation as ncu measures it (committed capture
            # of this kernel on this config; the 32 B model above counts only the
            # gather, ncu also sees the record broadcasts and the staging)
            "ncu_l1tex_pct": None if traffic is None else traffic.get("l1tex_throughput_pct"),
        }
        peak_source = "measured on this GPU by bench.py (mvb_peak_ffma, best of 3)"
    roof = {
        "kernel": kernel,
        "bound": bound,
        "achieved": achieved,
        "peak": peak,
        "unit": "TFLOP/s",
        "frac": achieved / peak,
        "traffic": None if traffic is None else traffic.get("dram_bytes_per_launch"),
        "traffic_source": None if traffic is None else
        f"profiles/ncu_synth_{name}.json (ncu --set full of this kernel on this config, "
        f"committed; not measured in this run)",
        "peak_source": peak_source,
        "algorithmic": f"{upd_per_launch} {'' if exact else 'non-zero '}updates (of {metric_upd} "
                       f"counted by the metric) x {w.fd_taps} taps x 2 flop per launch (SURVEY 8d: "
                       f"L FMAs per update)",
        "kernel_ms": kern_avg_ms,
        "kernel_share_of_step": kern_avg_ms / ms_step if ms_step else None,
        "hbm_leg": hbm_leg,
        "executed": executed,
    }
    gsize = {"c1": 1, "c2": 1, "c3": 1, "c4": 256, "c5": 1}[name]
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "updates/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        # c3 / c4 / c5 shard a fixed total over the ranks (strong, at every
        # N); c1 / c2 run replicas, the same job per rank (weak)
        "scaling": "weak" if parallel_mode(name) == "replicas" else "strong",
        "vs_baseline": None,
        "dtype": "f64" if precision == "fp64" else "f32 (fp64 delay anchors)",
        "data": "synthetic (seeded white Gaussian dry signal, seeded paths; SURVEY 8d)",
        "config": {
            "workload": name,
            "scenes": gsize,
            "channels": len(scenes[0].mics),
            "images_per_job": int(res.n_images.max()) if world == 1 else None,
            "out_len": [int(v) for v in res.lengths[:4]],
            "tiers": [list(t) for t in w.tiers],
            "fd": f"{w.fd_taps}-tap Hann-windowed sinc (Farrow fit" +
                  (", M=14, exact engine)" if exact else ", fp32 path degree 7)"),
            "rate": w.rate,
            "duration_s": w.duration,
            "parallelism": mode,
            "engine": ("RenderPlan: every kernel of the render re-run each step from two "
                       "CUDA graphs (geometry, synthesis) on two streams, so step k+1's "
                       "geometry overlaps step k's synthesis drain; inputs re-staged and the "
                       "decimation decision re-taken every step (speculative replay)")
                      if used_plan else "direct render_jobs per step",
            "rendered_by": rendered,
            "l2": "flushed before every timed step (256 MiB write, inside the timed region); per-step working set >L2",
        },
        "rtf": rtf,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "roofline": roof,
        "nonzero_updates_per_s": upd_per_launch * steps / (total_ms_all * 1e-3) * (
            world if shard is None and mode.startswith("replicas") else 1),
    }
    del res, jobs
    gc.collect()
    torch.cuda.empty_cache()
    return line, (wall0, wall1)


def summary(line, clk):
    """Compact per-config record for the headline line's per_config block."""
    r = line["roofline"]
    return {"value": line["value"], "ms_per_step": line["ms_per_step"], "steps": line["steps"],
            "warmup": line["warmup"], "dtype": line["dtype"],
            "e2e": None if line["e2e"] is None else line["e2e"]["value"],
            "kernel": r["kernel"], "kernel_ms": r["kernel_ms"], "frac": r["frac"],
            "peak": r["peak"], "bound": r["bound"],
            "frac_l1": r["executed"].get("frac_l1"), "rtf": line["rtf"],
            "parallelism": line["config"]["parallelism"],
            "rendered_by": line["config"]["rendered_by"], "clocks": clk}


def run_ours(args):
    import torch
    ctx = Ctx()
    peaks = None if args.profile else measured_peaks(ctx.dev)
    clocks = ClockSampler(ctx.local)
    if not args.profile:
        clocks.start()
        time.sleep(0.3)  # let nvidia-smi start before the warm-up
    line, win = measure(ctx, args.config, args.steps, args.warmup, peaks, args)
    if args.profile:
        return
    windows = {"main": win}
    per = {}
    if not args.no_per_config:
        k = max(3, min(args.steps, args.per_config_steps))
        wu = max(3, min(args.warmup, 5))
        todo = [c for c in ("c1", "c2", "c3", "c4", "c5") if c != args.config]
        for c in todo:
            ln, wn = measure(ctx, c, k, wu, peaks, args)
            per[c] = ln
            windows[c] = wn
        # same-precision (fp64) comparison on the largest single-scene config
        if ctx.world == 1:
            ln, wn = measure(ctx, "c3", 3, 3, peaks, args, precision="fp64", with_e2e=False)
            per["c3_fp64"] = ln
            windows["c3_fp64"] = wn
    clocks.stop()
    line["clocks"] = clocks.window(*windows["main"])
    # ---- CPU baseline (rank 0, N = 1) -----------------------------------------
    cpu = None
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu:
        from oracle import oracle as orc
        nth = orc.default_threads()
        v, desc, th, n_upd, dt = cpu_sample(args.config, args.cpu_seconds, nth)
        cpu = {"value": v, "unit": "updates/s", "cores": th, "kind": "port", "sample": desc,
               "seconds": dt,
               "matched": "the sample is mid-signal, where every update is non-zero; compare it "
                          "with this line's nonzero_updates_per_s (the GPU metric also counts the "
                          "exact zeros of S x out_len)",
               "l0": l0_samples(args.config, nth) if not args.no_l0 else None}
    line["cpu_baseline"] = cpu
    if per:
        line["per_config"] = {args.config: summary(line, line["clocks"])}
        for c, ln in per.items():
            line["per_config"][c] = summary(ln, clocks.window(*windows[c]))
    if ctx.rank == 0:
        print(json.dumps(line))
    if ctx.world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as orc
    nth = orc.default_threads()
    name = args.config
    total_upd, total_s = 0, 0.0
    per = max(2.0, args.cpu_seconds / max(1, args.steps))
    cpu_sample(name, 0.5, nth)  # warm-up: oracle setup (streams, tracks) + one slice
    desc = None
    for _ in range(args.steps):
        v, desc, th, n_upd, dt = cpu_sample(name, per, nth)
        total_upd += n_upd
        total_s += dt
    value = total_upd / total_s
    l0 = None if args.no_l0 else l0_samples(name, nth)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "updates/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_s / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded, same generators as the GPU arm)",
        "config": {"workload": name, "sample": desc},
        "cpu_baseline": {"value": value, "unit": "updates/s", "cores": nth, "kind": "port",
                         "sample": desc, "l0": l0},
        "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
