"""Where a W-rank image shard's step goes, on ONE GPU: host time per
RenderPlan.run, GPU step time, and the geometry / synthesis graph durations
of an isolated run (events on the plan streams).  Diagnostic only."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_03065_b200 import hann_sinc, workloads  # noqa: E402
from paper_2508_03065_b200.plan import RenderPlan  # noqa: E402

dev = torch.device("cuda", 0)
K = 20
out = {}
for cfg in os.environ.get("CFGS", "c3").split(","):
    scenes = workloads.make_scenes(cfg)
    jobs = bench.device_jobs(scenes, dev)
    f = hann_sinc(scenes[0].fd_taps, 14)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    for W in [int(w) for w in os.environ.get("WS", "1,8").split(",")]:
        shard = None if W == 1 else (0, W)
        plan = RenderPlan(jobs, f, shard=shard, dmax_hook=(lambda t: t) if W > 1 else None)
        for _ in range(3):
            plan.run(jobs)
        torch.cuda.synchronize()
        # isolated run: graph durations
        iso = []
        for _ in range(5):
            slot = plan.slots[plan.k % plan.DEPTH]
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            orig = plan._replay

            def timed(slot_, after, ev=ev):
                geo, syn = plan.geo_stream, plan.syn_stream
                geo.wait_event(after)
                ev[0].record(geo)
                with torch.cuda.stream(geo):
                    slot_.graphs[0].replay()
                    if plan.dmax_hook is not None:
                        plan.dmax_hook(slot_.dmax)
                    ev[1].record(geo)
                syn.wait_event(ev[1])
                with torch.cuda.stream(syn):
                    ev[2].record(syn)
                    slot_.graphs[1].replay()
                    ev[3].record(syn)
                    slot_.done = torch.cuda.Event()
                    slot_.done.record()
            plan._replay = timed
            t0 = time.perf_counter()
            plan.run(jobs)
            t1 = time.perf_counter()
            plan._replay = orig
            torch.cuda.synchronize()
            iso.append({"geo_ms": ev[0].elapsed_time(ev[1]), "syn_ms": ev[2].elapsed_time(ev[3]),
                        "geo_start_to_syn_end_ms": ev[0].elapsed_time(ev[3]),
                        "host_run_ms": 1e3 * (t1 - t0)})
        # steady loop: host time per run and device time per step
        host = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(K):
            flush.fill_(float(k))
            t0 = time.perf_counter()
            plan.run(jobs)
            host.append(1e3 * (time.perf_counter() - t0))
        plan.join()
        e1.record()
        torch.cuda.synchronize()
        res = {"step_ms": e0.elapsed_time(e1) / K, "host_run_ms_median": sorted(host)[K // 2],
               "host_run_ms_max": max(host), "isolated": iso[-3:],
               "launches": plan.slots[0].graph_launches, "misses": plan.misses}
        # no flush, same loop
        e0.record()
        for k in range(K):
            plan.run(jobs)
        plan.join()
        e1.record()
        torch.cuda.synchronize()
        res["step_ms_noflush"] = e0.elapsed_time(e1) / K
        # timeline of 6 steady steps (flush included): per step the flush end,
        # geometry start / end and synthesis start / end relative to e0, and
        # the host time at which run() enqueued the replay
        marks = []
        orig = plan._replay

        def traced(slot_, after):
            geo, syn = plan.geo_stream, plan.syn_stream
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            geo.wait_event(after)
            ev[0].record(geo)
            with torch.cuda.stream(geo):
                slot_.graphs[0].replay()
                if plan.dmax_hook is not None:
                    plan.dmax_hook(slot_.dmax)
                ev[1].record(geo)
            syn.wait_event(ev[1])
            with torch.cuda.stream(syn):
                ev[2].record(syn)
                slot_.graphs[1].replay()
                ev[3].record(syn)
                slot_.done = torch.cuda.Event()
                slot_.done.record()
            marks[-1]["ev"] = ev
            marks[-1]["host_replay"] = time.perf_counter()
        plan._replay = traced
        torch.cuda.synchronize()
        e0.record()
        h0 = time.perf_counter()
        for k in range(8):
            fe = torch.cuda.Event(enable_timing=True)
            flush.fill_(float(k))
            fe.record()
            marks.append({"flush": fe, "host_start": time.perf_counter()})
            plan.run(jobs)
            marks[-1]["host_end"] = time.perf_counter()
        plan.join()
        torch.cuda.synchronize()
        plan._replay = orig
        tl = []
        for m in marks:
            tl.append([round(e0.elapsed_time(m["flush"]), 3)] +
                      [round(e0.elapsed_time(e), 3) for e in m["ev"]] +
                      [round(1e3 * (m[k] - h0), 3) for k in ("host_start", "host_replay", "host_end")])
        res["timeline"] = tl
        print("timeline [flush_end, geo0, geo1, syn0, syn1 | host_start, host_replay, host_end]")
        for row in tl:
            print("   ", row)
        out[f"{cfg}_W{W}"] = res
        print(cfg, W, json.dumps(res), flush=True)
        del plan
print(json.dumps(out, indent=1))
