"""Render throughput of K back-to-back renders, direct (render_jobs) vs
CUDA-graph replays (plan.RenderPlan), device-resident inputs, one GPU."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2508_03065_b200 import hann_sinc, workloads
from paper_2508_03065_b200.plan import RenderPlan
from paper_2508_03065_b200.synth import render_jobs

dev = torch.device("cuda", 0)
out = {}
for cfg in os.environ.get("CFGS", "c1,c2,c3").split(","):
    w = workloads.WORKLOADS[cfg]
    scenes = workloads.make_scenes(cfg)
    jobs = bench.device_jobs(scenes, dev)
    f = hann_sinc(scenes[0].fd_taps, 14)
    prec = "fp64" if w.dtype == "f64" else "fp32"
    ready = torch.cuda.Event(); ready.record()
    plan = RenderPlan(jobs, f, precision=prec)
    res = {}
    for name, step in (("direct", lambda: render_jobs(jobs, f, precision=prec, inputs_ready=ready)),
                       ("plan", lambda: plan.run(jobs))):
        for _ in range(4):
            r = step()
        torch.cuda.synchronize()
        K = 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rs = [step() for _ in range(K)]
        rs[-1].wait()  # plan results: order e1 after the plan's streams
        plan.join()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        res[name] = {"ms_per_step": round(ms, 3), "updates_per_s": rs[-1].updates / (ms * 1e-3)}
    out[cfg] = res
print(json.dumps(out, indent=1))
