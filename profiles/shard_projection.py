"""Per-rank step time of the image-shard path on ONE GPU (rank 0's subset
alone, no collectives): a projection of strong scaling, not a multi-GPU
measurement."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2508_03065_b200 import hann_sinc, workloads
from paper_2508_03065_b200.plan import RenderPlan
from paper_2508_03065_b200.synth import render_jobs
dev = torch.device('cuda', 0)
out = {}
for cfg in os.environ.get('CFGS', 'c3,c5').split(','):
    scenes = workloads.make_scenes(cfg)
    jobs = bench.device_jobs(scenes, dev)
    f = hann_sinc(scenes[0].fd_taps, 14)
    ready = torch.cuda.Event(); ready.record()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    for mode in ("plan", "direct"):
        res = {}
        for W in (1, 2, 4, 8):
            shard = None if W == 1 else (0, W)
            hook = (lambda t: t) if W > 1 else None  # stands in for the all-reduce MAX
            if mode == "plan":
                plan = RenderPlan(jobs, f, shard=shard, dmax_hook=hook)
                step = lambda: plan.run(jobs)
            else:
                step = lambda: render_jobs(jobs, f, shard=shard, inputs_ready=ready, dmax_hook=hook)
            for _ in range(3):
                step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            K = 10
            e0.record()
            for k in range(K):
                flush.fill_(float(k))
                step()
            if mode == "plan":
                plan.join()  # the plan renders on its own streams
            e1.record(); torch.cuda.synchronize()
            res[W] = e0.elapsed_time(e1) / K
        out[f"{cfg}_{mode}"] = {W: {"ms_per_rank_step": round(t, 3),
                                    "projected_efficiency": round(res[1] / (W * t), 3)}
                                for W, t in res.items()}
print(json.dumps(out, indent=1))
