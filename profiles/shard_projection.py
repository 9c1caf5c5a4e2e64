"""Per-rank step time of the image-shard path on ONE GPU: every rank's
shard rendered alone (no collectives; dmax_hook stands in for the
all-reduce MAX), the max over ranks taken as the W-GPU step time -- a
projection of strong scaling, not a multi-GPU measurement (the driver's
8-GPU run measures that)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_03065_b200 import hann_sinc, workloads  # noqa: E402
from paper_2508_03065_b200.plan import RenderPlan  # noqa: E402

dev = torch.device("cuda", 0)
out = {}
K = 10
for cfg in os.environ.get("CFGS", "c3,c5").split(","):
    scenes = workloads.make_scenes(cfg)
    jobs = bench.device_jobs(scenes, dev)
    f = hann_sinc(scenes[0].fd_taps, 14)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    res = {}
    for W in (1, 2, 4, 8):
        per_rank = []
        for r in range(W):
            shard = None if W == 1 else (r, W)
            plan = RenderPlan(jobs, f, shard=shard, dmax_hook=(lambda t: t) if W > 1 else None)
            for _ in range(3):
                plan.run(jobs)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for k in range(K):
                flush.fill_(float(k))
                plan.run(jobs)
            plan.join()
            e1.record()
            torch.cuda.synchronize()
            per_rank.append(e0.elapsed_time(e1) / K)
            del plan
        res[W] = per_rank
    t1 = res[1][0]
    out[cfg] = {W: {"ms_per_rank_step_max": round(max(v), 3),
                    "ms_per_rank_step": [round(x, 3) for x in v],
                    "projected_efficiency": round(t1 / (W * max(v)), 3)} for W, v in res.items()}
    print(cfg, {W: d["projected_efficiency"] for W, d in out[cfg].items()}, flush=True)
print(json.dumps(out, indent=1))
