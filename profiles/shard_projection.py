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
from paper_2508_03065_b200 import engine, hann_sinc, parallel, room, workloads  # noqa: E402
from paper_2508_03065_b200.plan import RenderPlan  # noqa: E402

dev = torch.device("cuda", 0)
out = {}
K = 10
# (config, partition): images / time (collective: all-reduce MAX + reduce,
# excluded here), channels (no collective); default = parallel.shard_mode
cases = [c.split(":") for c in os.environ.get("CASES", "c3:time,c3:images,c5:channels").split(",")]
for cfg, kind in cases:
    scenes = workloads.make_scenes(cfg)
    jobs = bench.device_jobs(scenes, dev)
    f = hann_sinc(scenes[0].fd_taps, 14)
    # what the all-reduce MAX would return, device-resident (an async copy)
    gmax = torch.as_tensor(engine.Geometry(jobs).dmax, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)

    def hook(t):
        t.copy_(gmax)

    res, kern = {}, {W: [] for W in (1, 2, 4, 8)}
    kern = {W: v for W, v in kern.items()}
    for W in (1, 2, 4, 8):
        if kind.startswith("hybrid") and W > 1 and W % int(kind[6:] or 2):
            continue  # hybridK needs K | W
        per_rank = []
        for r in range(W):
            mine = jobs
            if W == 1:
                plan = RenderPlan(jobs, f)
            elif kind == "channels":  # independent jobs, no collective
                mine = [jobs[i] for i in parallel.channel_shard(len(jobs), r, W)]
                plan = RenderPlan(mine, f)
            elif kind == "scenes":  # c4: LPT over scenes (bench.build_workload's cost)
                cost = [room.image_count(sc.max_order) * len(sc.mics) *
                        (sc.T + sc.max_order * float(np.max(sc.dims)) * sc.rate / 343.0)
                        for sc in scenes]
                mine = [jobs[i] for i in parallel.lpt_assign(cost, W)[r]]
                plan = RenderPlan(mine, f)
            else:
                plan = RenderPlan(jobs, f, shard=(r, W, kind), dmax_hook=hook)
            for _ in range(3):
                plan.run(mine)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for k in range(K):
                flush.fill_(float(k))
                plan.run(mine)
            plan.join()
            e1.record()
            torch.cuda.synchronize()
            per_rank.append(e0.elapsed_time(e1) / K)
            km = plan.flush_timing()
            kern[W].append(float(np.mean([km[i] for i in sorted(km)[-K:]])))
            del plan
        res[W] = per_rank
    t1 = res[1][0]
    out[f"{cfg}:{kind}"] = {W: {"ms_per_rank_step_max": round(max(v), 3),
                                "ms_per_rank_step": [round(x, 3) for x in v],
                                "synthesis_ms_per_rank": [round(x, 3) for x in kern[W]],
                                "projected_efficiency": round(t1 / (W * max(v)), 3)}
                            for W, v in res.items()}
    print(cfg, kind, {W: d["projected_efficiency"] for W, d in out[f"{cfg}:{kind}"].items()},
          flush=True)
print(json.dumps(out, indent=1))
