"""SURVEY H2 A/B on the bench workload (c3): the fast synthesis with the
Farrow records (product) against the literal per-fraction-table gather
(engine.FD_GATHER = "table"), same tracks, same work list; synthesis kernel
time by CUDA events, accuracy against the oracle on windows.

    python profiles/table_ab.py [c3] > profiles/r2_table_ab.json
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from oracle import oracle as orc  # noqa: E402
from paper_2508_03065_b200 import engine, hann_sinc, workloads  # noqa: E402
from paper_2508_03065_b200.synth import render_jobs, scene_jobs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
sc = workloads.make_scenes(name)[0]
f = hann_sinc(sc.fd_taps, 14)
dev = torch.device("cuda", 0)
jobs = scene_jobs([sc])
o = orc.OracleScene(sc.s, sc.pos, sc.mics[0], sc.dims, sc.walls, sc.max_order, sc.tiers,
                    f.branches, sc.rate)
out = {"workload": name, "taps": sc.fd_taps, "table_rows": engine.TAB_P + 1}
for mode in ("farrow", "table"):
    engine.FD_GATHER = mode
    ms = []
    for it in range(4):
        t = []
        res = render_jobs(jobs, f, timing=t)
        torch.cuda.synchronize()
        ms.append(t[0][0].elapsed_time(t[0][1]))
    y = res.job(0).double().cpu().numpy()
    err = peak = 0.0
    for a in np.linspace(0, y.size - 2048, 4).astype(int):
        ref = o.render_window(int(a), int(a) + 2048)
        err = max(err, float(np.max(np.abs(y[a:a + 2048] - ref))))
        peak = max(peak, float(np.max(np.abs(ref))))
    upd = int(res.n_images[0]) * min(int(res.lengths[0]), sc.s.size + sc.fd_taps - 1)
    out[mode] = {"synth_ms": float(np.median(ms[1:])), "all_ms": ms,
                 "nonzero_updates": upd,
                 "taps_x_fma_tflops": upd * sc.fd_taps * 2 / (np.median(ms[1:]) * 1e-3) / 1e12,
                 "window_err_over_window_peak": err / peak}
    print(mode, out[mode], file=sys.stderr, flush=True)
out["speedup_farrow_over_table"] = out["table"]["synth_ms"] / out["farrow"]["synth_ms"]
print(json.dumps(out, indent=1))
