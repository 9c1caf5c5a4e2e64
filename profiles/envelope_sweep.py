"""fp32 fast-path error against the interval delay excursion (evidence for
engine.FP32_ENVELOPE).  The envelope guard is switched off, a straight
source path is rendered at increasing speeds with the largest decimation
of the configs (N = 256 at 48 kHz) and compared with the CPU oracle.

    python profiles/envelope_sweep.py > profiles/r2_envelope_sweep.json
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import oracle as orc  # noqa: E402
from paper_2508_03065_b200 import engine, hann_sinc  # noqa: E402
from paper_2508_03065_b200.synth import render_jobs  # noqa: E402

RATE, TIERS = 48000.0, ((2, 1), (6, 256))
DIMS, MIC = np.array([7.0, 5.0, 3.5]), np.array([3.0, 2.5, 1.4])
engine.FP32_ENVELOPE = float("inf")  # guard off: measure the fast path itself
f = hann_sinc(64, 14)
rows = []
for speed in (5.0, 20.0, 50.0, 100.0, 170.0, 250.0, 340.0, 450.0, 600.0):
    errs = []
    for seed in range(3):
        rng = np.random.default_rng(seed)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        T = 9600
        pos = np.array([2.0, 2.0, 1.5]) + d * speed * (np.arange(T)[:, None] / RATE)
        s = rng.standard_normal(T).astype(np.float32)
        job = engine.Job(s=s, pos=pos, mic=MIC, dims=DIMS, walls=0.9, max_order=6, tiers=TIERS,
                         rate=RATE)
        res = render_jobs([job], f, precision="fp32")
        y = res.job(0).double().cpu().numpy()
        ref = orc.OracleScene(s.astype(np.float64), pos, MIC, DIMS, 0.9, 6, TIERS, f.branches,
                              RATE).render()
        errs.append(float(np.max(np.abs(y - ref)) / np.max(np.abs(ref))))
    rows.append({"speed_mps": speed, "excursion_samples": speed * 256 / 343.0,
                 "max_err_over_peak": max(errs), "seeds": 3})
    print(json.dumps(rows[-1]), file=sys.stderr)
print(json.dumps({"what": "fp32 fast path, guard off, N=256 at 48 kHz, orders 3-6 decimated",
                  "envelope_samples": engine.FP32_ENVELOPE, "rows": rows}, indent=1))
