"""Small renders for compute-sanitizer (memcheck / racecheck / synccheck):
smoke() (fast + exact engines and a render plan), reduced c3 (3 tiers, 64
taps) and c5 (moving 2-mic array) on both engines, the reference-default
Farrow filter, a render plan with speculative replays, and the
static / splice kernels.  Run one tool per process:

    PYTORCH_NO_CUDA_MEMORY_CACHING=1 compute-sanitizer --tool memcheck \
        python profiles/sanitize_cases.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import __graft_entry__ as ge  # noqa: E402
from paper_2508_03065_b200 import hann_sinc, workloads  # noqa: E402
from paper_2508_03065_b200.plan import RenderPlan  # noqa: E402
from paper_2508_03065_b200.synth import render_jobs, scene_jobs  # noqa: E402

# PYTORCH_NO_CUDA_MEMORY_CACHING=1 (one allocation per tensor: memcheck sees
# exact bounds) forbids CUDA-graph capture: SAN_NO_PLAN=1 skips the plans
NO_PLAN = os.environ.get("SAN_NO_PLAN") == "1"
if not NO_PLAN:
    ge.smoke()
cases = [
    ("c3", workloads.make_scenes("c3", duration=0.03, max_order=6, tiers=((2, 1), (4, 32), (6, 256)))),
    ("c5", workloads.make_scenes("c5", duration=0.02, max_order=5, n_channels=2,
                                 tiers=((2, 1), (3, 32), (5, 256)))),
    ("c4", workloads.make_scenes("c4", duration=0.02, max_order=4, n_scenes=3, tiers=((2, 1), (4, 64)))),
]
for name, scenes in cases:
    sc = scenes[0]
    f = hann_sinc(sc.fd_taps, 14)
    jobs = scene_jobs(scenes)
    for prec in ("fp32", "fp64"):
        res = render_jobs(jobs, f, precision=prec)
        print(name, prec, [int(v) for v in res.lengths], float(res.out.abs().max()), flush=True)
    if NO_PLAN:
        continue
    plan = RenderPlan(jobs, f)
    for _ in range(3):
        r = plan.run(jobs)
    r.wait()
    print(name, "plan", plan.captures, float(r.out.abs().max()), flush=True)
    plan.join()
torch.cuda.synchronize()
# reference-default Farrow filter (M=3, L=8) on the fast engine
from paper_2508_03065_b200.farrow import FarrowFilter  # noqa: E402
g = np.load(os.path.join(ROOT, "tests", "golden", "kernels.npz"))
fd = FarrowFilter(3, 8, g["design_3_8_08"], 3, 0.8)
sc = cases[0][1][0]
res = render_jobs(scene_jobs([sc]), fd)
print("refdesign", float(res.out.abs().max()), flush=True)
# static responses / splice baseline kernels
import paper_2508_03065_b200 as mvb  # noqa: E402
room = mvb.Room(dims=np.array([5.0, 6.0, 4.0]), wall_reflection=np.full(6, 0.9))
mic = np.array([2.0, 3.0, 1.5])
rir = mvb.static_rir(room, np.array([1.0, 1.5, 1.2]), mic, 16000.0, 3)
y = mvb.static_render(np.random.default_rng(0).standard_normal(4000), rir)
pos = np.linspace([1.0, 1.0, 1.2], [4.0, 5.0, 1.2], 8000)
traj = mvb.Trajectory(rate=16000.0, positions=pos)
cfg = mvb.SynthesisConfig(audio_rate=16000.0, max_order=3)
z = mvb.splice_baseline(np.random.default_rng(1).standard_normal(8000), traj, room, mic, 1600, 160, cfg)
print("static", y.size, float(np.max(np.abs(y))), "splice", z.size, flush=True)
torch.cuda.synchronize()
print("SANITIZE_CASES_DONE")
