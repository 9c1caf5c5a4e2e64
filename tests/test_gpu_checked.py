"""The bounds-checked build (libmvb_checked.so, -DMVB_CHECKED) detects what
it is meant to detect: a render through it leaves every counter at zero,
and the same render with job tables that declare a one-row record buffer
(rec_rows = 1) trips the gather-row check on every update (the checks only
count; the kernels still read the real buffer, so the output is unchanged).
Runs in a subprocess with MVB_LIB=checked (the product loads libmvb.so).
The whole GPU suite under MVB_LIB=checked is the repo's memcheck stand-in
(profiles/r2_checked_gpu_tests.log).  Marker `gpu`."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = """
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2508_03065_b200 import _lib, engine, hann_sinc, workloads
from paper_2508_03065_b200.synth import render_jobs, scene_jobs
assert _lib.LIB_PATH.endswith("libmvb_checked.so"), _lib.LIB_PATH
sc = workloads.make_scenes("c3", duration=0.05, max_order=6, tiers=((2, 1), (4, 32), (6, 256)))[0]
f = hann_sinc(64, 14)
jobs = scene_jobs([sc])
y0 = render_jobs(jobs, f).job(0).cpu()
clean = _lib.check_violations()
orig = engine.pack_jobs
def shrunk(rows):
    a = orig(rows)
    if rows and "rec_rows" in rows[0]:
        a[:, 16:17].view(np.int32)[:, 1] = 1
    return a
engine.pack_jobs = shrunk
y1 = render_jobs(jobs, f).job(0).cpu()
bad = _lib.check_violations()
import json
print("RESULT " + json.dumps([clean, bad, bool(torch.equal(y0, y1))]))
"""


def test_checked_build_counts_out_of_bounds_gathers():
    env = dict(os.environ, MVB_LIB="checked")
    r = subprocess.run([sys.executable, "-c", CODE.format(root=ROOT)], env=env,
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT")][-1]
    clean, bad, same = json.loads(line[len("RESULT "):])
    assert not any(clean), clean
    assert bad[0] > 0, bad  # CHK_GATHER_ROW
    assert same
