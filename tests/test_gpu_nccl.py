"""The multi-GPU code path of a sharded render plan with a real NCCL process
group: the default dmax hook (all-reduce MAX, issued eagerly between the
plan's two graphs on its geometry stream) and the output reduce to rank 0
issued on the plan's synthesis stream, as `bench.py --gpus N` runs them.

Only one GPU is reachable, so the group has ONE rank (no rank waits on
another); the rank renders shard 0 of a world-2 partition, and the result
must equal the same shard rendered directly with an identity hook.  The
cross-rank semantics of the partition and the collectives are covered by
tests/test_parallel.py (gloo, world_size 2).  Marker `gpu`."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

from paper_2508_03065_b200 import hann_sinc, parallel, workloads  # noqa: E402
from paper_2508_03065_b200.plan import RenderPlan  # noqa: E402
from paper_2508_03065_b200.synth import render_jobs, scene_jobs  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture
def nccl_group():
    if not dist.is_nccl_available():
        pytest.skip("NCCL backend not available")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_sharded_plan_with_nccl_hooks(nccl_group):
    scenes = workloads.make_scenes("c5", duration=0.05, max_order=6, n_channels=2,
                                   tiers=((2, 1), (4, 32), (6, 256)))
    f = hann_sinc(64, 14)
    jobs = scene_jobs(scenes)
    # parallel.allreduce_max / reduce_to_root skip the collective for one rank:
    # issue the same NCCL operations directly so they really run on the plan's
    # streams (all-reduce MAX between the graphs, reduce after the synthesis)
    calls = []

    def hook(t):
        calls.append(1)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)

    plan = RenderPlan(jobs, f, shard=(0, 2), dmax_hook=hook)
    ref = render_jobs(jobs, f, shard=(0, 2), dmax_hook=lambda t: t)
    for it in range(4):  # capture both slots, then speculative replays
        res = plan.run(jobs)
        with torch.cuda.stream(res.stream):
            dist.reduce(res.out, dst=0, op=dist.ReduceOp.SUM)  # on the synthesis stream
        res.wait()
        assert np.array_equal(res.lengths, ref.lengths), it
        for j in range(len(jobs)):
            assert torch.equal(res.job(j), ref.job(j)), (it, j)
    plan.join()
    torch.cuda.synchronize()
    assert plan.captures == 2 and plan.misses == 0
    assert len(calls) == 4 + 2  # one per run plus the dry run of each capture
    assert parallel.shard_mode("c3", 2) == "images"
