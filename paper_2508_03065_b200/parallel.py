"""Partitioning of the render path over the GPUs of one node.

One process per GPU (torchrun), torch.distributed for the plumbing:

  image shards   c3, c5: rank r renders all output samples of every job from
                 the strided image subset r, r+W, r+2W, ... of its canonical
                 list (images are independent; striding keeps
                 every tier balanced), so enumeration-independent work --
                 coarse tracks, bounds, interval records, sort, synthesis --
                 divides by W.  Two exchanges: an all-reduce MAX of the
                 per-job track maxima (a few bytes; every rank then writes the
                 reference's out_len) and one reduce (sum) of the output
                 buffers to rank 0 -- NCCL over NVLink on B200, ~2 MB (c3) /
                 ~13 MB (c5) per render.
  scene shards   c4: independent scenes, longest-processing-time assignment
                 by update count; no collective.
  replicas       c1, c2: too small to split; every rank renders the job.

The partition functions are pure host logic (tested with gloo on CPU);
`reduce_to_root` is the only collective and works on any backend.
"""

from __future__ import annotations

import heapq

import numpy as np


def image_subset(images, rank: int, world: int) -> np.ndarray:
    """Canonical image positions owned by `rank`: every world-th entry of
    `images` (an image count or an index list) starting at `rank`; the
    subsets of ranks 0..world-1 partition it."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    idx = np.arange(int(images), dtype=np.int64) if np.ndim(images) == 0 \
        else np.asarray(images, dtype=np.int64)
    return idx[rank::world]


def allreduce_max(t, group=None):
    """In-place MAX over the ranks (no-op without a process group)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t


def lpt_assign(costs, world: int) -> list:
    """Longest-processing-time-first assignment of independent jobs: the
    heaviest job goes to the least-loaded rank (ties: lowest rank), jobs of
    equal cost in index order.  Returns one sorted index list per rank."""
    if world < 1:
        raise ValueError("world must be >= 1")
    costs = np.asarray(costs, dtype=np.float64)
    order = sorted(range(costs.size), key=lambda i: (-costs[i], i))
    heap = [(0.0, r) for r in range(world)]
    out = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + float(costs[i]), r))
    return [sorted(v) for v in out]


def shard_mode(workload: str, world: int) -> str:
    """'single' | 'images' | 'scenes' | 'replicas' for a BASELINE config."""
    if world == 1:
        return "single"
    return {"c3": "images", "c5": "images", "c4": "scenes"}.get(workload, "replicas")


def reduce_to_root(t, group=None, root: int = 0):
    """Sum a partial output buffer into `root` (in place on root)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.reduce(t, dst=root, op=dist.ReduceOp.SUM, group=group)
    return t
