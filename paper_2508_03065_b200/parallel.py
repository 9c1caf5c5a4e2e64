"""Partitioning of the render path over the GPUs of one node.

One process per GPU (torchrun), torch.distributed for the plumbing:

  image shards   c3, c5: rank r renders all output samples of every job from
                 its image shard (images are independent):
                 every decimation tier split into W contiguous delay bands
                 (image_shard: images ordered by |j . dims|, their distance
                 from the room's centre image -- structural, so a render
                 plan's shard never changes with the data), band r of every
                 tier to rank r.  Per-tier counts stay balanced (the records
                 of a N=32 image cost 8x those of a N=256 one) and a rank's
                 images keep nearby delays, so the synthesis gathers keep
                 the L1 locality of the unsharded delay sort (a strided
                 subset spreads them: +20% synthesis time at W=8).  All
                 per-image work -- coarse tracks, bounds, interval records,
                 sort, synthesis -- divides by W.  Two exchanges: an all-reduce MAX of the
                 per-job track maxima (a few bytes; every rank then writes the
                 reference's out_len) and one reduce (sum) of the output
                 buffers to rank 0 -- NCCL over NVLink on B200, ~2 MB (c3) /
                 ~13 MB (c5) per render.
  time shards    (shard=(rank, world, "time")): rank r renders output
                 samples [w0, w1) of every job from all images (time_window:
                 whole tiles, cut at equal estimated cost) -- every per-sample
                 stage (coarse tracks, bounds, interval records, exact
                 maxima, sort segments, synthesis) divides by W, where image
                 shards keep the per-job geometry on every rank.  The same two
                 exchanges: all-reduce MAX of the window maxima (the global
                 out_len) and the reduce (sum) of the outputs, zero outside a
                 rank's window, to rank 0.
  scene shards   c4: independent scenes, longest-processing-time assignment
                 by update count; no collective.
  channel shards c5: the receivers of a scene (independent jobs); no collective.
  replicas       c1, c2: too small to split; every rank renders the job.

The partition functions are pure host logic (tested with gloo on CPU);
`reduce_to_root` is the only collective and works on any backend.
"""

from __future__ import annotations

import heapq
import os
from functools import lru_cache

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


@lru_cache(maxsize=16)
def canonical_lattice(max_order: int) -> tuple:
    """(j (S, 3) int64, order (S,)) of the canonical image list (reference
    room.py:98-143: sorted by (order, lattice, parity) with lattice l =
    (j + q) // 2, parity q = j mod 2) -- the structure only, on the host.
    The image of a source at the room centre lies at j * dims from it."""
    K = int(max_order)
    r = np.arange(-K, K + 1)  # cached per order (a 20th-order lattice is 69k candidates)
    j = np.stack(np.meshgrid(r, r, r, indexing="ij"), axis=-1).reshape(-1, 3)
    order = np.abs(j).sum(axis=1)
    j, order = j[order <= K], order[order <= K]
    q = np.mod(j, 2)
    lat = (j + q) // 2
    keys = (q[:, 2], q[:, 1], q[:, 0], lat[:, 2], lat[:, 1], lat[:, 0], order)
    idx = np.lexsort(keys)  # last key primary: order, lattice x, y, z, parity x, y, z
    j, order = j[idx].astype(np.int64), order[idx].astype(np.int64)
    j.flags.writeable = order.flags.writeable = False  # cached
    return j, order


def image_shard(dims, max_order: int, tiers, rank: int, world: int, images=None) -> np.ndarray:
    """Canonical image positions owned by `rank` (sorted): every tier of
    `tiers` ((max_order, N), ...) ordered by |j * dims| (ties by canonical
    position) and cut into `world` contiguous bands of equal estimated cost
    (_band_cuts); band `rank` of every tier.  `images`: restrict to these canonical
    positions (e.g. a t60 cull).  The shards of ranks 0..world-1 partition
    the image list."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    key = (np.asarray(dims, dtype=np.float64).tobytes(), int(max_order),
           tuple((int(a), int(b)) for a, b in tiers), int(rank), int(world),
           None if images is None else np.asarray(images, dtype=np.int64).tobytes())
    return _image_shard(key)


@lru_cache(maxsize=256)
def _image_shard(key) -> np.ndarray:
    dims_b, max_order, tiers, rank, world, images_b = key
    dims = np.frombuffer(dims_b, dtype=np.float64)
    images = None if images_b is None else np.frombuffer(images_b, dtype=np.int64)
    j, order = canonical_lattice(max_order)
    idx = np.arange(order.size, dtype=np.int64) if images is None \
        else np.asarray(images, dtype=np.int64)
    key = np.linalg.norm(j[idx] * np.asarray(dims, dtype=np.float64).reshape(1, 3), axis=1)
    mine = []
    prev = -1
    for mo, _ in tiers:
        sel = np.nonzero((order[idx] > prev) & (order[idx] <= int(mo)))[0]
        prev = int(mo)
        band = sel[np.lexsort((idx[sel], key[sel]))]  # by distance, then canonical position
        cut = _band_cuts(key[band], world)
        mine.append(idx[band[cut[rank]:cut[rank + 1]]])
    out = np.sort(np.concatenate(mine)) if mine else np.zeros(0, np.int64)
    out.flags.writeable = False  # cached: shared by every caller
    return out


def band_order(dims, max_order: int, images=None) -> np.ndarray:
    """The job's canonical image positions (all, or `images`) ordered by
    |j * dims| (ties by canonical position): time-shard jobs build their
    image table in this order so independent sorts of consecutive runs
    (mvb_delay_sort_runs) approximate one delay sort.  Structural."""
    key = (np.asarray(dims, dtype=np.float64).tobytes(), int(max_order),
           None if images is None else np.asarray(images, dtype=np.int64).tobytes())
    return _band_order(key)


@lru_cache(maxsize=64)
def _band_order(key) -> np.ndarray:
    dims_b, max_order, images_b = key
    j, order = canonical_lattice(max_order)
    idx = np.arange(order.size, dtype=np.int64) if images_b is None \
        else np.frombuffer(images_b, dtype=np.int64)
    d = np.linalg.norm(j[idx] * np.frombuffer(dims_b, np.float64)[None, :], axis=1)
    out = idx[np.lexsort((idx, d))]
    out.flags.writeable = False
    return out


SPARSITY_COST = 0.4  # extra synthesis cost of an image ~ SPARSITY_COST / local density (per m)


def _band_cuts(keys: np.ndarray, world: int) -> np.ndarray:
    """Cut positions of `world` contiguous bands of the sorted distances
    `keys` at equal estimated synthesis cost: an image costs
    1 + SPARSITY_COST / rho, rho its local density (images per metre over
    +-16 neighbours) -- sparse delay bands (the far tips of the order
    octahedron) reuse fewer L1 lines per gather.  0.4 is the best of
    {0.4, 0.75} on c3 and c5 at W=8 (per-rank step spread c3 1.6%, c5 4.7%;
    profiles/r1_shard_projection.json)."""
    n = keys.size
    if n == 0:
        return np.zeros(world + 1, np.int64)
    p = np.arange(n)
    lo, hi = np.maximum(p - 16, 0), np.minimum(p + 16, n - 1)
    span = np.maximum(keys[hi] - keys[lo], 1e-9)
    w = 1.0 + SPARSITY_COST * span / np.maximum(hi - lo, 1)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    # targets nudged down by a rounding margin: equal weights give equal bands
    target = cum[-1] * np.arange(world + 1) / world - 1e-9 * cum[-1]
    cut = np.searchsorted(cum, target, side="left")
    cut[0], cut[-1] = 0, n
    return np.maximum.accumulate(np.clip(cut, 0, n)).astype(np.int64)


def shard_jobs(jobs, rank: int, world: int, by: str = "images") -> list:
    """Jobs restricted to their shard of `rank`, with explicit path / signal
    keys so shards of one batch still share them: by="images" the image
    shard (image_shard), by="time" the output window (time_window)."""
    from dataclasses import replace

    from . import engine
    if by.startswith("hybrid"):
        # "hybridK": K image bands x world/K output windows (rank = band *
        # (world/K) + window); the same two exchanges over all ranks
        K = int(by[len("hybrid"):] or 2)
        if K < 1 or world % K:
            raise ValueError("hybridK needs K | world")
        Wt = world // K
        band, win = divmod(rank, Wt)
        sub = shard_jobs(jobs, band, K, "images") if K > 1 else list(jobs)
        return shard_jobs(sub, win, Wt, "time") if Wt > 1 else sub
    if by not in ("images", "time"):
        raise ValueError("shard by 'images', 'time' or 'hybridK'")
    keys = [dict(signal_key=engine._key(jb.signal_key, jb.s),
                 path_key=engine._key(jb.path_key, jb.pos)) for jb in jobs]
    if by == "time":
        return [replace(jb, window=time_window(jb, rank, world),
                        image_index=band_order(jb.dims, jb.max_order, jb.image_index), **k)
                for jb, k in zip(jobs, keys)]
    return [replace(jb, image_index=image_shard(jb.dims, jb.max_order, jb.tiers, rank, world,
                                                jb.image_index), **k)
            for jb, k in zip(jobs, keys)]


def shard_kind(shard) -> str:
    """'images' (default) or 'time' of a shard tuple (rank, world[, kind])."""
    return str(shard[2]) if shard is not None and len(shard) > 2 else "images"


def _length(a) -> int:
    return int(a.shape[0]) if hasattr(a, "shape") else len(a)


TIME_GEOMETRY_COST = 0.1  # per-rank tracks + records per path sample and image, in updates
# an image with no contribution to a tile (before its first arrival, after
# the signal) still costs its staging and zero test, in updates per sample
TIME_SKIP_COST = float(os.environ.get("MVB_TIME_SKIP_COST", "0.2"))


def time_window(jb, rank: int, world: int) -> tuple:
    """Output window (w0, w1) of `rank` for the time shards of job `jb`
    (w1 = 0: to the end of the output).  Structural -- a function of the
    room, image order, path / signal lengths, rate and world only -- so
    every rank computes the same cuts and a render plan's shard never
    changes with the data.  Cost of output sample n: the images that
    contribute to it, #{i : tau_i <= n < Ts + tau_i} with tau_i estimated as
    kappa * |j_i * dims| (the image of the room centre; a few metres off for
    off-centre sources, i.e. a few hundred samples of a ~1e4-1e5-sample
    delay spread), plus TIME_GEOMETRY_COST * S for every path sample (the
    window's tracks and interval records) and TIME_SKIP_COST * S for every
    output sample (images skipped as exact zeros still cost their staging).
    Cuts land on whole TILEs."""
    from .engine import TILE
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    if world == 1:
        return (0, 0)
    T = _length(jb.pos)
    Ts = int(np.prod(jb.s.shape)) if hasattr(jb.s, "shape") else len(jb.s)
    key = (np.asarray(jb.dims, dtype=np.float64).tobytes(), int(jb.max_order),
           None if jb.image_index is None else np.asarray(jb.image_index, np.int64).tobytes(),
           int(T), int(Ts), float(jb.rate) / float(jb.c), int(world), int(TILE), TIME_SKIP_COST)
    cuts = _time_cuts(key)
    return (int(cuts[rank]) * TILE, int(cuts[rank + 1]) * TILE if rank + 1 < world else 0)


@lru_cache(maxsize=256)
def _time_cuts(key) -> np.ndarray:
    dims_b, max_order, images_b, T, Ts, kappa, world, tile, skip = key
    j, _ = canonical_lattice(max_order)
    if images_b is not None:
        j = j[np.frombuffer(images_b, dtype=np.int64)]
    tau = np.sort(kappa * np.linalg.norm(j * np.frombuffer(dims_b, np.float64)[None, :], axis=1))
    S = tau.size
    n_tiles = -(-int(Ts + np.ceil(tau[-1]) + 64) // tile)
    if n_tiles < world:
        raise ValueError(f"{n_tiles} output tiles cannot be cut into {world} time shards")
    x = np.arange(n_tiles + 1, dtype=np.float64) * tile
    pre = np.concatenate([[0.0], np.cumsum(tau)])

    def ramp(y):  # sum_i max(y - tau_i, 0)
        m = np.searchsorted(tau, y, side="left")
        return m * y - pre[m]

    cost = ramp(x) - ramp(x - Ts) + TIME_GEOMETRY_COST * S * np.minimum(x, T) + \
        skip * S * x
    target = cost[-1] * np.arange(world + 1) / world
    cuts = np.searchsorted(cost, target, side="left")
    cuts[0], cuts[-1] = 0, n_tiles
    for r in range(1, world + 1):  # every rank at least one tile
        cuts[r] = max(cuts[r], cuts[r - 1] + 1)
    for r in range(world - 1, -1, -1):
        cuts[r] = min(cuts[r], cuts[r + 1] - 1)
    out = cuts.astype(np.int64)
    out.flags.writeable = False
    return out


# Every collective this process issued, in order: (name, elements).  The
# ranks of a sharded render must issue the same sequence (a rank that skips
# or adds one hangs the group); tests compare the logs across ranks.
COLLECTIVE_LOG: list = []


def _group_size(group):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group)
    return 1


def _host_staged(group) -> bool:
    """gloo groups run their collectives on host tensors: device buffers
    are copied through the host (the CPU test harness and the one-GPU
    multi-process rehearsal; NCCL reduces device buffers in place)."""
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo"


def allreduce_max(t, group=None):
    """In-place MAX over the ranks (no-op without a process group)."""
    import torch.distributed as dist
    if _group_size(group) > 1:
        COLLECTIVE_LOG.append(("all_reduce_max", int(t.numel())))
        if t.is_cuda and _host_staged(group):
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.MAX, group=group)
            t.copy_(h)
        else:
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
    """'single' | 'images' | 'scenes' | 'channels' | 'replicas' for a
    BASELINE config.  c5 (one scene, 8 receivers) shards its channels --
    independent (scene, channel) jobs, no collective, SURVEY 8(e)'s
    "each GPU takes one channel" -- so each rank's geometry shrinks with W
    as well (image shards replicate the per-job geometry on every rank:
    projected W = 8 efficiency 0.79)."""
    if world == 1:
        return "single"
    return {"c3": "images", "c5": "channels", "c4": "scenes"}.get(workload, "replicas")


def channel_shard(n_channels: int, rank: int, world: int) -> list:
    """Channels of a multi-receiver scene rendered by `rank`: LPT over
    equal-cost channels, i.e. round-robin (rank r takes r, r + W, ...)."""
    return lpt_assign(np.ones(int(n_channels)), world)[rank]


def reduce_to_root(t, group=None, root: int = 0):
    """Sum a partial output buffer into `root` (in place on root), on the
    current stream."""
    import torch.distributed as dist
    if _group_size(group) > 1:
        COLLECTIVE_LOG.append(("reduce_sum", int(t.numel())))
        if t.is_cuda and _host_staged(group):
            h = t.cpu()
            dist.reduce(h, dst=root, op=dist.ReduceOp.SUM, group=group)
            if dist.get_rank(group) == root:
                t.copy_(h)
        else:
            dist.reduce(t, dst=root, op=dist.ReduceOp.SUM, group=group)
    return t
