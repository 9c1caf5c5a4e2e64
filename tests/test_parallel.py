"""Multi-GPU partitioning logic on CPU: image_shard / image_subset /
lpt_assign properties and a world_size-2 gloo run of the image-shard path
-- per-tier delay-band shards, the all-reduce MAX of the track maxima and the
sum-reduce of the outputs -- with the CPU oracle rendering each rank's
shard (test infrastructure stands in for the GPU renderer; the partition
and the collectives are the product code)."""

import os
import socket
import tempfile

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_03065_b200 import parallel


def test_image_subsets_partition_and_balance():
    for n in (0, 1, 7, 11521):
        for world in (1, 2, 3, 8):
            got = [parallel.image_subset(n, r, world) for r in range(world)]
            assert np.array_equal(np.sort(np.concatenate(got)), np.arange(n))
            assert max(g.size for g in got) - min(g.size for g in got) <= 1
    sub = np.array([3, 5, 8, 13, 21])
    assert parallel.image_subset(sub, 1, 2).tolist() == [5, 13]


def test_time_windows_partition_on_tiles():
    """Time shards (parallel.time_window): whole TILEs, increasing, the
    last open-ended; the same cuts on every rank (structural); the
    estimated cost balanced (c3 shape: within 2% at W = 8)."""
    from paper_2508_03065_b200 import engine, workloads
    from paper_2508_03065_b200.engine import TILE
    sc = workloads.make_scenes("c3", duration=10.0)[0]
    jb = engine.Job(s=sc.s, pos=sc.pos, mic=sc.mics[0], dims=sc.dims, walls=sc.walls,
                    max_order=sc.max_order, tiers=sc.tiers, rate=sc.rate)
    for world in (1, 2, 3, 8):
        w = [parallel.time_window(jb, r, world) for r in range(world)]
        assert w[0][0] == 0 and w[-1][1] == 0
        for r in range(world - 1):
            assert w[r][1] == w[r + 1][0] and w[r][0] < w[r][1] and w[r][1] % TILE == 0
        if world > 1:  # cost estimate per window (same model, evaluated here)
            j, _ = parallel.canonical_lattice(sc.max_order)
            tau = sc.rate / 343.0 * np.linalg.norm(j * sc.dims, axis=1)
            T = sc.T

            def cost(x):
                return np.clip(x - tau, 0, T).sum() + tau.size * (
                    parallel.TIME_GEOMETRY_COST * min(x, T) + parallel.TIME_SKIP_COST * x)
            end = T + tau.max() + 64
            c = [cost(min(w1 if w1 else end, end)) - cost(w0) for w0, w1 in w]
            assert max(c) / min(c) < 1.02, (world, c)
    with np.testing.assert_raises(ValueError):
        parallel.shard_jobs([jb], 0, 2, by="stripes")


def test_window_fields():
    """mvb_job window words: path range [p0, p1) and the sort-segment
    centres (engine.window_fields mirrors win_p0 / win_p1)."""
    from paper_2508_03065_b200 import engine
    from paper_2508_03065_b200.engine import SEG_LEN, TILE
    assert engine.window_fields(1000, None) == dict(w0=0, w1=0, e0=0, e1=0)
    T = 5 * SEG_LEN + 100
    f = engine.window_fields(T, (SEG_LEN + TILE, 2 * SEG_LEN))
    # tiles of segment 1 read its centre 1.5 SEG_LEN; the window's path range is inside
    assert f == dict(w0=SEG_LEN + TILE, w1=2 * SEG_LEN, e0=SEG_LEN + TILE, e1=2 * SEG_LEN)
    f = engine.window_fields(T, (TILE, 3 * TILE))  # centre of segment 0 lies past the window
    assert f["e0"] == TILE and f["e1"] == SEG_LEN // 2 + 1
    f = engine.window_fields(T, (6 * SEG_LEN, 0))  # tail window: held track, last segment
    assert f["e0"] == T - 1 and f["e1"] == T
    for bad in ((1, 0), (TILE, TILE), (2 * TILE, TILE), (-TILE, 0)):
        with np.testing.assert_raises(ValueError):
            engine.window_fields(T, bad)


def test_canonical_lattice_matches_enumeration():
    """The host's structural copy of the canonical order (room.py:98-143)
    equals the oracle enumeration (itself pinned to the reference goldens)."""
    from oracle import oracle as orc
    for K in (0, 1, 2, 5, 8, 20):
        j, order = parallel.canonical_lattice(K)
        im = orc.enumerate_images([5.0, 6.0, 4.0], 0.9, K)
        assert np.array_equal(j, im.j.astype(np.int64)), K
        assert np.array_equal(order, im.order.astype(np.int64)), K


def test_image_shards_partition_balance_and_locality():
    tiers = ((2, 1), (8, 32), (20, 256))
    dims = np.array([20.0, 15.0, 8.0])
    j, order = parallel.canonical_lattice(20)
    dist = np.linalg.norm(j * dims, axis=1)
    for world in (1, 2, 3, 8):
        parts = [parallel.image_shard(dims, 20, tiers, r, world) for r in range(world)]
        assert np.array_equal(np.sort(np.concatenate(parts)), np.arange(order.size))
        for lo, hi in ((-1, 2), (2, 8), (8, 20)):  # every tier balanced (cost-weighted cuts)
            cnt = [int(np.sum((order[p] > lo) & (order[p] <= hi))) for p in parts]
            n = int(np.sum((order > lo) & (order <= hi)))
            assert max(cnt) <= 1.2 * n / world + 2 and min(cnt) >= 0.7 * n / world - 2, (world, cnt)
        if world > 1:  # contiguous delay bands: rank r's far tier lies beyond rank r-1's
            far = [dist[p[order[p] > 8]] for p in parts]
            assert all(far[r].min() >= far[r - 1].max() - 1e-9 for r in range(1, world))
    sub = np.arange(0, order.size, 3)  # restricted to a subset (t60 cull)
    parts = [parallel.image_shard(dims, 20, tiers, r, 4, sub) for r in range(4)]
    assert np.array_equal(np.sort(np.concatenate(parts)), sub)
    with np.testing.assert_raises(ValueError):
        parallel.image_shard(dims, 20, tiers, 4, 4)
    # equal-cost cuts: a uniform key gives equal counts, a sparse tail a smaller last band
    assert np.diff(parallel._band_cuts(np.arange(800.0), 8)).tolist() == [100] * 8
    tail = np.concatenate([np.arange(700) * 0.01, 7.0 + np.arange(100) * 1.0])
    sizes = np.diff(parallel._band_cuts(tail, 4))
    assert sizes.sum() == 800 and sizes[-1] < sizes[0]


def test_lpt_assign_balances_and_covers():
    rng = np.random.default_rng(0)
    costs = rng.uniform(1, 2, size=256)
    parts = parallel.lpt_assign(costs, 8)
    assert sorted(i for p in parts for i in p) == list(range(256))
    loads = [costs[p].sum() for p in parts]
    assert max(loads) / min(loads) < 1.02
    assert parallel.lpt_assign([5, 1, 1], 2) == [[0], [1, 2]]


def test_shard_modes():
    assert parallel.shard_mode("c3", 8) == "images"
    assert parallel.shard_mode("c4", 8) == "scenes"
    assert parallel.shard_mode("c5", 8) == "channels"
    assert parallel.channel_shard(8, 3, 8) == [3]
    assert parallel.channel_shard(8, 1, 4) == [1, 5]
    got = sorted(c for r in range(3) for c in parallel.channel_shard(8, r, 3))
    assert got == list(range(8))
    assert parallel.shard_mode("c2", 4) == "replicas"
    assert parallel.shard_mode("c3", 1) == "single"


def _scene(images=None):
    from oracle import oracle as orc
    from paper_2508_03065_b200 import hann_sinc, workloads
    sc = workloads.make_scenes("c3", duration=0.06, max_order=5, tiers=((1, 1), (3, 32), (5, 256)))[0]
    f = hann_sinc(sc.fd_taps, 14)
    im = None
    if images is not None:
        im = orc.enumerate_images(sc.dims, sc.walls, sc.max_order).take(images)
    return orc.OracleScene(sc.s, sc.pos, sc.mics[0], sc.dims, sc.walls, sc.max_order, sc.tiers,
                           f.branches, sc.rate, images=im)


def _worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_03065_b200 import workloads
    sc = workloads.make_scenes("c3", duration=0.06, max_order=5, tiers=((1, 1), (3, 32), (5, 256)))[0]
    mine = parallel.image_shard(sc.dims, sc.max_order, sc.tiers, rank, world)
    o = _scene(mine)
    dmax = torch.tensor([o.track_max()], dtype=torch.float64)
    parallel.allreduce_max(dmax)  # batch-wide maximum -> the reference's out_len
    out_len = o.s.size + int(np.ceil(o.rate * float(dmax[0]) / o.c)) + o.L
    t = torch.from_numpy(o.render_window(0, out_len))
    parallel.reduce_to_root(t)
    if rank == 0:
        np.save(os.path.join(outdir, "reduced.npy"), t.numpy())
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_image_shards_reduce_to_full_render_gloo():
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        got = np.load(os.path.join(d, "reduced.npy"))
    full = _scene().render()
    assert got.shape == full.shape
    assert np.max(np.abs(got - full)) <= 1e-12 * np.max(np.abs(full))


def test_shard_batches_groups_are_rank_independent():
    """Sub-batch groups come from the unsharded jobs: with a
    budget that splits the batch, every rank gets the same groups even
    though the shards' own footprints differ."""
    from paper_2508_03065_b200 import workloads
    from paper_2508_03065_b200.synth import job_footprint, scene_jobs, shard_batches
    scenes = workloads.make_scenes("c5", duration=0.2, max_order=9, n_channels=4,
                                   tiers=((2, 1), (5, 32), (9, 256)))
    jobs = scene_jobs(scenes)
    budget = int(2.5 * job_footprint(jobs[0], 64))
    out = [shard_batches(jobs, (r, 3), budget, 64) for r in range(3)]
    assert all(g == out[0][0] for g, _ in out)
    assert sorted(j for g in out[0][0] for j in g) == list(range(len(jobs)))
    assert len(out[0][0]) > 1
    foot = [[job_footprint(jb, 64) for jb in sj] for _, sj in out]
    assert foot[0] != foot[1]  # the shards' own footprints are rank-specific


def test_hybrid_shards_cover_images_times_windows():
    """shard_jobs(by="hybridK"): K image bands x W/K output windows; every
    (image, output tile) pair belongs to exactly one rank."""
    from paper_2508_03065_b200 import engine, workloads
    from paper_2508_03065_b200.engine import TILE
    sc = workloads.make_scenes("c3", duration=1.0, max_order=8)[0]
    jb = engine.Job(s=sc.s, pos=sc.pos, mic=sc.mics[0], dims=sc.dims, walls=sc.walls,
                    max_order=sc.max_order, tiers=((2, 1), (5, 32), (8, 256)), rate=sc.rate)
    S = parallel.canonical_lattice(sc.max_order)[0].shape[0]
    n_tiles = 400
    for K, W in ((2, 8), (4, 8), (2, 4)):
        cover = np.zeros((S, n_tiles), np.int64)
        for r in range(W):
            (sj,) = parallel.shard_jobs([jb], r, W, f"hybrid{K}")
            w0, w1 = sj.window
            t1 = n_tiles if w1 == 0 else w1 // TILE
            cover[np.asarray(sj.image_index)[:, None], np.arange(w0 // TILE, t1)[None, :]] += 1
        assert (cover == 1).all(), (K, W)
    with np.testing.assert_raises(ValueError):
        parallel.shard_jobs([jb], 0, 6, by="hybrid4")
