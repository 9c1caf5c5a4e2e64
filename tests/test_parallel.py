"""Multi-GPU partitioning logic on CPU: image_slice / lpt_assign properties
and a world_size-2 gloo run of the image-shard + reduce path, with the CPU
oracle rendering each rank's shard (test infrastructure stands in for the
GPU renderer; the partition and the collective are the product code)."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_03065_b200 import parallel


def test_image_slices_tile_the_list():
    for n in (0, 1, 7, 11521):
        for world in (1, 2, 3, 8):
            got = [parallel.image_slice(n, r, world) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            assert max(h - l for l, h in got) - min(h - l for l, h in got) <= 1


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
    assert parallel.shard_mode("c2", 4) == "replicas"
    assert parallel.shard_mode("c3", 1) == "single"


SEG = 2048  # samples per sort segment in this test


def _scene():
    from oracle import oracle as orc
    from paper_2508_03065_b200 import hann_sinc, workloads
    sc = workloads.make_scenes("c3", duration=0.06, max_order=5, tiers=((1, 1), (3, 32), (5, 256)))[0]
    f = hann_sinc(sc.fd_taps, 14)
    return orc.OracleScene(sc.s, sc.pos, sc.mics[0], sc.dims, sc.walls, sc.max_order, sc.tiers,
                           f.branches, sc.rate)


def _segment_order(o, s):
    """Delay-sort of the images at the centre of segment s (engine rule)."""
    t = min(o.T - 1, s * SEG + SEG // 2)
    key = np.empty(len(o.images))
    for i in range(len(o.images)):
        if o.factor[i] == 1:
            d = o.images.offset[i] + o.images.sign[i] * o.pos[t] - o.mic
            key[i] = np.sqrt(d @ d)
        else:
            k = min(t // o.factor[i], o.coarse_len[i] - 1)
            key[i] = o.coarse[o.coarse_off[i] + k]
    return np.argsort(key, kind="stable")


def _worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = _scene()
    out_len = o.out_len()
    part = np.zeros(out_len)
    n_seg = -(-o.T // SEG)
    for s in range(n_seg):
        order = _segment_order(o, s)
        lo, hi = parallel.image_slice(order.size, rank, world)
        mine = np.sort(order[lo:hi])
        n0 = s * SEG
        n1 = out_len if s == n_seg - 1 else (s + 1) * SEG  # hold tail: last segment
        sub = o._struct(mine)
        import ctypes
        from oracle.oracle import lib, _p
        buf = np.empty(n1 - n0)
        lib().orc_render_window(ctypes.byref(sub), n0, n1, _p(buf), 1)
        part[n0:n1] = buf
    t = torch.from_numpy(part)
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
