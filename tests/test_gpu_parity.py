"""GPU parity: libmvb (through its C ABI) against the CPU oracle and the
golden vectors the reference produced.  Needs a B200 (marker `gpu`).

Bars (north_star): fp64 (exact engine) max |err| <= 1e-10 of the output
peak -- in practice bit-identical to the oracle; fp32 fast path <= 1e-5 of
the peak.  Integer/index work (enumeration, out_len) is exact.
"""

import numpy as np
import pytest

from conftest import golden, rel_err
from oracle import oracle as orc
from paper_2508_03065_b200 import workloads
from paper_2508_03065_b200.farrow import hann_sinc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2508_03065_b200 import engine, kernels, room as mroom  # noqa: E402
from paper_2508_03065_b200.synth import render_jobs, scene_jobs  # noqa: E402

FP32_TOL = 1e-5
FP64_TOL = 1e-10


# ---------------------------------------------------------------- operators
def test_kernel_trio_bitwise(kernels_golden):
    g = kernels_golden
    d = kernels.distance_streams(g["dist_offset"], g["dist_sign"], g["dist_mic"], g["dist_pos"])
    assert np.array_equal(d, g["dist_out"])
    out = np.zeros(g["acc_out"].size)
    kernels.accumulate_images(out, g["acc_streams"], g["acc_tau"], g["acc_amp"], 8, 3)
    assert np.array_equal(out, g["acc_out"])
    for N in (16, 64):
        up = kernels.upsample_stream(g[f"up{N}_coarse"], g[f"table{N}"], N, g[f"up{N}_out"].size)
        assert np.array_equal(up, g[f"up{N}_out"])


def test_branch_filter_matches_oracle(kernels_golden):
    g = kernels_golden
    v = kernels.branch_filter(g["acc_x"], g["design_3_8_08"])
    assert np.array_equal(v, orc.branch_filter(g["acc_x"], g["design_3_8_08"]))
    assert rel_err(v, g["acc_streams"]) < 1e-15


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_enumeration(kernels_golden, tag):
    g = kernels_golden
    t = mroom.image_table(g[f"enum_{tag}_dims"], g[f"enum_{tag}_walls"], int(g[f"enum_{tag}_order"]))
    assert np.array_equal(t.order[0].cpu().numpy(), g[f"enum_{tag}_ord"])
    assert np.array_equal(t.lattice[0].cpu().numpy(), g[f"enum_{tag}_lattice"])
    assert np.array_equal(t.parity[0].cpu().numpy(), g[f"enum_{tag}_parity"])
    assert np.array_equal(t.offset[0].cpu().numpy(), g[f"enum_{tag}_offset"])
    assert np.array_equal(t.sign[0].cpu().numpy(), g[f"enum_{tag}_sign"])
    np.testing.assert_allclose(t.beta[0].cpu().numpy(), g[f"enum_{tag}_beta"], rtol=4e-16, atol=0)


def test_enumeration_batch_and_large_order():
    rng = np.random.default_rng(0)
    dims = rng.uniform(3, 10, size=(5, 3))
    walls = rng.uniform(0.6, 0.95, size=(5, 6))
    t = mroom.image_table(dims, walls, 12)
    for r in range(5):
        im = orc.enumerate_images(dims[r], walls[r], 12)
        assert np.array_equal(t.offset[r].cpu().numpy(), im.offset)
        assert np.array_equal(t.order[r].cpu().numpy(), im.order)
        np.testing.assert_allclose(t.beta[r].cpu().numpy(), im.beta, rtol=4e-16, atol=0)
    t = mroom.image_table([20.0, 15.0, 8.0], 0.9, 40)
    im = orc.enumerate_images([20.0, 15.0, 8.0], np.full(6, 0.9), 40)
    assert np.array_equal(t.lattice[0].cpu().numpy(), im.lattice)
    assert np.array_equal(t.parity[0].cpu().numpy(), im.parity)


# ---------------------------------------------------------------- renders
CASES = {
    "c1": ("c1", dict()),
    "c1_refdesign": ("c1", dict(tiers=((1, 1), (3, 32)))),
    "c2": ("c2", dict(duration=0.25)),
    "c3": ("c3", dict(duration=0.1, max_order=8, tiers=((2, 1), (5, 32), (8, 256)))),
    "c4": ("c4", dict(duration=0.25, max_order=6, n_scenes=3)),
    "c5": ("c5", dict(duration=0.1, max_order=6, n_channels=4, tiers=((2, 1), (4, 32), (6, 256)))),
}


def _scenes(case):
    wl, over = CASES[case]
    g = golden(f"render_{case}.npz")
    scenes = workloads.make_scenes(wl, **over)
    chans = [int(c) for c in g["channels"]] if wl == "c5" else None
    return g, scenes, chans


def _filter_of(g, L):
    from paper_2508_03065_b200.farrow import FarrowFilter
    b = g["branches"]
    return FarrowFilter(b.shape[0] - 1, b.shape[1], b, (b.shape[1] - 1) // 2, 1.0)


def _oracle(scenes, chans, branches):
    ys = []
    for sc in scenes:
        for ch in (chans if chans is not None else range(len(sc.mics))):
            ys.append(orc.OracleScene(sc.s, sc.pos, sc.mics[ch], sc.dims, sc.walls, sc.max_order,
                                      sc.tiers, branches, sc.rate).render())
    return ys


@pytest.mark.parametrize("case", list(CASES))
def test_exact_engine_matches_oracle_and_reference(case):
    g, scenes, chans = _scenes(case)
    f = _filter_of(g, scenes[0].fd_taps)
    res = render_jobs(scene_jobs(scenes, chans), f, precision="fp64")
    ys = [res.job(j).cpu().numpy() for j in range(len(res.lengths))]
    assert [y.size for y in ys] == [int(v) for v in g["lens"]]
    y = np.concatenate(ys)
    assert rel_err(y, g["y"]) <= FP64_TOL
    ref = np.concatenate(_oracle(scenes, chans, g["branches"]))
    # same arithmetic and order as the oracle: bit-identical up to the last
    # ulp (the reference itself differs from both by np.convolve's summation
    # order, ~1e-15).  c4's billiard paths trigger the reference's anti-alias
    # low-pass (bandwidth 244 Hz > Nyquist_out 125 Hz), an FFT filter whose
    # cuFFT and pocketfft roundings differ by ~1e-15 m in the coarse paths.
    assert rel_err(y, ref) <= (1e-12 if case == "c4" else 1e-15)


@pytest.mark.parametrize("case", ["c2", "c3", "c4", "c5", "c1"])
def test_fast_engine_matches_oracle(case):
    g, scenes, chans = _scenes(case)
    f = _filter_of(g, scenes[0].fd_taps)
    res = render_jobs(scene_jobs(scenes, chans), f, precision="fp32")
    ys = [res.job(j).double().cpu().numpy() for j in range(len(res.lengths))]
    assert [y.size for y in ys] == [int(v) for v in g["lens"]]
    for y, ref in zip(ys, _oracle(scenes, chans, g["branches"])):
        assert rel_err(y, ref) <= FP32_TOL


def test_fast_engine_reference_design_filter():
    """The reference's own default filter design(3, 8, 0.8) on the fast
    path (Farrow M=3, 16-byte records)."""
    g, scenes, chans = _scenes("c1_refdesign")
    f = _filter_of(g, 8)
    sc = scenes[0]
    s32 = sc.s.astype(np.float32)
    res = render_jobs(scene_jobs(scenes), f, precision="fp32", signals=[s32])
    y = res.job(0).double().cpu().numpy()
    ref = orc.OracleScene(s32.astype(np.float64), sc.pos, sc.mics[0], sc.dims, sc.walls,
                          sc.max_order, sc.tiers, g["branches"], sc.rate).render()
    assert y.size == ref.size
    assert rel_err(y, ref) <= FP32_TOL


@pytest.mark.parametrize("tag", ["slow", "fast"])
def test_decimate_on_device_matches_reference(kernels_golden, tag):
    """Bandwidth decision (cuFFT + mvb_energy_index) and the anti-alias
    low-pass (trajectory.py:279-298); 'fast' triggers the low-pass."""
    from paper_2508_03065_b200.trajectory import Trajectory, bandwidth_estimate_dev, decimate
    g = kernels_golden
    pos = g[f"dec_{tag}_in"]
    tr = decimate(Trajectory(rate=1000.0, positions=pos), int(g[f"dec_{tag}_N"]))
    np.testing.assert_allclose(tr.positions, g[f"dec_{tag}_out"], rtol=0, atol=1e-12)
    bw = bandwidth_estimate_dev(torch.as_tensor(pos, device="cuda"), 1000.0)
    assert bw == orc.bandwidth_estimate(pos, 1000.0)


def test_mixed_job_groups_in_one_batch():
    """Jobs with different max_order / tiers / image subsets in one batch
    (several enumeration groups, class selections at group offsets) render
    like the oracle, each on both engines."""
    import dataclasses
    from paper_2508_03065_b200 import engine
    base = workloads.make_scenes("c2", duration=0.1)[0]
    f = hann_sinc(32, 14)
    variants = [dict(max_order=4, tiers=((1, 1), (4, 32))),
                dict(max_order=6, tiers=((2, 1), (4, 64), (6, 128))),
                dict(max_order=3, tiers=((3, 1),)),
                dict(max_order=4, tiers=((1, 1), (4, 32)), image_index=np.arange(5, 60, 3))]
    for precision, tol in (("fp64", 1e-13), ("fp32", FP32_TOL)):
        sig = base.s.astype(np.float64 if precision == "fp64" else np.float32)
        jobs = [engine.Job(s=sig, pos=base.pos, mic=base.mics[0], dims=base.dims, walls=base.walls,
                           rate=base.rate, **v) for v in variants]
        res = render_jobs(jobs, f, precision=precision)
        for j, v in enumerate(variants):
            im = orc.enumerate_images(base.dims, base.walls, v["max_order"])
            if "image_index" in v:
                im = im.take(v["image_index"])
            ref = orc.OracleScene(base.s, base.pos, base.mics[0], base.dims, base.walls,
                                  v["max_order"], v["tiers"], f.branches, base.rate,
                                  images=im).render()
            if precision == "fp32":
                ref = orc.OracleScene(sig.astype(np.float64), base.pos, base.mics[0], base.dims,
                                      base.walls, v["max_order"], v["tiers"], f.branches,
                                      base.rate, images=im).render()
            y = res.job(j).double().cpu().numpy()
            assert y.size == ref.size, (precision, j)
            assert rel_err(y, ref) <= tol, (precision, j)


def test_image_shards_sum_to_full_render():
    """Image shards (parallel.image_shard) rendered one after another on
    this GPU: per-shard track maxima -> batch-wide maximum (the value the
    all-reduce MAX produces across ranks, fed through dmax_hook) -> every
    shard writes the full out_len and the shard outputs sum to the render
    (no rank waits on another: the shards run sequentially)."""
    import dataclasses
    from paper_2508_03065_b200 import engine, parallel
    g, scenes, chans = _scenes("c5")
    f = _filter_of(g, scenes[0].fd_taps)
    jobs = scene_jobs(scenes, chans)
    world = 3
    full = render_jobs(jobs, f, precision="fp32")
    local = []
    for r in range(world):
        local.append(engine.Geometry(parallel.shard_jobs(jobs, r, world)).dmax)
    gmax = np.max(np.stack(local), axis=0)

    def hook(t):
        t.copy_(torch.as_tensor(gmax, device=t.device))

    parts = [render_jobs(jobs, f, precision="fp32", shard=(r, world), dmax_hook=hook)
             for r in range(world)]
    assert all(np.array_equal(p.lengths, full.lengths) for p in parts)
    assert sum(p.updates for p in parts) == full.updates
    total = np.concatenate([sum(p.job(j).double() for p in parts).cpu().numpy()
                            for j in range(len(jobs))])
    ref = np.concatenate(_oracle(scenes, chans, g["branches"]))
    assert rel_err(total, ref) <= FP32_TOL
    with pytest.raises(ValueError):
        render_jobs(jobs, f, precision="fp64", shard=(0, 2))


def _time_shard_case(case):
    if case == "c3long":  # several sort segments and exact-maximum chunks
        scenes = workloads.make_scenes("c3", duration=1.0, max_order=8,
                                       tiers=((2, 1), (5, 32), (8, 256)))
        return None, scenes, None, hann_sinc(scenes[0].fd_taps, 14)
    g, scenes, chans = _scenes(case)
    return g, scenes, chans, _filter_of(g, scenes[0].fd_taps)


@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("case", ["c5", "c3long"])
def test_time_shards_sum_to_full_render(case, world):
    """Time shards (parallel.time_window): every rank renders its output
    window from all images.  The window maxima, MAX-reduced (the all-reduce
    the ranks issue; here through dmax_hook, shards in sequence on one GPU),
    equal the unsharded exact maximum bit for bit; each rank's output is
    zero outside its window; the windows cover the output; the ranks'
    outputs sum to the full render (fp32 summation-order differences only)
    and, for c5, to the oracle within the fp32 bar."""
    from paper_2508_03065_b200 import parallel
    g, scenes, chans, f = _time_shard_case(case)
    jobs = scene_jobs(scenes, chans)
    full_geom = engine.Geometry(jobs)
    full = render_jobs(jobs, f, precision="fp32")
    shards = [parallel.shard_jobs(jobs, r, world, "time") for r in range(world)]
    gmax = np.max(np.stack([engine.Geometry(sj).dmax for sj in shards]), axis=0)
    assert np.array_equal(gmax, full_geom.dmax)

    def hook(t):
        t.copy_(torch.as_tensor(gmax, device=t.device))

    parts = [render_jobs(jobs, f, precision="fp32", shard=(r, world, "time"), dmax_hook=hook)
             for r in range(world)]
    for j in range(len(jobs)):
        n = int(full.lengths[j])
        assert all(int(p.lengths[j]) == n for p in parts)
        cover = np.zeros(n, np.int64)
        for r, p in enumerate(parts):
            w0, w1 = shards[r][j].window
            w1 = n if w1 == 0 else min(w1, n)
            y = p.job(j).double().cpu().numpy()
            assert not y[:w0].any() and not y[w1:].any(), (r, j)
            cover[w0:w1] += 1
        assert (cover == 1).all(), j
        total = sum(p.job(j).double() for p in parts).cpu().numpy()
        ref = full.job(j).double().cpu().numpy()
        assert rel_err(total, ref) <= 1e-6, (j, rel_err(total, ref))
    if g is not None:
        total = np.concatenate([sum(p.job(j).double() for p in parts).cpu().numpy()
                                for j in range(len(jobs))])
        assert rel_err(total, np.concatenate(_oracle(scenes, chans, g["branches"]))) <= FP32_TOL


def test_render_plan_time_shards():
    """Time-sharded render plans: captured windows replay; the ranks'
    replays sum to the full render, data changing between runs."""
    import dataclasses
    from paper_2508_03065_b200 import parallel
    from paper_2508_03065_b200.plan import RenderPlan
    _, scenes, _, f = _time_shard_case("c3long")
    jobs = scene_jobs(scenes)
    world = 3
    plans = None
    for it in range(4):
        jb = [dataclasses.replace(j, pos=scenes[0].pos + 0.05 * it,
                                  s=(scenes[0].s * (1 + it)).astype(np.float32)) for j in jobs]
        gmax = np.max(np.stack([engine.Geometry(parallel.shard_jobs(jb, r, world, "time")).dmax
                                for r in range(world)]), axis=0)

        def hook(t, gmax=gmax):
            t.copy_(torch.as_tensor(gmax, device=t.device))

        if plans is None:
            hooks = {"h": hook}
            plans = [RenderPlan(jobs, f, shard=(r, world, "time"),
                                dmax_hook=lambda t: hooks["h"](t)) for r in range(world)]
        hooks["h"] = hook
        parts = [p.run(jb) for p in plans]
        full = render_jobs(jb, f)
        total = sum(p.job(0).double() for p in parts).cpu().numpy()
        ref = full.job(0).double().cpu().numpy()
        assert np.array_equal(parts[0].lengths, full.lengths)
        assert rel_err(total, ref) <= 1e-6, (it, rel_err(total, ref))
    assert all(p.captures == 2 for p in plans)


def test_memory_split_batches_match_single_batch():
    """A batch forced into sub-batches (max_batch_bytes) renders the same
    lengths and, within the fp32 bar, the same outputs as one batch."""
    from paper_2508_03065_b200.synth import job_footprint
    scenes = workloads.make_scenes("c4", duration=0.25, max_order=6, n_scenes=5)
    f = hann_sinc(32, 14)
    jobs = scene_jobs(scenes)
    whole = render_jobs(jobs, f)
    split = render_jobs(jobs, f, max_batch_bytes=2 * max(job_footprint(j, 32) for j in jobs))
    assert np.array_equal(whole.lengths, split.lengths)
    assert whole.updates == split.updates
    for j in range(len(jobs)):
        a = whole.job(j).double().cpu().numpy()
        b = split.job(j).double().cpu().numpy()
        assert np.max(np.abs(a - b)) <= 1e-6 * np.max(np.abs(a))


def test_render_plan_replays_match_direct_renders():
    """CUDA-graph render plans (plan.RenderPlan): replays equal direct
    renders bit for bit, follow new inputs (signals, paths), alternate
    their two slots, and re-capture when new data exceed the captured
    output capacity."""
    import dataclasses
    from paper_2508_03065_b200.plan import RenderPlan
    scenes = workloads.make_scenes("c5", duration=0.05, max_order=6, n_channels=3,
                                   tiers=((2, 1), (4, 32), (6, 256)))
    f = hann_sinc(64, 14)
    jobs = scene_jobs(scenes)
    plan = RenderPlan(jobs, f)
    rng = np.random.default_rng(3)
    for it in range(4):
        s = (scenes[0].s * (1.0 + it)).astype(np.float32)
        pos = scenes[0].pos + 0.01 * it
        jb = [dataclasses.replace(j, s=s, pos=pos) for j in jobs]
        got = plan.run(jb)
        ref = render_jobs(jb, f)
        assert np.array_equal(got.lengths, ref.lengths)
        for j in range(len(jb)):
            assert torch.equal(got.job(j), ref.job(j)), (it, j)
    assert plan.captures == 2  # one per slot
    # a source path pushed far away exceeds the captured capacity: re-capture
    far = scenes[0].pos + np.array([30.0, 0.0, 0.0])
    jb = [dataclasses.replace(j, pos=far) for j in jobs]
    got = plan.run(jb)
    ref = render_jobs(jb, f)
    # the slot replayed speculatively; on first use of the result the
    # readbacks show the overflow: one miss, the run re-captured
    assert plan.captures == 2 and plan.misses == 0  # validation is deferred
    assert np.array_equal(got.lengths, ref.lengths)
    assert plan.captures == 3 and plan.misses == 1
    assert torch.equal(got.job(0), ref.job(0))
    with pytest.raises(ValueError):
        plan.run(jobs[:1])
    # jobs without explicit keys: fresh arrays each run, same sharing pattern
    anon = [dataclasses.replace(j, path_key=None, signal_key=None, pos=scenes[0].pos.copy(),
                                s=scenes[0].s.astype(np.float32)) for j in jobs[:1]]
    plan1 = RenderPlan(anon, f)
    for it in range(3):
        jb = [dataclasses.replace(anon[0], pos=scenes[0].pos + 0.001 * it,
                                  s=(scenes[0].s * (it + 1)).astype(np.float32))]
        assert torch.equal(plan1.run(jb).job(0), render_jobs(jb, f).job(0))


def test_render_plan_full_rate_paths_change():
    """A plan whose images are all full-rate bounds them from the path boxes
    inside its graph: the boxes of each run (not the capture's) must be
    used -- paths move between runs without re-capturing, lengths and
    outputs equal direct renders bit for bit (fp64 and fp32)."""
    import dataclasses
    from paper_2508_03065_b200.plan import RenderPlan
    sc = workloads.make_scenes("c1", duration=0.1)[0]
    f = hann_sinc(32, 14)
    for prec in ("fp64", "fp32"):
        s = sc.s.astype(np.float64 if prec == "fp64" else np.float32)
        job = engine.Job(s=s, pos=sc.pos, mic=sc.mics[0], dims=sc.dims, walls=sc.walls,
                         max_order=2, tiers=((2, 1),), rate=sc.rate)
        plan = RenderPlan([job], f, precision=prec)
        for it, shift in enumerate((0.0, 0.25, -0.3, 0.4, 0.1)):
            jb = [dataclasses.replace(job, pos=sc.pos + np.array([shift, -0.5 * shift, 0.0]))]
            got, ref = plan.run(jb), render_jobs(jb, f, precision=prec)
            assert np.array_equal(got.lengths, ref.lengths), (prec, it)
            assert torch.equal(got.job(0), ref.job(0)), (prec, it)
        assert plan.captures == 2, plan.captures  # one per slot: the moves stayed in capacity


def test_render_plan_lowpass_decision_change():
    """A speculative replay whose staging shows a changed anti-alias
    decision (trajectory.py:279-298: low-pass only when Nyquist_out <
    bandwidth < 2 Nyquist_out) is redone with a re-captured graph: the path
    oscillates below the decimated tier's output Nyquist in one run and
    between one and two Nyquist in the next; both equal direct renders."""
    import dataclasses
    from paper_2508_03065_b200.plan import RenderPlan
    rate, T, N = 16000.0, 8000, 64  # tier output Nyquist: 125 Hz
    t = np.arange(T) / rate
    dims = np.array([6.0, 5.0, 3.0])

    def path(freq):
        return np.stack([3.0 + 0.02 * np.sin(2 * np.pi * freq * t), 2.5 + 0.0 * t,
                         1.5 + 0.0 * t], axis=1)

    x = np.random.default_rng(4).standard_normal(T).astype(np.float32)
    job = engine.Job(s=x, pos=path(40.0), mic=np.array([1.0, 1.2, 1.1]), dims=dims, walls=0.8,
                     max_order=3, tiers=((1, 1), (3, N)), rate=rate)
    f = hann_sinc(32, 14)
    plan = RenderPlan([job], f)
    decisions = []
    for freq in (40.0, 40.0, 40.0, 180.0, 180.0, 40.0):
        jb = [dataclasses.replace(job, pos=path(freq))]
        got, ref = plan.run(jb), render_jobs(jb, f)
        geom = engine.Geometry(jb)
        decisions.append(any(len(d) for d in geom.lowpass_decision()))
        assert np.array_equal(got.lengths, ref.lengths), freq
        assert torch.equal(got.job(0), ref.job(0)), freq
    assert decisions == [False, False, False, True, True, False], decisions
    assert plan.misses >= 2  # 40 -> 180 Hz and back, on a captured slot


def test_render_plan_image_shards():
    """Sharded plans: geometry graph, eager dmax hook, render graph; the
    shards' replays sum to the full render (shards in sequence on one GPU)."""
    from paper_2508_03065_b200 import engine, parallel
    from paper_2508_03065_b200.plan import RenderPlan
    import dataclasses
    g, scenes, chans = _scenes("c5")
    f = _filter_of(g, scenes[0].fd_taps)
    jobs = scene_jobs(scenes, chans)
    world = 2
    local = []
    for r in range(world):
        local.append(engine.Geometry(parallel.shard_jobs(jobs, r, world)).dmax)
    gmax = np.max(np.stack(local), axis=0)

    def hook(t):
        t.copy_(torch.as_tensor(gmax, device=t.device))

    plans = [RenderPlan(jobs, f, shard=(r, world), dmax_hook=hook) for r in range(world)]
    for _ in range(3):  # capture, then replays on both slots
        parts = [p.run(jobs) for p in plans]
        total = np.concatenate([sum(p.job(j).double() for p in parts).cpu().numpy()
                                for j in range(len(jobs))])
        ref = np.concatenate(_oracle(scenes, chans, g["branches"]))
        assert rel_err(total, ref) <= FP32_TOL


def test_fraction_table_gather_ab_matches_oracle(monkeypatch):
    """The SURVEY H2 A/B kernel (literal per-fraction table, linear in mu,
    direct L-tap gather; measurement only) renders the same scene within the
    fp32 bar -- so the A/B compares two correct kernels."""
    from paper_2508_03065_b200 import engine
    monkeypatch.setattr(engine, "FD_GATHER", "table")
    sc = workloads.make_scenes("c3", duration=0.05, max_order=6, tiers=((2, 1), (4, 32), (6, 256)))[0]
    f = hann_sinc(sc.fd_taps, 14)
    y = render_jobs(scene_jobs([sc]), f).job(0).double().cpu().numpy()
    ref = orc.OracleScene(sc.s, sc.pos, sc.mics[0], sc.dims, sc.walls, sc.max_order, sc.tiers,
                          f.branches, sc.rate).render()
    assert y.size == ref.size
    assert rel_err(y, ref) <= 1e-5


@pytest.mark.parametrize("case", ["c2", "c3", "c4", "c5", "c3long"])
def test_active_ranges_bit_identical(case, monkeypatch):
    """Per-tile active image ranges (mvb_synthesize_f32_ranged, the default)
    skip only images that read nothing but zero pads over a tile: the
    output equals the walk over every image of the chunk bit for bit --
    unsharded, and for time shards (sorted runs, windows) of c3long."""
    if case == "c3long":
        g, scenes, chans, f = _time_shard_case(case)
        shards = [(r, 3, "time") for r in range(3)]
    else:
        g, scenes, chans = _scenes(case)
        f = _filter_of(g, scenes[0].fd_taps)
        shards = [None]
    jobs = scene_jobs(scenes, chans)
    for shard in shards:
        kw = {}
        if shard is not None:
            from paper_2508_03065_b200 import parallel
            gmax = np.max(np.stack([engine.Geometry(parallel.shard_jobs(jobs, r, 3, "time")).dmax
                                    for r in range(3)]), axis=0)
            kw = dict(shard=shard, dmax_hook=lambda t: t.copy_(torch.as_tensor(gmax, device=t.device)))
        outs = []
        for on in (False, True):
            monkeypatch.setattr(engine, "ACTIVE_RANGES", on)
            res = render_jobs(jobs, f, precision="fp32", **kw)
            outs.append(torch.cat([res.job(j) for j in range(len(jobs))]))
        assert torch.equal(outs[0], outs[1]), (case, shard)


@pytest.mark.parametrize("budget", [1, 60_000])
def test_record_groups_bit_identical(budget, monkeypatch):
    """Batches whose interval records exceed RECORD_BUDGET compute them group
    by group into two alternating buffers inside the synthesis launch: the
    output equals the all-at-once render bit for bit (direct render and a
    render plan's replays), and the oracle within the fp32 bar."""
    g, scenes, chans = _scenes("c4")
    f = _filter_of(g, scenes[0].fd_taps)
    jobs = scene_jobs(scenes, chans)
    ref = render_jobs(jobs, f, precision="fp32")
    refs = [ref.job(j).clone() for j in range(len(jobs))]
    monkeypatch.setattr(engine, "RECORD_BUDGET", float(budget))
    geom = engine.Geometry(jobs)
    groups = engine._record_groups(geom)
    assert groups and len(groups) >= 2 and groups[0][0] == 0 and groups[-1][1] == len(jobs)
    res = render_jobs(jobs, f, precision="fp32")
    for j in range(len(jobs)):
        assert torch.equal(res.job(j), refs[j]), j
    from paper_2508_03065_b200.plan import RenderPlan
    plan = RenderPlan(jobs, f, precision="fp32")
    for _ in range(3):
        r = plan.run(jobs)
        for j in range(len(jobs)):
            assert torch.equal(r.job(j), refs[j]), j
    ys = [refs[j].double().cpu().numpy() for j in range(len(jobs))]
    for y, o in zip(ys, _oracle(scenes, chans, g["branches"])):
        assert rel_err(y, o) <= FP32_TOL


@pytest.mark.parametrize("mode", [1, 2])
def test_texture_gather_variant_bit_identical(mode, monkeypatch):
    """The measurement variant that fetches the branch-record rows through
    the texture pipe (mvb_synthesize_f32_tex; DESIGN 5.3) evaluates the same
    rows with the same Horner: bit-identical to the LDG.256 product path."""
    g, scenes, chans = _scenes("c3")
    f = _filter_of(g, scenes[0].fd_taps)
    jobs = scene_jobs(scenes, chans)
    base = render_jobs(jobs, f, precision="fp32")
    ref = torch.cat([base.job(j) for j in range(len(jobs))])
    monkeypatch.setattr(engine, "TEX_GATHER", mode)
    res = render_jobs(jobs, f, precision="fp32")
    assert torch.equal(torch.cat([res.job(j) for j in range(len(jobs))]), ref)
