"""The drop-in API on the GPU, checked the way the reference checks itself
(reference pkg/tests/test_synth.py, test_reference.py) and against the CPU
oracle.  Marker `gpu`."""

import numpy as np
import pytest

from conftest import golden, rel_err
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2508_03065_b200 as mvb  # noqa: E402
from paper_2508_03065_b200.farrow import FarrowFilter  # noqa: E402

RATE = 16000.0
ROOM = mvb.Room(dims=np.array([5.0, 6.0, 4.0]), wall_reflection=np.full(6, 0.9))
MIC = np.array([1.25, 2.6, 2.75])


def design_filter():
    """The reference's default design(3, 8, 0.8), from the golden file."""
    b = golden("kernels.npz")["design_3_8_08"]
    return FarrowFilter(3, 8, b, 3, 0.8)


def sine(freq, n):
    return np.sin(2 * np.pi * freq * np.arange(n) / RATE)


def moving(n, seed=3):
    """Sine-like path inside ROOM (the reference tests use generate('sine'))."""
    t = np.arange(n) / RATE
    rng = np.random.default_rng(seed)
    d = rng.normal(size=3)
    d /= np.linalg.norm(d)
    amp = 1.0 / (2 * np.pi * 2.0)
    return mvb.Trajectory(rate=RATE, positions=ROOM.dims / 2 + amp * np.sin(2 * np.pi * 2.0 * t)[:, None] * d)


def static(pos, n):
    return mvb.Trajectory(rate=RATE, positions=np.tile(np.asarray(pos, float), (n, 1)))


def oracle_render(s, traj, mic, f, cfg, images=None):
    o = orc.OracleScene(np.asarray(s, np.float64), traj.positions, mic, ROOM.dims,
                        ROOM.wall_reflection, cfg.max_order, cfg.tier_table(), f.branches,
                        cfg.audio_rate, cfg.sound_speed, cfg.d_min,
                        images=None if images is None else orc.enumerate_images(
                            ROOM.dims, ROOM.wall_reflection, cfg.max_order).take(images))
    return o.render()


def test_output_length_formula():
    f = design_filter()
    n = 4000
    tr = static([0.8, 4.1, 2.75], n)
    cfg = mvb.SynthesisConfig(max_order=1, decimation=1)
    st = mvb.prepare_streams(tr, ROOM, MIC, cfg)
    y = mvb.synthesize(sine(440.0, n), st, f, cfg)
    tau_max = RATE * float(st.d.max()) / cfg.sound_speed
    assert y.size == n + int(np.ceil(tau_max)) + f.branch_len


def test_direct_path_is_scaled_delay():
    f = mvb.hann_sinc(32, 14)
    n = 4000
    src = np.array([2.0, 3.5, 2.0])
    cfg = mvb.SynthesisConfig(max_order=0, decimation=1)
    for x in (sine(750.0, n), sine(750.0, n).astype(np.float32)):  # exact and fast engines
        y = mvb.render(x, static(src, n), ROOM, MIC, f, cfg)
        d = float(np.linalg.norm(src - MIC))
        ref = np.sin(2 * np.pi * 750.0 * (np.arange(y.size) / RATE - d / 343.0)) / (4 * np.pi * d)
        err = y[200:n - 200] - ref[200:n - 200]
        snr = 10 * np.log10(np.sum(ref[200:n - 200] ** 2) / np.sum(err ** 2))
        assert snr >= 60.0


def test_linearity_and_superposition():
    f = design_filter()
    n = 2000
    tr = moving(n)
    rng = np.random.default_rng(1)
    x = rng.standard_normal(n)
    cfg = mvb.SynthesisConfig(max_order=2, decimation=1)
    y1 = mvb.render(x, tr, ROOM, MIC, f, cfg)
    y3 = mvb.render(3.0 * x, tr, ROOM, MIC, f, cfg)
    assert np.allclose(y3, 3.0 * y1, rtol=1e-12, atol=1e-14)
    images = mvb.enumerate_images(ROOM, 2)
    half = len(images) // 2
    full = mvb.synthesize(x, mvb.prepare_streams(tr, ROOM, MIC, cfg, images=images), f, cfg)
    a = mvb.synthesize(x, mvb.prepare_streams(tr, ROOM, MIC, cfg, images=images[:half]), f, cfg)
    b = mvb.synthesize(x, mvb.prepare_streams(tr, ROOM, MIC, cfg, images=images[half:]), f, cfg)
    m = min(full.size, a.size, b.size)
    assert np.max(np.abs(full[:m] - (a[:m] + b[:m]))) <= 1e-10 * max(1.0, np.max(np.abs(full)))
    # image subsets render like the oracle restricted to the same images
    ref = oracle_render(x, tr, MIC, f, cfg, images=np.arange(half))
    assert rel_err(a, ref) <= 1e-15


def test_repeat_runs_identical_both_engines():
    f = mvb.hann_sinc(32, 14)
    n = 4000
    tr = moving(n)
    cfg = mvb.SynthesisConfig(max_order=3, order_split=1, decimation=64)
    x = sine(640.0, n)
    assert np.array_equal(mvb.render(x, tr, ROOM, MIC, f, cfg), mvb.render(x, tr, ROOM, MIC, f, cfg))
    x32 = x.astype(np.float32)
    assert np.array_equal(mvb.render(x32, tr, ROOM, MIC, f, cfg),
                          mvb.render(x32, tr, ROOM, MIC, f, cfg))


def test_reference_default_config_generic_factor():
    """SynthesisConfig() defaults: order_split 1, decimation 3200 (not a
    power of two: the fast engine's generic interval path)."""
    f = design_filter()
    n = 16000
    tr = moving(n, seed=5)
    cfg = mvb.SynthesisConfig()
    rng = np.random.default_rng(2)
    x = rng.standard_normal(n)
    ref = oracle_render(x, tr, MIC, f, cfg)
    y64 = mvb.render(x, tr, ROOM, MIC, f, cfg)
    assert y64.size == ref.size and rel_err(y64, ref) <= 1e-13
    y32 = mvb.render(x.astype(np.float32), tr, ROOM, MIC, f, cfg)
    ref32 = oracle_render(x.astype(np.float32), tr, MIC, f, cfg)
    assert rel_err(y32, ref32) <= 1e-5


def test_signal_longer_and_shorter_than_trajectory():
    f = mvb.hann_sinc(32, 14)
    tr = moving(3000)
    cfg = mvb.SynthesisConfig(max_order=3, order_split=1, decimation=32)
    rng = np.random.default_rng(4)
    for n in (1000, 5000):
        x = rng.standard_normal(n)
        y = mvb.render(x, tr, ROOM, MIC, f, cfg)
        ref = oracle_render(x, tr, MIC, f, cfg)
        assert y.size == ref.size and rel_err(y, ref) <= 1e-13
        y32 = mvb.render(x.astype(np.float32), tr, ROOM, MIC, f, cfg)
        ref32 = oracle_render(x.astype(np.float32), tr, MIC, f, cfg)
        assert rel_err(y32, ref32) <= 1e-5


def test_t60_cull_and_tracks():
    tr = static([2.0, 3.0, 2.0], 500)
    cut = mvb.SynthesisConfig(max_order=3, decimation=1, t60=0.02)
    st = mvb.prepare_streams(tr, ROOM, MIC, cut)
    full = mvb.prepare_streams(tr, ROOM, MIC, mvb.SynthesisConfig(max_order=3, decimation=1))
    assert 0 < st.image_count() < full.image_count()
    assert np.all(st.d[:, 0] <= 343.0 * 0.02 + 1e-12)


def test_delay_streams_tracks_match_reference_kernels():
    """DelayStreams.d (GPU) equals the oracle's low/high-order tracks."""
    tr = moving(6000)
    cfg = mvb.SynthesisConfig(max_order=3, order_split=1, decimation=64)
    st = mvb.prepare_streams(tr, ROOM, MIC, cfg)
    im = orc.enumerate_images(ROOM.dims, ROOM.wall_reflection, 3)
    low = im.order <= 1
    exact = orc.distance_streams(im.offset, im.sign, MIC, tr.positions)
    assert np.array_equal(st.d[low], exact[low])
    coarse = orc.distance_streams(im.offset[~low], im.sign[~low], MIC,
                                  orc.decimate_positions(tr.positions, RATE, 64))
    tab = orc.phase_table(64)
    up = np.stack([orc.upsample_stream(c, tab, 64, len(tr)) for c in coarse])
    assert np.array_equal(st.d[~low], up)
    assert st.eval_count == int(low.sum()) * len(tr) + int((~low).sum()) * coarse.shape[1]


def test_full_rate_oracle_and_budget():
    f = design_filter()
    n = 3000
    tr = moving(n)
    cfg = mvb.SynthesisConfig(max_order=2, decimation=3200)
    x = np.random.default_rng(6).standard_normal(n)
    y = mvb.full_rate_moving_oracle(x, tr, ROOM, MIC, f, cfg)
    y1 = mvb.render(x, tr, ROOM, MIC, f, mvb.SynthesisConfig(max_order=2, order_split=2))
    assert np.array_equal(y, y1)
    with pytest.raises(mvb.BudgetError):
        mvb.full_rate_moving_oracle(x, tr, ROOM, MIC, f,
                                    mvb.SynthesisConfig(max_order=2, eval_budget=10.0))


def test_validation_errors():
    f = design_filter()
    tr = static([2.0, 3.0, 2.0], 100)
    cfg = mvb.SynthesisConfig(max_order=0, decimation=1)
    st = mvb.prepare_streams(tr, ROOM, MIC, cfg)
    with pytest.raises(ValueError):
        mvb.synthesize(np.array([]), st, f, cfg)
    bad = np.ones(100)
    bad[5] = np.inf
    with pytest.raises(ValueError):
        mvb.synthesize(bad, st, f, cfg)
    with pytest.raises(ValueError):
        mvb.prepare_streams(mvb.Trajectory(rate=8000.0, positions=tr.positions), ROOM, MIC, cfg)
    with pytest.raises(ValueError):
        mvb.prepare_streams(tr, ROOM, [7.0, 3.0, 2.0], cfg)


def test_moving_receiver_exact_engine():
    """A (T,3) receiver path: exact fp64 engine vs the oracle."""
    n = 3000
    tr = moving(n)
    t = np.arange(n) / RATE
    mic_path = MIC[None, :] + np.stack([0.2 * t, 0 * t, 0 * t], axis=1)
    f = mvb.hann_sinc(32, 14)
    cfg = mvb.SynthesisConfig(max_order=3, tiers=((1, 1), (3, 32)))
    x = np.random.default_rng(8).standard_normal(n)
    y = mvb.render(x, tr, ROOM, mic_path, f, cfg)
    ref = oracle_render(x, tr, mic_path, f, cfg)
    assert y.size == ref.size and rel_err(y, ref) <= 1e-13


def test_source_modulation_matches_reference_golden():
    """modulate='source' (synth.py:228-242) against the reference's own
    output (tests/golden/render_c1_source.npz), and close to receiver
    modulation for slow motion (reference test_synth.py:263-277)."""
    from paper_2508_03065_b200 import workloads
    g = golden("render_c1_source.npz")
    sc = workloads.make_scenes("c1", duration=0.25, tiers=((1, 1), (3, 32)))[0]
    f = FarrowFilter(3, 8, g["branches"], 3, 0.8)
    room = mvb.Room(dims=sc.dims, wall_reflection=sc.walls)
    tr = mvb.Trajectory(rate=sc.rate, positions=sc.pos)
    cfg = mvb.SynthesisConfig(audio_rate=sc.rate, max_order=sc.max_order, tiers=sc.tiers,
                              modulate="source")
    y = mvb.render(sc.s, tr, room, sc.mics[0], f, cfg)
    assert y.size == g["y"].size
    assert rel_err(y, g["y"]) <= 1e-12
    from dataclasses import replace
    y_rx = mvb.render(sc.s, tr, room, sc.mics[0], f, replace(cfg, modulate="receiver"))
    m = min(y.size, y_rx.size)
    err = y[200:m - 200] - y_rx[200:m - 200]
    assert 10 * np.log10(np.sum(y_rx[200:m - 200] ** 2) / np.sum(err ** 2)) >= 30.0


@pytest.mark.parametrize("case", ["single_position", "single_sample_signal", "order0_fast",
                                  "factor_exceeds_T", "odd_factor_fast", "short_signal"])
def test_edge_cases_match_oracle(case):
    """Degenerate sizes the reference accepts: T = 1, len(s) = 1, no
    reflections, N > T (one coarse sample), odd N on the fast engine, a
    signal shorter than the filter."""
    f = mvb.hann_sinc(32, 14)
    rng = np.random.default_rng(11)
    n, T = 2000, 2000
    cfg = mvb.SynthesisConfig(max_order=3, order_split=1, decimation=32)
    if case == "single_position":
        T = 1
    elif case == "single_sample_signal":
        n = 1
    elif case == "order0_fast":
        cfg = mvb.SynthesisConfig(max_order=0, decimation=1)
    elif case == "factor_exceeds_T":
        T = 100
        cfg = mvb.SynthesisConfig(max_order=3, order_split=1, decimation=256)
    elif case == "odd_factor_fast":
        cfg = mvb.SynthesisConfig(max_order=4, order_split=1, decimation=37)
    elif case == "short_signal":
        n = 20
    tr = moving(T) if T > 1 else static([2.0, 3.0, 2.0], 1)
    x = rng.standard_normal(n)
    # fp64: 1e-13 of the peak; 1e-12 when decimate()'s anti-alias low-pass runs
    # (odd_factor_fast: the path's bandwidth falls in (Nyquist_out, 2 Nyquist_out)):
    # libmvb's FFT and the oracle's pocketfft round differently (~1e-15 m in the
    # coarse path), still far inside the north_star's 1e-10 fp64 bar
    tol64 = 1e-12 if case == "odd_factor_fast" else 1e-13
    for xx, tol in ((x, tol64), (x.astype(np.float32), 1e-5)):
        y = mvb.render(xx, tr, ROOM, MIC, f, cfg)
        ref = oracle_render(np.asarray(xx, np.float64), tr, MIC, f, cfg)
        assert y.size == ref.size, case
        assert rel_err(y, ref) <= tol, case


def test_render_reuses_a_plan_for_repeated_structure():
    """render() replays a cached RenderPlan from the second repeat of a
    structure on: outputs equal the direct path bit for bit; a different
    structure or MVB_PLAN_CACHE=0 renders directly."""
    import os
    from paper_2508_03065_b200 import synth
    f = design_filter()
    n = 3000
    tr = moving(n)
    cfg = mvb.SynthesisConfig(max_order=4, order_split=1, decimation=32)
    synth.release_plans()
    ys = [mvb.render(sine(300.0 * (k + 1), n).astype(np.float32), tr, ROOM, MIC, f, cfg)
          for k in range(4)]
    assert len(synth._PLANS) == 1
    os.environ["MVB_PLAN_CACHE"] = "0"
    try:
        direct = [mvb.render(sine(300.0 * (k + 1), n).astype(np.float32), tr, ROOM, MIC, f, cfg)
                  for k in range(4)]
    finally:
        del os.environ["MVB_PLAN_CACHE"]
    for a, b in zip(ys, direct):
        assert np.array_equal(a, b)
    # exact engine through a plan: still bit-identical to the oracle path
    x = sine(700.0, n)
    y64 = [mvb.render(x, tr, ROOM, MIC, f, cfg) for _ in range(3)]
    assert all(np.array_equal(y64[0], y) for y in y64[1:])
    synth.release_plans()
    assert not synth._PLANS


def test_copy_batch_pinned_pageable_and_device():
    """mvb_copy_batch (batched input staging): page-locked sources are
    copied, pageable ones skipped when require_pinned (the caller stages
    them), device-to-device entries copied without the requirement."""
    from paper_2508_03065_b200._staging import copy_batch
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(5)
    pinned = torch.empty(1000, dtype=torch.float64, pin_memory=True).numpy()
    pinned[:] = rng.normal(size=1000)
    pageable = rng.normal(size=700)
    empty = np.zeros(0)
    d1 = torch.zeros(1000, dtype=torch.float64, device=dev)
    d2 = torch.zeros(700, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    issued = copy_batch([(d1.data_ptr(), pinned.ctypes.data, pinned.nbytes),
                         (d2.data_ptr(), pageable.ctypes.data, pageable.nbytes),
                         (d2.data_ptr(), empty.ctypes.data, 0)], st, require_pinned=True)
    torch.cuda.synchronize()
    assert issued.tolist() == [True, False, True]
    assert np.array_equal(d1.cpu().numpy(), pinned)
    assert not d2.any()
    d3 = torch.empty(1000, dtype=torch.float64, device=dev)
    issued = copy_batch([(d3.data_ptr(), d1.data_ptr(), 8 * 1000)], st, require_pinned=False)
    torch.cuda.synchronize()
    assert issued.tolist() == [True] and torch.equal(d3, d1)
