"""Reference API around the render path on the GPU: the stream builders
(reference synth.py:122-179), the Farrow single-stream operators
(farrow.py:214-274) and bandwidth_estimate (trajectory.py:316-339),
checked the way the reference's own tests check them (pkg/tests/
test_synth.py:65-133, test_farrow.py:145-233, test_trajectory.py) and against
the CPU oracle and the reference goldens.  Marker `gpu`."""

import numpy as np
import pytest

from conftest import golden, rel_err
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2508_03065_b200 as mvb  # noqa: E402
from paper_2508_03065_b200 import farrow, synth, trajectory, workloads  # noqa: E402
from paper_2508_03065_b200.farrow import FarrowFilter  # noqa: E402
from paper_2508_03065_b200.room import as_arrays  # noqa: E402

ROOM = mvb.Room(dims=np.array([5.0, 6.0, 4.0]), wall_reflection=np.full(6, 0.9))
MIC = mvb.MicPosition(pos=np.array([1.25, 2.6, 2.75]))


def design_filter():
    return FarrowFilter(3, 8, golden("kernels.npz")["design_3_8_08"], 3, 0.8)


def moving_traj(n, duration, seed=5):
    rate = n / duration
    t = np.arange(n) / rate
    d = np.random.default_rng(seed).normal(size=3)
    d /= np.linalg.norm(d)
    pos = ROOM.dims / 2 + 0.3 * np.sin(2 * np.pi * 0.7 * t)[:, None] * d
    return mvb.Trajectory(rate=rate, positions=pos)


def sine(freq, dur, rate):
    return np.sin(2 * np.pi * freq * np.arange(int(dur * rate)) / rate)


def snr_db(a, ref):
    return 10 * np.log10(np.sum(ref ** 2) / np.sum((a - ref) ** 2))


# ------------------------------------------------------------ stream builders
def test_low_order_matches_oracle_and_direct_norm():
    tr = moving_traj(8000, 0.5)
    images = mvb.enumerate_images(ROOM, 1)
    st = synth.low_order_distances(images, tr, MIC, ROOM)
    assert st.d.shape == (len(images), len(tr))
    offset, sign, _, _ = as_arrays(images, ROOM)
    assert np.array_equal(st.d, orc.distance_streams(offset, sign, MIC.pos, tr.positions))
    for i in range(len(images)):
        want = np.linalg.norm(offset[i] + sign[i] * tr.positions - MIC.pos, axis=1)
        assert np.allclose(st.d[i], want, atol=1e-12)
    assert st.eval_count == st.d.size
    empty = synth.low_order_distances([], tr, MIC, ROOM)
    assert empty.image_count() == 0 and empty.d.shape == (0, len(tr))


def test_high_order_factor_one_equals_low():
    tr = moving_traj(4000, 0.25)
    images = [sp for sp in mvb.enumerate_images(ROOM, 2) if sp.order == 2]
    low = synth.low_order_distances(images, tr, MIC, ROOM)
    high = synth.high_order_distances(images, tr, MIC, ROOM, len(tr), 1)
    assert np.array_equal(low.d, high.d)
    longer = synth.high_order_distances(images, tr, MIC, ROOM, len(tr) + 50, 1)
    assert np.array_equal(longer.d[:, len(tr):], np.repeat(low.d[:, -1:], 50, axis=1))


def test_high_order_matches_oracle_upsampler_and_counts():
    n = 32000
    tr = moving_traj(n, 2.0)
    coarse = mvb.decimate(tr, 3200)
    images = [sp for sp in mvb.enumerate_images(ROOM, 2) if sp.order == 2]
    high = synth.high_order_distances(images, coarse, MIC, ROOM, n, 3200)
    assert high.d.shape == (len(images), n)
    assert high.eval_count == len(images) * len(coarse)
    assert high.rate == coarse.rate * 3200
    offset, sign, _, _ = as_arrays(images, ROOM)
    c = orc.distance_streams(offset, sign, MIC.pos, coarse.positions)
    tab = orc.phase_table(3200)
    want = np.stack([orc.upsample_stream(row, tab, 3200, n) for row in c])
    assert np.array_equal(high.d, want)


def test_high_order_interior_accuracy():
    n = 16 * 16000
    tr = moving_traj(n, 16.0)
    coarse = mvb.decimate(tr, 3200)
    images = [sp for sp in mvb.enumerate_images(ROOM, 2) if sp.order == 2][:4]
    high = synth.high_order_distances(images, coarse, MIC, ROOM, n, 3200)
    exact = synth.low_order_distances(images, tr, MIC, ROOM)
    guard = 33 * 3200
    assert np.max(np.abs(high.d[:, guard:-guard] - exact.d[:, guard:-guard])) < 5e-4


def test_merge_restores_canonical_order():
    tr = moving_traj(2000, 0.125)
    images = mvb.enumerate_images(ROOM, 2)
    a = synth.low_order_distances([sp for sp in images if sp.order <= 1], tr, MIC, ROOM)
    b = synth.low_order_distances([sp for sp in images if sp.order > 1], tr, MIC, ROOM)
    merged = synth.merge_streams(a, b)
    assert merged.specs == images
    direct = synth.low_order_distances(images, tr, MIC, ROOM)
    assert np.array_equal(merged.d, direct.d)
    assert merged.eval_count == a.eval_count + b.eval_count


def test_merge_with_empty_side_and_errors():
    tr = moving_traj(1000, 0.0625)
    images = mvb.enumerate_images(ROOM, 1)
    a = synth.low_order_distances(images, tr, MIC, ROOM)
    empty = synth.low_order_distances([], tr, MIC, ROOM)
    assert synth.merge_streams(a, empty) is a
    assert synth.merge_streams(empty, a) is a
    other = synth.high_order_distances(images, tr, MIC, ROOM, len(tr) + 1, 1)
    with pytest.raises(ValueError):
        synth.merge_streams(a, other)
    slow = mvb.DelayStreams(rate=tr.rate / 2, specs=images, d=a.d)
    with pytest.raises(ValueError):
        synth.merge_streams(a, slow)


def tier_streams(images, traj, mic, room, tiers):
    """The reference's stream composition (synth.py:273-288 generalised to
    a tier table, as tests/golden/make_golden.py builds its goldens)."""
    streams, prev = None, -1
    for mo, N in tiers:
        sel = [sp for sp in images if prev < sp.order <= mo]
        prev = mo
        st = synth.low_order_distances(sel, traj, mic, room) if N == 1 else \
            synth.high_order_distances(sel, mvb.decimate(traj, N), mic, room, len(traj), N)
        streams = st if streams is None else synth.merge_streams(streams, st)
    return streams


BUILT = {
    "c1_refdesign": ("c1", dict(tiers=((1, 1), (3, 32)))),
    "c3": ("c3", dict(duration=0.1, max_order=8, tiers=((2, 1), (5, 32), (8, 256)))),
}


@pytest.mark.parametrize("case", list(BUILT))
def test_builders_then_synthesize_match_reference_render(case):
    """The public stream builders composed as the reference composes them,
    synthesised on the exact track path, equal the reference's own render
    (tests/golden/render_<case>.npz) and the fused exact engine."""
    g = golden(f"render_{case}.npz")
    wl, over = BUILT[case]
    sc = workloads.make_scenes(wl, **over)[0]
    b = g["branches"]
    f = FarrowFilter(b.shape[0] - 1, b.shape[1], b, (b.shape[1] - 1) // 2, 1.0)
    room = mvb.Room(dims=sc.dims, wall_reflection=sc.walls)
    tr = mvb.Trajectory(rate=sc.rate, positions=sc.pos)
    mic = mvb.MicPosition(pos=sc.mics[0])
    streams = tier_streams(mvb.enumerate_images(room, sc.max_order), tr, mic, room, sc.tiers)
    cfg = mvb.SynthesisConfig(audio_rate=sc.rate, max_order=sc.max_order, tiers=sc.tiers)
    s64 = np.asarray(sc.s, np.float64)
    y = mvb.synthesize(s64, streams, f, cfg)
    n0 = int(g["lens"][0])
    assert y.size == n0
    assert rel_err(y, g["y"][:n0]) <= 1e-12
    eng = mvb.render(s64, tr, room, mic, f, cfg)
    assert np.array_equal(y, eng)  # same arithmetic and order: bit-identical
    # the reference dataclass form, numpy tracks built by hand, renders the same
    hand = mvb.DelayStreams(streams.rate, streams.specs, np.array(streams.d), streams.eval_count)
    assert np.array_equal(mvb.synthesize(s64, hand, f, cfg), y)


def test_source_modulation_on_built_streams():
    g = golden("render_c1_source.npz")
    sc = workloads.make_scenes("c1", duration=0.25, tiers=((1, 1), (3, 32)))[0]
    f = FarrowFilter(3, 8, g["branches"], 3, 0.8)
    room = mvb.Room(dims=sc.dims, wall_reflection=sc.walls)
    tr = mvb.Trajectory(rate=sc.rate, positions=sc.pos)
    images = mvb.enumerate_images(room, 3)
    low = synth.low_order_distances([sp for sp in images if sp.order <= 1], tr, sc.mics[0], room)
    high = synth.high_order_distances([sp for sp in images if sp.order > 1],
                                      mvb.decimate(tr, 32), sc.mics[0], room, len(tr), 32)
    cfg = mvb.SynthesisConfig(audio_rate=sc.rate, max_order=3, order_split=1, decimation=32,
                              modulate="source")
    y = mvb.synthesize(sc.s, synth.merge_streams(low, high), f, cfg)
    assert y.size == g["y"].size and rel_err(y, g["y"]) <= 1e-12


# ------------------------------------------------------------ Farrow operators
def test_branch_filter_shape_dc_and_oracle():
    f = design_filter()
    v = farrow.branch_filter(np.ones(100), f)
    assert v.shape == (4, 107)
    v = farrow.branch_filter(np.ones(64), f)
    assert np.allclose(v[0, 10:50], 1.0, atol=1e-9)
    assert np.allclose(v[1:, 10:50], 0.0, atol=1e-9)
    x = np.random.default_rng(7).standard_normal(999)
    assert np.array_equal(farrow.branch_filter(x, f), orc.branch_filter(x, f.branches))
    xd = torch.from_numpy(x).cuda()
    out = farrow.branch_filter(xd, f)
    assert out.is_cuda and np.array_equal(out.cpu().numpy(), orc.branch_filter(x, f.branches))
    for bad in (np.ones((2, 3)), np.array([1.0, np.nan]), np.array([])):
        with pytest.raises(ValueError):
            farrow.branch_filter(bad, f)


def test_horner_matches_power_sum_and_bounds():
    f = design_filter()
    v = farrow.branch_filter(np.random.default_rng(7).standard_normal(256), f)
    for total in (5.3, 11.75, 40.0):
        sp = mvb.split_delay(total, f)
        for n in range(60, 90):
            a = farrow.evaluate(v, n, sp)
            b = farrow.evaluate_power_sum(v, n, sp)
            assert abs(a - b) <= 1e-12 * max(1.0, abs(b))
    sp = mvb.split_delay(5.5, f)
    assert farrow.evaluate(v, -1, sp) == 0.0
    assert farrow.evaluate(v, v.shape[1] + 10, sp) == 0.0


def test_delay_stream_matches_oracle_and_evaluate():
    f = design_filter()
    x = np.random.default_rng(11).standard_normal(3000)
    tau = 4.0 + 30.0 * (0.5 + 0.5 * np.sin(np.arange(3200) / 300.0))
    y = farrow.delay_stream(x, f, tau)
    want = np.zeros(tau.size)
    orc.accumulate_images(want, orc.branch_filter(x, f.branches), tau[None], np.ones((1, tau.size)),
                          0, f.nominal_delay)
    assert np.array_equal(y, want)
    v = farrow.branch_filter(x, f)
    for n in (100, 1500, 2999):
        assert abs(y[n] - farrow.evaluate(v, n, mvb.split_delay(tau[n], f))) <= 1e-12
    yd = farrow.delay_stream(torch.from_numpy(x).cuda(), f, torch.from_numpy(tau).cuda())
    assert yd.is_cuda and np.array_equal(yd.cpu().numpy(), y)


@pytest.mark.parametrize("tau_val", [3.0, 8.25, 20.37, 33.999])
def test_delay_stream_constant_delay_sine(tau_val):
    f = design_filter()
    rate = 16000.0
    x = sine(500.0, 0.25, rate)
    y = farrow.delay_stream(x, f, np.full(x.size, tau_val))
    t = np.arange(x.size) / rate
    ref = np.sin(2 * np.pi * 500.0 * (t - tau_val / rate))
    assert snr_db(y[100:-100], ref[100:-100]) >= 60.0


def test_delay_stream_linear_delay_scales_frequency():
    f = design_filter()
    rate, f0, slope = 16000.0, 1000.0, 1.0 / 343.0
    x = sine(f0, 1.0, rate)
    y = farrow.delay_stream(x, f, 10.0 + slope * np.arange(x.size))
    from scipy.signal import hilbert
    phase = np.unwrap(np.angle(hilbert(y[1000:-1000])))
    inst = np.diff(phase) * rate / (2 * np.pi)
    assert np.mean(inst[500:-500]) == pytest.approx(f0 * (1.0 - slope), abs=0.05)


def test_delay_stream_rejects():
    f = design_filter()
    with pytest.raises(ValueError):
        farrow.delay_stream(np.ones(32), f, np.full(32, 1.0))
    tau = np.full(32, 5.0)
    tau[3] = np.nan
    with pytest.raises(ValueError):
        farrow.delay_stream(np.ones(32), f, tau)
    with pytest.raises(ValueError):
        farrow.delay_stream(np.ones(32), f, np.full((2, 16), 5.0))


# ------------------------------------------------------------ bandwidth
def test_bandwidth_estimate_matches_oracle():
    rng = np.random.default_rng(2)
    rate = 16000.0
    t = np.arange(8000) / rate
    for freq in (0.5, 3.0, 40.0):
        pos = np.stack([1 + 0.2 * np.sin(2 * np.pi * freq * t), 2 + 0 * t,
                        1.5 + 0.01 * rng.standard_normal(t.size)], axis=1)
        tr = mvb.Trajectory(rate=rate, positions=pos)
        for frac in (0.5, 0.99):
            assert trajectory.bandwidth_estimate(tr, frac) == orc.bandwidth_estimate(pos, rate, frac)
    still = mvb.Trajectory(rate=rate, positions=np.tile([1.0, 2.0, 1.5], (100, 1)))
    assert trajectory.bandwidth_estimate(still) == 0.0
    one = mvb.Trajectory(rate=rate, positions=np.array([[1.0, 2.0, 1.5]]))
    assert trajectory.bandwidth_estimate(one) == 0.0
    for bad in (0.0, 1.0, -0.5):
        with pytest.raises(ValueError):
            trajectory.bandwidth_estimate(still, bad)
