"""Static responses, convolution, splice baseline and compare on the GPU
(SURVEY.md 8f row 3), against the reference's own outputs
(tests/golden/static.npz), the CPU oracle, and the behaviours the
reference's tests/test_reference.py checks.  Marker `gpu`."""

import numpy as np
import pytest

from conftest import golden
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2508_03065_b200 as mvb  # noqa: E402

RATE = 16000.0
ROOM = mvb.Room(dims=np.array([5.0, 6.0, 4.0]), wall_reflection=np.full(6, 0.9))
MIC = mvb.MicPosition(pos=np.array([1.25, 2.6, 2.75]))
SRCS = {"far": [2.0, 3.5, 2.0], "near": [1.5, 2.8, 2.5], "corner": [0.3, 5.6, 0.4]}
TOL = 1e-12  # fp64 bar is 1e-10 of the peak; sin/i0/sqrt roundings differ by ulps


def sine(freq, n):
    return np.sin(2 * np.pi * freq * np.arange(n) / RATE)


def static_traj(pos, n):
    return mvb.Trajectory(rate=RATE, positions=np.tile(np.asarray(pos, float), (n, 1)))


def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


# --------------------------------------------------------------- golden parity
def test_static_rir_matches_reference_golden():
    g = golden("static.npz")
    for tag, src in SRCS.items():
        for order in (0, 2, 3):
            r = mvb.static_rir(ROOM, np.array(src), MIC, RATE, order)
            ref = g[f"rir_{tag}_{order}"]
            assert r.taps.size == ref.size
            assert r.image_count == int(g[f"rir_{tag}_{order}_count"])
            assert rel(r.taps, ref) <= TOL


def test_static_render_matches_reference_golden():
    g = golden("static.npz")
    rir = mvb.static_rir(ROOM, np.array(SRCS["far"]), MIC, RATE, 2)
    for tag in ("small", "large"):  # reference: np.convolve / fftconvolve branches
        y = mvb.static_render(g[f"x_{tag}"], rir)
        ref = g[f"render_{tag}"]
        assert y.size == ref.size
        assert rel(y, ref) <= TOL


def test_splice_matches_reference_golden():
    g = golden("static.npz")
    traj = mvb.Trajectory(rate=RATE, positions=g["splice_pos"])
    cfg = mvb.SynthesisConfig(max_order=2, decimation=1)
    for hop, cf in ((640, 0), (640, 128), (640, 200), (600, 100), (1000, 1000)):
        y = mvb.splice_baseline(g["splice_x"], traj, ROOM, MIC, hop, cf, cfg)
        ref = g[f"splice_{hop}_{cf}"]
        assert y.size == ref.size
        assert rel(y, ref) <= TOL


def test_compare_matches_reference_golden():
    g = golden("static.npz")
    kws = {"ab": dict(passband=0.8, rate=RATE, interior=0.05),
           "aa": dict(passband=1.0, rate=RATE, interior=0.1),
           "noisy": dict(passband=0.9, rate=RATE, interior=0.0)}
    for tag, kw in kws.items():
        rep = mvb.compare(g[f"cmp_{tag}_a"], g[f"cmp_{tag}_b"], **kw)
        assert rep.snr_db == pytest.approx(float(g[f"cmp_{tag}_snr"]), rel=1e-9, abs=1e-9)
        assert rep.envelope_max_jump == pytest.approx(float(g[f"cmp_{tag}_jump"]), rel=1e-9)
        tr = g[f"cmp_{tag}_track"]
        assert rep.inst_freq_track.shape == tr.shape
        assert np.max(np.abs(rep.inst_freq_track - tr)) <= 1e-8


def test_static_rir_and_splice_match_oracle_larger():
    """Order 8 in a larger room (thousands of overlapping images per tap)
    and a 1 s splice, against the CPU oracle."""
    room = mvb.Room(dims=np.array([10.0, 8.0, 4.0]), wall_reflection=np.full(6, 0.85))
    mic = np.array([3.0, 2.5, 1.5])
    src = np.array([6.0, 5.0, 2.0])
    r = mvb.static_rir(room, src, mic, 48000.0, 8)
    ref = orc.static_rir_taps(room.dims, room.wall_reflection, src, mic, 48000.0, 8)
    assert r.taps.size == ref.size and rel(r.taps, ref) <= TOL
    n = 16000
    t = np.arange(n) / RATE
    pos = np.stack([2.0 + 2.0 * t, 3.0 + 0.5 * t, np.full(n, 2.0)], axis=1)
    x = np.random.default_rng(5).standard_normal(n)
    cfg = mvb.SynthesisConfig(max_order=4, decimation=1)
    y = mvb.splice_baseline(x, mvb.Trajectory(rate=RATE, positions=pos), room, mic, 512, 64, cfg)
    yo = orc.splice_baseline(x, pos, room.dims, room.wall_reflection, mic, RATE, 4, 512, 64)
    assert y.size == yo.size and rel(y, yo) <= TOL


# ------------------------------------------ reference test_reference.py behaviours
def test_unit_and_two_tap_responses():
    y = mvb.static_render(np.arange(10.0), mvb.StaticRIR(RATE, np.array([1.0]), 1, 0))
    assert np.allclose(y, np.arange(10.0))
    y = mvb.static_render(np.array([1.0, 2.0, 3.0]), mvb.StaticRIR(RATE, np.array([0.5, 0.0, 0.25]), 2, 1))
    assert np.allclose(y, 0.5 * np.array([1, 2, 3, 0, 0.0]) + 0.25 * np.array([0, 0, 1, 2, 3.0]))
    with pytest.raises(ValueError):
        mvb.static_render(np.ones(4), mvb.StaticRIR(RATE, np.ones(3), 1, 0), rate=8000.0)


def test_matches_naive_convolution_all_shapes():
    rng = np.random.default_rng(0)
    for n, m in ((400, 37), (5, 3000), (3000, 1), (1, 1), (2049, 1025)):
        x, taps = rng.standard_normal(n), rng.standard_normal(m)
        y = mvb.static_render(x, mvb.StaticRIR(RATE, taps, 1, 0))
        naive = np.zeros(n + m - 1)
        for i, v in enumerate(x):
            naive[i:i + m] += v * taps
        assert rel(y, naive) <= 1e-12


def test_direct_tap_amplitude_delay_and_sine():
    src = np.array([2.0, 3.5, 2.0])
    rir = mvb.static_rir(ROOM, src, MIC, RATE, 0)
    d = float(np.linalg.norm(src - MIC.pos))
    tau, amp = RATE * d / 343.0, 1.0 / (4 * np.pi * d)
    assert rir.image_count == 1
    assert np.sum(rir.taps) == pytest.approx(amp, rel=1e-3)
    centroid = np.sum(np.arange(rir.taps.size) * rir.taps) / np.sum(rir.taps)
    assert centroid == pytest.approx(tau, abs=0.05)
    x = sine(900.0, 8000)
    y = mvb.static_render(x, rir)
    ref = amp * np.sin(2 * np.pi * 900.0 * (np.arange(y.size) / RATE - d / 343.0))
    err = y[200:7800] - ref[200:7800]
    assert 10 * np.log10(np.sum(ref[200:7800] ** 2) / np.sum(err ** 2)) >= 60.0


def test_static_rir_validation_and_counts():
    with pytest.raises(ValueError):
        mvb.static_rir(ROOM, np.array([9.0, 1.0, 1.0]), MIC, RATE, 1)
    with pytest.raises(ValueError):
        mvb.static_rir(ROOM, np.array([2.0, 3.0, 2.0]), np.array([1.0, 7.0, 1.0]), RATE, 1)
    assert mvb.static_rir(ROOM, np.array([2.0, 3.5, 2.0]), MIC, RATE, 2).image_count == 1 + 6 + 18


def test_static_limit_of_moving_oracle():
    """full_rate_moving_oracle with a frozen path ~ static render (>= 60 dB)."""
    src = np.array([0.8, 4.1, 2.75])
    n = 8000
    b = golden("kernels.npz")["design_3_8_08"]
    f = mvb.FarrowFilter(3, 8, b, 3, 0.8)
    cfg = mvb.SynthesisConfig(max_order=2, decimation=1)
    y = mvb.full_rate_moving_oracle(sine(1000.0, n), static_traj(src, n), ROOM, MIC, f, cfg)
    ref = mvb.static_render(sine(1000.0, n), mvb.static_rir(ROOM, src, MIC, RATE, 2))
    assert mvb.compare(y, ref, passband=0.8, rate=RATE).snr_db >= 60.0


def test_splice_static_equals_static_render_and_crossfade():
    src = np.array([0.8, 4.1, 2.75])
    n = 4000
    x = sine(700.0, n)
    cfg = mvb.SynthesisConfig(max_order=1, decimation=1)
    y0 = mvb.splice_baseline(x, static_traj(src, n), ROOM, MIC, 640, 0, cfg)
    ref = mvb.static_render(x, mvb.static_rir(ROOM, src, MIC, RATE, 1))
    m = min(y0.size, ref.size)
    assert np.allclose(y0[:m], ref[:m], atol=1e-12)
    y1 = mvb.splice_baseline(x, static_traj(src, n), ROOM, MIC, 640, 128, cfg)
    assert np.allclose(y0[:m], y1[:m], atol=1e-10)
    tr = static_traj([2.0, 3.0, 2.0], 1000)
    with pytest.raises(ValueError):
        mvb.splice_baseline(np.ones(1000), tr, ROOM, MIC, 100, 101, cfg)
    with pytest.raises(ValueError):
        mvb.splice_baseline(np.ones(1000), tr, ROOM, MIC, 0, 0, cfg)


def test_moving_source_splice_envelope_jumps():
    n = 16000
    t = np.arange(n) / RATE
    pos = np.stack([1.0 + 0.9 * t, np.full(n, 3.0), np.full(n, 2.0)], axis=1)
    traj = mvb.Trajectory(rate=RATE, positions=pos)
    b = golden("kernels.npz")["design_3_8_08"]
    f = mvb.FarrowFilter(3, 8, b, 3, 0.8)
    cfg = mvb.SynthesisConfig(max_order=0, decimation=1)
    x = sine(1000.0, n)
    y_s = mvb.splice_baseline(x, traj, ROOM, MIC, 640, 0, cfg)
    y_e = mvb.render(x, traj, ROOM, MIC, f, cfg)
    r_s = mvb.compare(y_s, y_s, passband=1.0, rate=RATE)
    r_e = mvb.compare(y_e, y_e, passband=1.0, rate=RATE)
    assert r_s.envelope_max_jump > 5.0 * r_e.envelope_max_jump


def test_compare_behaviours():
    rng = np.random.default_rng(1)
    b = rng.standard_normal(32000)
    noise = rng.standard_normal(32000)
    noise *= np.sqrt(np.sum(b ** 2) / np.sum(noise ** 2)) * 10 ** (-40 / 20)
    assert mvb.compare(b + noise, b, passband=1.0, rate=RATE, interior=0.0).snr_db == pytest.approx(40.0, abs=0.2)
    x = sine(440.0, 4000)
    assert mvb.compare(x, x, passband=1.0, rate=RATE).snr_db == 200.0
    assert mvb.compare(np.concatenate([x, np.ones(500)]), x, passband=1.0, rate=RATE).snr_db == 200.0
    with pytest.raises(ValueError):
        mvb.compare(np.ones(1000), np.zeros(1000), passband=1.0)
    with pytest.raises(ValueError):
        mvb.compare(x, x, passband=1.1)
    with pytest.raises(ValueError):
        mvb.compare(np.ones(4), np.ones(4))
    n = 32000
    tt = np.arange(n) / RATE
    bb = np.sin(2 * np.pi * 1000.0 * tt)
    aa = bb + 0.5 * np.sin(2 * np.pi * 7000.0 * tt)
    assert mvb.compare(aa, bb, passband=0.8, rate=RATE).snr_db >= 100.0
    assert mvb.compare(aa, bb, passband=1.0, rate=RATE).snr_db < 20.0
    tone = sine(997.0, 16000)
    rep = mvb.compare(tone, tone, passband=1.0, rate=RATE, interior=0.1, runtime_counts={"evals": 42})
    assert np.mean(rep.inst_freq_track) == pytest.approx(997.0, abs=0.05)
    assert rep.runtime_counts == {"evals": 42}
