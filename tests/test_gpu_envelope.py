"""The fp32 fast path's accuracy envelope.

The fast engine carries the delay inside a coarse interval as an fp32
residual around an fp64 anchor (the reference carries tau in fp64,
synth.py:218, _kernels.py:112-116); its rounding grows with the interval's
delay excursion kappa * speed * N / rate.  Geometry.interval_excursion
bounds that excursion from the device-measured largest path steps, and a
render beyond engine.FP32_ENVELOPE samples routes to the exact fp64 engine
-- through render_jobs, RenderPlan (a slot re-captures when the envelope
decision changes) and the public render().  Marker `gpu`."""

import numpy as np
import pytest

from conftest import rel_err
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2508_03065_b200 import (Room, SynthesisConfig, Trajectory, engine, hann_sinc,  # noqa: E402
                                   render)
from paper_2508_03065_b200.plan import RenderPlan  # noqa: E402
from paper_2508_03065_b200.synth import render_jobs  # noqa: E402

RATE = 48000.0
TIERS = ((1, 1), (3, 256))
DIMS = np.array([7.0, 5.0, 3.5])
MIC = np.array([3.0, 2.5, 1.4])


def _path(speed, T=4800, seed=0):
    rng = np.random.default_rng(seed)
    d = rng.normal(size=3)
    d /= np.linalg.norm(d)
    t = np.arange(T)[:, None] / RATE
    return np.array([2.0, 2.0, 1.5]) + d * speed * t


def _job(pos, s):
    return engine.Job(s=s, pos=pos, mic=MIC, dims=DIMS, walls=0.9, max_order=3, tiers=TIERS,
                      rate=RATE)


def _oracle(pos, s, f):
    return orc.OracleScene(np.asarray(s, np.float64), pos, MIC, DIMS, 0.9, 3, TIERS, f.branches,
                           RATE).render()


@pytest.mark.parametrize("speed", [3.0, 170.0, 570.0])
def test_fast_request_meets_the_bar_at_any_speed(speed):
    f = hann_sinc(64, 14)
    s = np.random.default_rng(1).standard_normal(2400).astype(np.float32)
    pos = _path(speed)
    exc = speed * 256 / 343.0
    res = render_jobs([_job(pos, s)], f, precision="fp32")
    want = "fp32" if exc <= engine.FP32_ENVELOPE else "fp64"
    assert res.precision == want, (speed, exc)
    y = res.job(0).double().cpu().numpy()
    ref = _oracle(pos, s, f)
    assert y.size == ref.size
    assert rel_err(y, ref) <= 1e-5


def test_interval_excursion_bounds_the_path():
    pos = _path(100.0)
    g = engine.Geometry([_job(pos, np.zeros(8, np.float32))])
    step = np.max(np.linalg.norm(np.diff(pos, axis=0), axis=1))
    exc = g.interval_excursion()[0]
    assert abs(exc - RATE / 343.0 * step * 256) <= 1e-9 * exc
    # moving receiver: its steps add
    mic = MIC + np.zeros((pos.shape[0], 3))
    mic[:, 0] += np.arange(pos.shape[0]) * (10.0 / RATE)
    g2 = engine.Geometry([engine.Job(s=np.zeros(8, np.float32), pos=pos, mic=mic, dims=DIMS,
                                     walls=0.9, max_order=3, tiers=TIERS, rate=RATE)])
    assert g2.interval_excursion()[0] == pytest.approx(RATE / 343.0 * (step + 10.0 / RATE) * 256,
                                                       rel=1e-9)


def test_plan_recaptures_when_the_envelope_decision_changes():
    f = hann_sinc(64, 14)
    s = np.random.default_rng(2).standard_normal(2400).astype(np.float32)
    slow, fast = _path(4.0, seed=3), _path(570.0, seed=3)
    plan = RenderPlan([_job(slow, s)], f, precision="fp32")
    for pos in (slow, slow, fast, fast, slow):
        res = plan.run([_job(pos, s)])
        y = res.job(0).double().cpu().numpy()
        ref = _oracle(pos, s, f)
        assert y.size == ref.size and rel_err(y, ref) <= 1e-5
        assert res.precision == ("fp64" if pos is fast else "fp32")


def test_public_render_routes_fast_sources():
    f = hann_sinc(64, 14)
    s = np.random.default_rng(4).standard_normal(2400).astype(np.float32)
    pos = _path(570.0, seed=5)
    cfg = SynthesisConfig(audio_rate=RATE, max_order=3, tiers=TIERS)
    for _ in range(3):  # first call direct, then the cached plan
        y = render(s, Trajectory(rate=RATE, positions=pos), Room(dims=DIMS, wall_reflection=0.9),
                   MIC, f, cfg)
        assert rel_err(y, _oracle(pos, s, f)) <= 1e-5
