"""The hand-written fp64 FFT path of decimate() (csrc/fft.cu): the batched
complex FFT against numpy (smooth lengths through the mixed-radix Stockham
passes, other lengths through Bluestein, both directions), the bandwidth
decision against the oracle's restatement of the reference
(trajectory.py:316-339) and the anti-alias low-pass against it
(trajectory.py:214-232).  Marker `gpu`."""

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2508_03065_b200 import _lib  # noqa: E402
from paper_2508_03065_b200._dev import ptr, stream_handle  # noqa: E402
from paper_2508_03065_b200.trajectory import bandwidth_batch, lowpass_batch  # noqa: E402

DEV = torch.device("cuda", 0)


def _fft(x: np.ndarray, sign: int) -> np.ndarray:
    rows, n = x.shape
    d = torch.from_numpy(np.ascontiguousarray(x.astype(np.complex128))).to(DEV)
    scratch = torch.empty(int(_lib.lib().mvb_fft_scratch_elems(rows, n)) * 2, dtype=torch.float64,
                          device=DEV)
    _lib.call("mvb_fft_c2c", ptr(d), rows, n, sign, ptr(scratch), stream_handle(DEV))
    return d.cpu().numpy()


@pytest.mark.parametrize("n", [2, 3, 4, 5, 7, 8, 12, 49, 60, 97, 360, 1000, 2999, 4096, 7919,
                               64000, 96000, 480000])
def test_fft_matches_numpy(n):
    rng = np.random.default_rng(n)
    rows = 3 if n < 100000 else 1
    x = rng.standard_normal((rows, n)) + 1j * rng.standard_normal((rows, n))
    y = _fft(x, -1)
    ref = np.fft.fft(x, axis=1)
    assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))
    z = _fft(x, +1)
    ref_inv = np.fft.ifft(x, axis=1) * n
    assert np.max(np.abs(z - ref_inv)) <= 1e-12 * np.max(np.abs(ref_inv))


def _paths(G, T, seed, rate):
    rng = np.random.default_rng(seed)
    t = np.arange(T) / rate
    out = []
    for g in range(G):
        f = rng.uniform(0.5, 0.45 * rate, size=3)
        a = rng.uniform(0.1, 2.0, size=3)
        out.append(np.stack([a[i] * np.sin(2 * np.pi * f[i] * t + g) + 0.01 * rng.standard_normal(T)
                             for i in range(3)], axis=1) + rng.uniform(1, 4, size=3))
    return np.stack(out)


@pytest.mark.parametrize("T", [2, 17, 1000, 4099, 64000])
def test_bandwidth_decision_matches_oracle(T):
    rate = 16000.0
    x = _paths(5, T, T, rate)
    got = bandwidth_batch(torch.from_numpy(x).to(DEV), rate)
    want = np.array([orc.bandwidth_estimate(x[g], rate) for g in range(x.shape[0])])
    assert np.array_equal(got, want), (got, want)


@pytest.mark.parametrize("T", [3, 40, 1001, 6000, 64000])
def test_lowpass_matches_oracle(T):
    rate = 16000.0
    x = _paths(3, T, T + 1, rate)
    cutoff = 0.9 * 0.5 * rate / 64
    got = lowpass_batch(torch.from_numpy(x).to(DEV), rate, cutoff).cpu().numpy()
    for g in range(x.shape[0]):
        ref = orc.lowpass_columns(x[g], rate, cutoff)
        assert np.max(np.abs(got[g] - ref)) <= 1e-11 * max(1.0, np.max(np.abs(ref)))
