"""The L0 CPU baseline (oracle/l0.py) runs the reference's own code from
baseline/_ref: its window trick reproduces the oracle's render window, and
its whole render equals the oracle (itself pinned to the reference
goldens).  Skipped when the reference is not installed there."""

import numpy as np
import pytest

from oracle import oracle as orc

l0 = pytest.importorskip("oracle.l0")
try:
    l0.load()
except ImportError as e:  # pragma: no cover - environment dependent
    pytest.skip(f"reference not installed: {e}", allow_module_level=True)

from paper_2508_03065_b200 import hann_sinc, workloads  # noqa: E402


def test_kernel_window_matches_oracle():
    sc = workloads.make_scenes("c3", duration=0.2, max_order=6, tiers=((2, 1), (4, 32), (6, 256)))[0]
    f = hann_sinc(sc.fd_taps, 14)
    o = orc.OracleScene(sc.s, sc.pos, sc.mics[0], sc.dims, sc.walls, sc.max_order, sc.tiers,
                        f.branches, sc.rate)
    ks = l0.KernelSample(o, f.branches, 5000, 700, 4)
    y, dt = ks.run(4)
    ref = o.render_window(5000, 5700)
    assert dt > 0 and np.max(np.abs(y - ref)) <= 1e-11 * np.max(np.abs(ref))


def test_whole_render_matches_oracle():
    sc = workloads.make_scenes("c2", duration=0.1, max_order=5, tiers=((2, 1), (5, 16)))[0]
    f = hann_sinc(sc.fd_taps, 14)
    r = l0.render_sample(sc, f.branches, 4)
    ref = orc.OracleScene(sc.s, sc.pos, sc.mics[0], sc.dims, sc.walls, sc.max_order, sc.tiers,
                          f.branches, sc.rate).render()
    assert r["numba"] and r["out"].size == ref.size
    assert np.max(np.abs(r["out"] - ref)) <= 1e-12 * np.max(np.abs(ref))
