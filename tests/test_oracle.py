"""Pin the CPU oracle against golden vectors produced by the reference
itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import golden, rel_err
from oracle import oracle as orc
from paper_2508_03065_b200 import workloads
from paper_2508_03065_b200.farrow import hann_sinc


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_enumerate_matches_reference(kernels_golden, tag):
    g = kernels_golden
    im = orc.enumerate_images(g[f"enum_{tag}_dims"], g[f"enum_{tag}_walls"],
                              int(g[f"enum_{tag}_order"]))
    assert np.array_equal(im.order, g[f"enum_{tag}_ord"])
    assert np.array_equal(im.lattice, g[f"enum_{tag}_lattice"])
    assert np.array_equal(im.parity, g[f"enum_{tag}_parity"])
    assert np.array_equal(im.offset, g[f"enum_{tag}_offset"])
    assert np.array_equal(im.sign, g[f"enum_{tag}_sign"])
    np.testing.assert_allclose(im.beta, g[f"enum_{tag}_beta"], rtol=2e-16, atol=0)


def test_image_counts():
    for o in range(0, 25):
        assert orc.image_count(o) == 1 + sum(4 * k * k + 2 for k in range(1, o + 1))


def test_distance_bitwise(kernels_golden):
    g = kernels_golden
    d = orc.distance_streams(g["dist_offset"], g["dist_sign"], g["dist_mic"], g["dist_pos"])
    assert np.array_equal(d, g["dist_out"])


def test_accumulate_bitwise(kernels_golden):
    g = kernels_golden
    out = np.zeros(g["acc_out"].size)
    orc.accumulate_images(out, g["acc_streams"], g["acc_tau"], g["acc_amp"], 8, 3)
    assert np.array_equal(out, g["acc_out"])


@pytest.mark.parametrize("N", [16, 64])
def test_upsample_and_table(kernels_golden, N):
    g = kernels_golden
    tab = orc.phase_table(N)
    np.testing.assert_allclose(tab, g[f"table{N}"], rtol=0, atol=1e-16)
    up = orc.upsample_stream(g[f"up{N}_coarse"], g[f"table{N}"], N, g[f"up{N}_out"].size)
    assert np.array_equal(up, g[f"up{N}_out"])


def test_branch_filter(kernels_golden):
    g = kernels_golden
    v = orc.branch_filter(g["acc_x"], g["design_3_8_08"])
    assert rel_err(v, g["acc_streams"]) < 1e-15


@pytest.mark.parametrize("tag", ["slow", "fast"])
def test_decimate(kernels_golden, tag):
    g = kernels_golden
    out = orc.decimate_positions(g[f"dec_{tag}_in"], 1000.0, int(g[f"dec_{tag}_N"]))
    np.testing.assert_allclose(out, g[f"dec_{tag}_out"], rtol=0, atol=1e-13)


def test_hann_sinc_fit_matches_exact_taps():
    for L in (32, 64):
        f = hann_sinc(L, 14)
        mu = np.linspace(0, 1, 1001)
        h = (mu[:, None] ** np.arange(15)[None, :]) @ f.branches
        assert np.max(np.abs(h - orc.hann_sinc_taps(L, mu))) < 2e-14


CASES = {
    "c1": ("c1", dict()),
    "c1_refdesign": ("c1", dict(tiers=((1, 1), (3, 32)))),
    "c2": ("c2", dict(duration=0.25)),
    "c3": ("c3", dict(duration=0.1, max_order=8, tiers=((2, 1), (5, 32), (8, 256)))),
    "c4": ("c4", dict(duration=0.25, max_order=6, n_scenes=3)),
    "c5": ("c5", dict(duration=0.1, max_order=6, n_channels=4,
                      tiers=((2, 1), (4, 32), (6, 256)))),
}


def oracle_outputs(case):
    wl, over = CASES[case]
    g = golden(f"render_{case}.npz")
    scenes = workloads.make_scenes(wl, **over)
    ys = []
    for sc in scenes:
        for ch in [int(c) for c in g["channels"]] if wl == "c5" else range(len(sc.mics)):
            o = orc.OracleScene(sc.s, sc.pos, sc.mics[ch], sc.dims, sc.walls, sc.max_order,
                                sc.tiers, g["branches"], sc.rate)
            ys.append(o.render())
    return g, ys


@pytest.mark.parametrize("case", list(CASES))
def test_oracle_render_matches_reference(case):
    g, ys = oracle_outputs(case)
    lens = [y.size for y in ys]
    assert lens == [int(v) for v in g["lens"]]
    y = np.concatenate(ys)
    # same tracks and streams up to np.convolve's summation order (and, for
    # c5, the reference's moving-mic source transform): ~1e-15 relative
    assert rel_err(y, g["y"]) < 1e-12


# ---------------------------------------------------------------- static row
ROOM_DIMS, ROOM_WALLS = np.array([5.0, 6.0, 4.0]), np.full(6, 0.9)
MIC_STD = np.array([1.25, 2.6, 2.75])
STATIC_SRCS = {"far": [2.0, 3.5, 2.0], "near": [1.5, 2.8, 2.5], "corner": [0.3, 5.6, 0.4]}


def test_oracle_static_rir_matches_reference():
    g = golden("static.npz")
    for tag, src in STATIC_SRCS.items():
        for order in (0, 2, 3):
            ref = g[f"rir_{tag}_{order}"]
            taps = orc.static_rir_taps(ROOM_DIMS, ROOM_WALLS, src, MIC_STD, 16000.0, order)
            assert taps.size == ref.size
            assert np.max(np.abs(taps - ref)) <= 1e-13 * np.max(np.abs(ref))
            assert int(g[f"rir_{tag}_{order}_count"]) == orc.image_count(order)


def test_oracle_splice_matches_reference():
    g = golden("static.npz")
    for hop, cf in ((640, 0), (640, 128), (640, 200), (600, 100), (1000, 1000)):
        ref = g[f"splice_{hop}_{cf}"]
        y = orc.splice_baseline(g["splice_x"], g["splice_pos"], ROOM_DIMS, ROOM_WALLS, MIC_STD,
                                16000.0, 2, hop, cf)
        assert y.size == ref.size
        assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))
