"""CPU-only checks of the host layer and the C ABI library (no GPU)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "mvb.h")
LIB = os.path.join(ROOT, "paper_2508_03065_b200", "libmvb.so")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|int64_t|const char\*)\s+(mvb_\w+)\(", txt, re.M)))


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    lib = ctypes.CDLL(LIB)
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s


def test_struct_layout_matches_binding():
    from paper_2508_03065_b200 import _lib
    _lib.lib()  # raises on mismatch


def test_abi_version_and_counts():
    from paper_2508_03065_b200 import _lib
    assert _lib.lib().mvb_abi_version() == 1
    for o in (0, 1, 5, 20):
        assert _lib.image_count(o) == 1 + sum(4 * k * k + 2 for k in range(1, o + 1))
    hdr = open(os.path.join(ROOT, "include", "mvb.h")).read()
    assert re.search(r"#define MVB_DELAY_SORT_MAX (\d+)", hdr).group(1) == str(_lib.DELAY_SORT_MAX)
    assert re.search(r"#define MVB_EXACT_LIST_WORDS (\d+)", hdr).group(1) == str(_lib.EXACT_LIST_WORDS)


def test_product_refuses_to_run_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2508_03065_b200 import MvbError, Room, SynthesisConfig, Trajectory, hann_sinc, render
    room = Room(dims=np.array([5.0, 6.0, 4.0]), wall_reflection=0.9)
    tr = Trajectory(rate=16000.0, positions=np.tile([2.0, 3.0, 2.0], (100, 1)))
    with pytest.raises(MvbError):
        render(np.ones(100), tr, room, [1.0, 1.0, 1.0], hann_sinc(32), SynthesisConfig(max_order=1))


def test_host_api_helpers():
    """attenuation (reference room.py:168-172, test_room.py:143-151), the
    DelayStreams dataclass form (synth.py:94-119) and the Farrow scalar
    helpers (farrow.py:146-149, 232-250) -- host arithmetic, no GPU."""
    import paper_2508_03065_b200 as mvb
    from paper_2508_03065_b200 import farrow
    assert mvb.attenuation(0.5, 2.0) == pytest.approx(0.5 / (8 * np.pi), rel=1e-12)
    assert mvb.attenuation(1.0, 5.0) == pytest.approx(0.015915, abs=5e-7)
    with pytest.raises(ValueError):
        mvb.attenuation(1.0, 0.0)
    specs = [mvb.ImageSourceSpec(0, (0, 0, 0), (False, False, False), 1.0),
             mvb.ImageSourceSpec(1, (0, 0, 0), (True, False, False), 0.9)]
    d = np.array([[1.0, 2.0, 0.01], [3.0, 4.0, 5.0]])
    st = mvb.DelayStreams(rate=16000.0, specs=specs, d=d)
    cfg = mvb.SynthesisConfig()
    assert st.image_count() == 2 and st.eval_count == 0
    assert np.array_equal(st.tau(cfg), 16000.0 * d / 343.0)
    amp = st.amplitude(cfg)
    assert amp[0, 2] == pytest.approx(specs[0].beta / (4 * np.pi * 0.05))
    f = mvb.FarrowFilter(1, 2, np.array([[1.0, 0.0], [-1.0, 1.0]]), 0, 1.0)
    assert np.allclose(farrow.impulse_response(f, 0.25), [0.75, 0.25])
    v = np.array([[1.0, 2.0, 3.0], [0.5, 0.5, 0.5]])
    sp = mvb.split_delay(1.25, f)
    assert farrow.evaluate(v, 2, sp) == pytest.approx(2.0 + 0.25 * 0.5)
    assert farrow.evaluate(v, 2, sp) == farrow.evaluate_power_sum(v, 2, sp)
    assert farrow.evaluate(v, 0, sp) == 0.0


def test_config_validation():
    from paper_2508_03065_b200 import SynthesisConfig
    for kw in [{"audio_rate": 0.0}, {"decimation": 0}, {"order_split": -1}, {"max_order": -1},
               {"sound_speed": 0.0}, {"d_min": 0.0}, {"workers": 0}, {"eval_budget": 0.0},
               {"modulate": "both"}, {"t60": -1.0}, {"precision": "fp16"},
               {"tiers": ((2, 1), (1, 4))}, {"max_order": 5, "tiers": ((2, 1), (4, 8))}]:
        with pytest.raises(ValueError):
            SynthesisConfig(**kw)
    c = SynthesisConfig()
    assert c.tier_table() == ((1, 1), (3, 3200))
    assert SynthesisConfig(max_order=1, order_split=1).tier_table() == ((1, 1),)


def test_cost_report_matches_reference_numbers():
    from paper_2508_03065_b200 import SynthesisConfig, cost_report
    cfg = SynthesisConfig(audio_rate=16000.0, order_split=1, decimation=3200)
    rep = cost_report(cfg, 45000, 1.0)
    assert rep["naive_evals"] == 45000 * 16000
    assert rep["images_low"] == 7 and rep["images_high"] == 45000 - 7
    assert rep["high_order_reduction"] >= 100.0
    assert rep["hierarchical_evals"] == 7 * 16000 + (45000 - 7) * 5


def test_fast_bank_reduction():
    from paper_2508_03065_b200.engine import fast_bank
    from paper_2508_03065_b200.farrow import hann_sinc
    cb, M1, nb = fast_bank(hann_sinc(64, 14))
    assert (M1, nb) == (8, 8)
    mu = np.linspace(0, 1, 501)
    h = ((mu - 0.5)[:, None] ** np.arange(8)[None, :]) @ cb
    from oracle.oracle import hann_sinc_taps
    assert np.max(np.abs(h - hann_sinc_taps(64, mu))) < 6e-7


def test_farrow_centering_is_exact():
    from paper_2508_03065_b200.farrow import centered_branches, hann_sinc
    f = hann_sinc(32, 14)
    cb = centered_branches(f.branches)
    mu = np.linspace(0, 1, 101)
    a = (mu[:, None] ** np.arange(15)[None, :]) @ f.branches
    b = ((mu - 0.5)[:, None] ** np.arange(15)[None, :]) @ cb
    assert np.max(np.abs(a - b)) < 1e-13


def test_track_fit_accuracy_against_oracle_upsampler():
    """The fast path's interval polynomials, formed as in k_coeffs (summation
    by parts over fp32 coarse increments, sequential fp32 accumulation),
    reproduce the reference's 65-tap upsampled tracks to
    < 5e-9 m, i.e. < 7e-7 samples of delay at 48 kHz."""
    from oracle import oracle as orc
    from paper_2508_03065_b200.trajectory import phase_fit, phase_table
    from paper_2508_03065_b200 import workloads
    sc = workloads.make_scenes("c3", duration=1.0)[0]
    dims = sc.dims
    for N in (32, 256):
        cpos = sc.pos[::N]
        off = 2 * np.array([3.0, -2.0, 5.0]) * dims
        sg = np.array([1.0, -1.0, 1.0])
        coarse = orc.distance_streams(off[None], sg[None], dims / 2, cpos)[0]
        ref = orc.upsample_stream(coarse, phase_table(N), N, sc.T)
        F = phase_fit(N)
        G = np.zeros((9, 64))
        for j in range(64):
            G[:, j] = F[:, j + 1:].sum(1) if j >= 32 else -F[:, :j + 1].sum(1)
        G32 = G.astype(np.float32)
        K = coarse.size
        idx = np.clip(np.arange(K)[:, None] + np.arange(65)[None, :] - 32, 0, K - 1)
        dw = np.diff(coarse[idx], axis=1).astype(np.float32)  # (K, 64)
        acc = np.zeros((K, 9), np.float32)
        for j in range(64):
            acc = (acc + dw[:, j:j + 1] * G32[None, :, j]).astype(np.float32)
        g = acc.astype(np.float64)
        g[:, 0] += coarse
        u = 2 * np.arange(N) / N - 1
        d = (g @ (u[None, :] ** np.arange(9)[:, None])).reshape(-1)[:sc.T]
        assert np.max(np.abs(d - ref)) < 5e-9


def test_pack_jobs_matches_c_layout():
    """engine.pack_jobs writes the exact byte layout of mvb_job (mvb.h)."""
    from paper_2508_03065_b200.engine import pack_jobs

    class Job(ctypes.Structure):
        _fields_ = [(n, ctypes.c_int64) for n in
                    ("out_off", "out_len", "part_off", "rec_base", "ls", "img_off", "n_img",
                     "pos_off", "mic_off")] + \
                   [(n, ctypes.c_int32) for n in ("T", "mic_moving", "L", "d0", "n_chunks", "nb")] + \
                   [(n, ctypes.c_double) for n in ("rate", "c", "d_min", "kappa")] + \
                   [("img_stride", ctypes.c_int32), ("pad", ctypes.c_int32)]

    assert ctypes.sizeof(Job) == 136
    row = dict(out_off=1, out_len=2, part_off=3, rec_base=4, ls=5, img_off=6, n_img=7, pos_off=8,
               mic_off=9, T=10, mic_moving=1, L=64, d0=31, n_chunks=3, nb=8, rate=48000.0,
               c=343.0, d_min=0.05, kappa=48000.0 / 343.0, img_stride=11521)
    raw = pack_jobs([row]).tobytes()
    j = Job.from_buffer_copy(raw)
    for k, v in row.items():
        assert getattr(j, k) == v, k


def test_parallel_copy_chunks_and_casts():
    from paper_2508_03065_b200._staging import parallel_copy
    rng = np.random.default_rng(0)
    big = rng.standard_normal((3_000_000, 3))           # 72 MB: thread pool, many chunks
    small = rng.standard_normal(1000).astype(np.float32)
    dst_big = np.empty_like(big)
    dst_small = np.empty(1000, np.float64)
    parallel_copy([(dst_big, big), (dst_small, small)], chunk_bytes=1 << 20)
    assert np.array_equal(dst_big, big)
    assert np.array_equal(dst_small, small.astype(np.float64))


def test_class_table_layout():
    import ctypes
    from paper_2508_03065_b200 import _lib
    # mvb_class_table: int32 n + 3 x int32[8] (100 B) padded to 104, + 2 x int64[8]
    assert ctypes.sizeof(_lib.ClassTable) == 104 + 128
    assert _lib.ClassTable.table.offset == 104


def test_memory_groups_split_by_footprint():
    from paper_2508_03065_b200 import engine, workloads
    from paper_2508_03065_b200.synth import _memory_groups, job_footprint, scene_jobs
    scenes = workloads.make_scenes("c4", duration=0.5, n_scenes=6)
    jobs = scene_jobs(scenes)
    fp = [job_footprint(jb, 32) for jb in jobs]
    assert all(b > 0 for b in fp)
    # interval records dominate: 56 B x decimated images x coarse samples
    jb = jobs[0]
    assert fp[0] >= 56 * 2600 * -(-jb.pos.shape[0] // 64)
    groups = _memory_groups(jobs, 2 * max(fp), 32)
    assert [j for g in groups for j in g] == list(range(6))
    assert all(sum(fp[j] for j in g) <= 2 * max(fp) for g in groups) and len(groups) >= 3
    assert _memory_groups(jobs, 1, 32) == [[j] for j in range(6)]  # never empty groups
    assert _memory_groups(jobs, 10 ** 15, 32) == [list(range(6))]


def test_record_groups_partition(monkeypatch):
    """engine._record_groups: consecutive job ranges covering the batch,
    each within the budget when one job fits, None under the budget or for a
    non-uniform layout (host logic; the GPU test checks bit-identity)."""
    import types

    from paper_2508_03065_b200 import engine
    rng = np.random.default_rng(3)
    per_job = rng.integers(1000, 5000, size=37).astype(np.int64)
    kbase = np.concatenate([[0], np.cumsum(per_job)[:-1]])
    geom = types.SimpleNamespace(rec_layout=dict(kbase=kbase, per_job=per_job, sel={}),
                                 n_coarse_total=int(per_job.sum()), jobs=[None] * 37, dev=None)
    monkeypatch.setattr(engine, "RECORD_BUDGET", float(48 * per_job.sum() + 1))
    assert engine._record_groups(geom) is None
    budget = 48 * 20000
    monkeypatch.setattr(engine, "RECORD_BUDGET", float(budget))
    groups = engine._record_groups(geom)
    assert groups[0][0] == 0 and groups[-1][1] == 37
    assert all(a < b for a, b in groups)
    assert all(groups[i][1] == groups[i + 1][0] for i in range(len(groups) - 1))
    assert len(groups) == -(-48 * int(per_job.sum()) // budget)
    sizes = [48 * int(per_job[a:b].sum()) for a, b in groups]
    assert max(sizes) <= 1.3 * budget  # cut at equal record counts, whole jobs
    geom.rec_layout = None
    assert engine._record_groups(geom) is None


def test_work_list_cost_order(monkeypatch):
    """engine._work_list with jobs (order 3): each job's items are a
    permutation of the chunk-major list, jobs stay contiguous, tiles come by
    non-increasing total estimated cost (active images of each chunk over
    the tile) with their chunks adjacent; small grids (the auto rule) keep
    the chunk-major order."""
    from paper_2508_03065_b200 import engine
    monkeypatch.setattr(engine, "WORK_ORDER", 3)
    jobs, rows, n_img, out_len, n_seg = [], [], [], [], []
    for q, (dims, order, T) in enumerate([((6., 4., 3.), 6, 20000), ((9., 7., 3.5), 5, 12000)]):
        jobs.append(engine.Job(s=np.zeros(T, np.float32), pos=np.zeros((T, 3)), mic=np.zeros(3),
                               dims=dims, walls=0.8, max_order=order, tiers=((2, 1), (order, 32)),
                               rate=16000.0))
        S = len(engine._delay_estimates(jobs[-1]))
        tau = engine._delay_estimates(jobs[-1])
        n_img.append(S)
        out_len.append(T + int(np.ceil(tau[-1])) + 32)
        rows.append(dict(ls=T + 31))
        n_seg.append(-(-T // engine.SEG_LEN))
    work, _ = engine._work_list(np.array(n_img), np.array(out_len), n_seg, 148,
                                [dict(r) for r in rows], jobs)
    plain, _ = engine._work_list(np.array(n_img), np.array(out_len), n_seg, 148,
                                 [dict(r) for r in rows])
    assert np.all(np.diff(work[:, 0]) >= 0)  # jobs contiguous, in order
    for j in range(2):
        a, b = work[work[:, 0] == j], plain[plain[:, 0] == j]
        assert sorted(map(tuple, a.tolist())) == sorted(map(tuple, b.tolist()))
        tau, W = engine._delay_estimates(jobs[j]), engine._cost_prefix(jobs[j])
        n0 = a[:, 1].astype(float) * engine.TILE
        lo = np.clip(np.searchsorted(tau, n0 - rows[j]["ls"], side="right"), a[:, 2], a[:, 3])
        hi = np.clip(np.searchsorted(tau, n0 + engine.TILE, side="right"), a[:, 2], a[:, 3])
        cost = (W[hi] - W[lo]) + 0.05 * (a[:, 3] - a[:, 2])
        tc = np.bincount(a[:, 1] - a[:, 1].min(), weights=cost)[a[:, 1] - a[:, 1].min()]
        assert np.all(np.diff(tc) <= 1e-9)  # tiles by total cost
        for t in np.unique(a[:, 1]):  # chunks of a tile adjacent
            idx = np.flatnonzero(a[:, 1] == t)
            assert idx[-1] - idx[0] == len(idx) - 1
    monkeypatch.setattr(engine, "WORK_ORDER", -1)  # auto: these grids are small
    auto, _ = engine._work_list(np.array(n_img), np.array(out_len), n_seg, 148,
                                [dict(r) for r in rows], jobs)
    assert np.array_equal(auto, plain)
