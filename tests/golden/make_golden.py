"""Generate golden vectors from the REFERENCE implementation itself.

Runs only in the build container, where /root/reference (the unmodified
`moverb` package) can be imported; the committed .npz files travel, this
script's inputs do not.  Nothing under tests/ reads /root/reference at test
time.

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Renders use the reference's own functions composed as SURVEY.md 8c (L0):
per-tier low_order_distances / high_order_distances(decimate(traj, N)),
chained merge_streams, then synthesize; moving receivers through the
per-parity-group source transform p' = p + s*(m0 - q(t)).
"""

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from moverb import _kernels, farrow as rfarrow  # noqa: E402
from moverb.room import MicPosition, Room, as_arrays, enumerate_images  # noqa: E402
from moverb.synth import (SynthesisConfig, high_order_distances,  # noqa: E402
                          low_order_distances, merge_streams, synthesize)
from moverb.trajectory import Trajectory, _phase_table, decimate  # noqa: E402

from paper_2508_03065_b200 import workloads  # noqa: E402
from paper_2508_03065_b200.farrow import hann_sinc  # noqa: E402

assert _kernels.using_numba()


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def tier_streams(images, traj, mic, room, tiers):
    streams = None
    prev = -1
    for mo, N in tiers:
        sel = [sp for sp in images if prev < sp.order <= mo]
        prev = mo
        if N == 1:
            st = low_order_distances(sel, traj, mic, room)
        else:
            st = high_order_distances(sel, decimate(traj, N), mic, room, len(traj), N)
        streams = st if streams is None else merge_streams(streams, st)
    return streams


def l0_render(scene, f, mic_index=0, workers=8):
    room = Room(dims=scene.dims, wall_reflection=scene.walls)
    images = enumerate_images(room, scene.max_order)
    mic = scene.mics[mic_index]
    traj = Trajectory(rate=scene.rate, positions=scene.pos)
    if mic.ndim == 1:
        streams = tier_streams(images, traj, MicPosition(pos=mic), room, scene.tiers)
    else:
        m0 = mic[0].copy()
        streams = None
        _, sign, _, _ = as_arrays(images, room)
        groups = {}
        for sp, sg in zip(images, sign):
            groups.setdefault(tuple(sg), []).append(sp)
        for sg, sel in sorted(groups.items()):
            p2 = scene.pos + np.asarray(sg)[None, :] * (m0[None, :] - mic)
            tr = Trajectory(rate=scene.rate, positions=p2)
            st = tier_streams(sel, tr, MicPosition(pos=m0), room, scene.tiers)
            streams = st if streams is None else merge_streams(streams, st)
    cfg = SynthesisConfig(audio_rate=scene.rate, max_order=scene.max_order, workers=workers)
    y = synthesize(np.asarray(scene.s, dtype=np.float64), streams, f, cfg)
    return y, len(images)


def render_cases():
    cases = {
        # name: (workload, overrides, filter)
        "c1": ("c1", dict(), "hann14"),
        "c1_refdesign": ("c1", dict(tiers=((1, 1), (3, 32))), "design"),
        "c2": ("c2", dict(duration=0.25), "hann14"),
        "c3": ("c3", dict(duration=0.1, max_order=8, tiers=((2, 1), (5, 32), (8, 256))), "hann14"),
        "c4": ("c4", dict(duration=0.25, max_order=6, n_scenes=3), "hann14"),
        "c5": ("c5", dict(duration=0.1, max_order=6, n_channels=4,
                          tiers=((2, 1), (4, 32), (6, 256))), "hann14"),
    }
    design = rfarrow.design(3, 8, 0.8)
    for name, (wl, over, fk) in cases.items():
        scenes = workloads.make_scenes(wl, **over)
        out = {}
        ys, lens, nimg = [], [], []
        for sc in scenes:
            f = design if fk == "design" else hann_sinc(sc.fd_taps, 14)
            chans = range(len(sc.mics)) if wl != "c5" else [0, 3]
            for ch in chans:
                y, S = l0_render(sc, f, ch)
                ys.append(y)
                lens.append(y.size)
                nimg.append(S)
        out["y"] = np.concatenate(ys)
        out["lens"] = np.array(lens, np.int64)
        out["n_images"] = np.array(nimg, np.int64)
        out["branches"] = np.asarray(f.branches)
        out["inputs_sha"] = np.array(digest(*[a for sc in scenes for a in (sc.s, sc.pos, *sc.mics)]))
        out["channels"] = np.array([0, 3] if wl == "c5" else [0], np.int64)
        np.savez_compressed(os.path.join(HERE, f"render_{name}.npz"), **out)
        print(name, "out_lens", lens, "images", nimg, "peak", float(np.abs(out["y"]).max()))


def kernel_cases():
    rng = np.random.default_rng(7)
    out = {}
    # enumeration (room.py:108-143 + as_arrays)
    for tag, dims, walls, order in [
        ("a", [5.0, 6.0, 4.0], [0.9] * 6, 4),
        ("b", [6.0, 4.0, 3.0], [0.7, 0.75, 0.8, 0.85, 0.6, 0.9], 5),
        ("c", [20.0, 15.0, 8.0], [0.9] * 6, 0),
    ]:
        room = Room(dims=np.array(dims), wall_reflection=np.array(walls))
        specs = enumerate_images(room, order)
        off, sign, beta, ordr = as_arrays(specs, room)
        out[f"enum_{tag}_dims"] = np.array(dims)
        out[f"enum_{tag}_walls"] = np.array(walls)
        out[f"enum_{tag}_order"] = np.array(order)
        out[f"enum_{tag}_offset"] = off
        out[f"enum_{tag}_sign"] = sign
        out[f"enum_{tag}_beta"] = beta
        out[f"enum_{tag}_ord"] = ordr
        out[f"enum_{tag}_lattice"] = np.array([s.lattice for s in specs], np.int64)
        out[f"enum_{tag}_parity"] = np.array([s.parity for s in specs], np.int64)
    # distance kernel (_kernels.py:54-62)
    offset = rng.normal(size=(9, 3)) * 10
    sign = np.where(rng.random((9, 3)) < 0.5, -1.0, 1.0)
    mic = rng.random(3) * 4
    pos = rng.random((300, 3)) * 5
    d = np.empty((9, 300))
    _kernels._distance_numba(offset, sign, mic, pos, d)
    out.update(dist_offset=offset, dist_sign=sign, dist_mic=mic, dist_pos=pos, dist_out=d)
    # accumulate kernel (_kernels.py:109-123) with the default design(3,8,.8)
    f = rfarrow.design(3, 8, 0.8)
    x = rng.standard_normal(700)
    streams = rfarrow.branch_filter(x, f)
    tau = 3.0 + 40.0 * rng.random((5, 760))
    amp = rng.random((5, 760))
    acc = np.zeros(760)
    _kernels._accumulate_numba(acc, streams, tau, amp, f.branch_len, f.nominal_delay)
    out.update(acc_x=x, acc_streams=streams, acc_tau=tau, acc_amp=amp, acc_out=acc,
               design_3_8_08=np.asarray(f.branches))
    # upsample kernel (_kernels.py:164-181) and phase tables (trajectory.py:235-257)
    for N in (16, 64):
        coarse = rng.normal(size=40).cumsum()
        tab = _phase_table(N)
        up = np.empty(40 * N + 17)
        _kernels._upsample_numba(coarse, tab, N, up)
        out[f"up{N}_coarse"] = coarse
        out[f"up{N}_out"] = up
        out[f"table{N}"] = np.asarray(tab)
    # decimate (trajectory.py:279-298), one case with the anti-alias branch
    t = np.arange(4000) / 1000.0
    slow = np.stack([2 + 0.5 * np.sin(2 * np.pi * 0.7 * t), 2 + 0.3 * np.cos(2 * np.pi * 0.4 * t),
                     1.5 + 0 * t], axis=1)
    fast = np.stack([2 + 0.5 * np.sin(2 * np.pi * 30.0 * t), 2 + 0.3 * np.cos(2 * np.pi * 0.4 * t),
                     1.5 + 0 * t], axis=1)
    for tag, p, N in [("slow", slow, 50), ("fast", fast, 20)]:
        tr = decimate(Trajectory(rate=1000.0, positions=p), N)
        out[f"dec_{tag}_in"] = p
        out[f"dec_{tag}_N"] = np.array(N)
        out[f"dec_{tag}_out"] = tr.positions
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)
    print("kernels.npz written")


def source_modulation_case():
    """synth.py:228-242: gain applied at emission time (validation switch)."""
    from dataclasses import replace
    sc = workloads.make_scenes("c1", duration=0.25, tiers=((1, 1), (3, 32)))[0]
    f = rfarrow.design(3, 8, 0.8)
    room = Room(dims=sc.dims, wall_reflection=sc.walls)
    images = enumerate_images(room, sc.max_order)
    traj = Trajectory(rate=sc.rate, positions=sc.pos)
    streams = tier_streams(images, traj, MicPosition(pos=sc.mics[0]), room, sc.tiers)
    cfg = SynthesisConfig(audio_rate=sc.rate, max_order=sc.max_order, modulate="source")
    y = synthesize(np.asarray(sc.s, dtype=np.float64), streams, f, cfg)
    np.savez_compressed(os.path.join(HERE, "render_c1_source.npz"), y=y,
                        branches=np.asarray(f.branches),
                        inputs_sha=np.array(digest(sc.s, sc.pos, sc.mics[0])))
    print("c1_source out_len", y.size)


def static_cases():
    """reference.py:67-251: static_rir, static_render (direct and FFT
    branches), splice_baseline (butt-joined, cross-faded, short last block)
    and compare, on the reference test suite's room and mic."""
    from moverb import reference as rref
    room = Room(dims=np.array([5.0, 6.0, 4.0]), wall_reflection=np.full(6, 0.9))
    mic = MicPosition(pos=np.array([1.25, 2.6, 2.75]))
    rate = 16000.0
    out = {}
    srcs = {"far": np.array([2.0, 3.5, 2.0]), "near": np.array([1.5, 2.8, 2.5]),
            "corner": np.array([0.3, 5.6, 0.4])}
    for tag, src in srcs.items():
        for order in (0, 2, 3):
            r = rref.static_rir(room, src, mic, rate, order)
            out[f"rir_{tag}_{order}"] = r.taps
            out[f"rir_{tag}_{order}_count"] = np.array(r.image_count)
    rng = np.random.default_rng(11)
    x_small = rng.standard_normal(1600)   # 1600 * 638 < 5e6: np.convolve
    x_large = rng.standard_normal(16000)  # > 5e6 products: fftconvolve
    out["x_small"], out["x_large"] = x_small, x_large
    rir = rref.static_rir(room, srcs["far"], mic, rate, 2)
    out["render_small"] = rref.static_render(x_small, rir)
    out["render_large"] = rref.static_render(x_large, rir)
    n = 4000
    t = np.arange(n) / rate
    pos = np.stack([1.0 + 0.9 * t, np.full(n, 3.0), np.full(n, 2.0)], axis=1)
    traj = Trajectory(rate=rate, positions=pos)
    x = np.sin(2 * np.pi * 700.0 * t) + 0.3 * rng.standard_normal(n)
    out["splice_x"], out["splice_pos"] = x, pos
    cfg = SynthesisConfig(max_order=2, decimation=1)
    for hop, cf in ((640, 0), (640, 128), (640, 200), (600, 100), (1000, 1000)):
        out[f"splice_{hop}_{cf}"] = rref.splice_baseline(x, traj, room, mic, hop, cf, cfg)
    a = out["splice_640_0"]
    b = out["splice_640_128"]
    for tag, (u, v, kw) in {"ab": (a, b, dict(passband=0.8, rate=rate, interior=0.05)),
                            "aa": (a, a, dict(passband=1.0, rate=rate, interior=0.1)),
                            "noisy": (b + 1e-3 * rng.standard_normal(b.size), b,
                                      dict(passband=0.9, rate=rate, interior=0.0))}.items():
        rep = rref.compare(u, v, **kw)
        out[f"cmp_{tag}_a"], out[f"cmp_{tag}_b"] = u, v
        out[f"cmp_{tag}_snr"] = np.array(rep.snr_db)
        out[f"cmp_{tag}_jump"] = np.array(rep.envelope_max_jump)
        out[f"cmp_{tag}_track"] = rep.inst_freq_track
    np.savez_compressed(os.path.join(HERE, "static.npz"), **out)
    print("static.npz written")


def cli_cases():
    """reference cli.py simulate (4 modes, --dump-image) and compare, run
    through the reference's own main() on files written here; inputs and
    outputs land in tests/golden/cli/."""
    import shutil
    import tempfile
    from moverb import cli as rcli, io_formats as rio
    out_dir = os.path.join(HERE, "cli")
    os.makedirs(out_dir, exist_ok=True)
    rate = 16000.0
    n = 4000
    t = np.arange(n) / rate
    pos = np.stack([1.0 + 0.8 * t, 3.0 + 0.3 * t, np.full(n, 2.0)], axis=1)
    rng = np.random.default_rng(21)
    x = (0.5 * np.sin(2 * np.pi * 440.0 * t) + 0.2 * rng.standard_normal(n)).astype(np.float32)
    tmp = tempfile.mkdtemp()
    rio.write_trajectory(os.path.join(tmp, "path.txt"), Trajectory(rate=rate, positions=pos))
    rio.write_wav(os.path.join(tmp, "dry.wav"), rate, x)
    cfg = ("room.dims = 5 6 4\nroom.reflection = 0.9\nmic.pos = 1.25 2.6 2.75\n"
           "traj.file = {tmp}/path.txt\nsynth.rate = 16000\nsynth.N = 64\nsynth.K = 1\n"
           "synth.max_order = 3\n")
    with open(os.path.join(tmp, "run.cfg"), "w") as fh:
        fh.write(cfg.format(tmp=tmp))
    for mode, extra in (("hierarchical", ["--dump-image", "7", "--dump-csv",
                                          os.path.join(tmp, "image7.csv")]),
                        ("oracle", []), ("splice", ["--crossfade", "64"]), ("static", [])):
        rc = rcli.main(["simulate", "--config", os.path.join(tmp, "run.cfg"), "--mode", mode,
                        "--in", os.path.join(tmp, "dry.wav"),
                        "--out", os.path.join(tmp, f"{mode}.wav")] + extra)
        assert rc == 0, mode
    rc = rcli.main(["compare", os.path.join(tmp, "hierarchical.wav"), os.path.join(tmp, "oracle.wav"),
                    "--report", os.path.join(tmp, "report.txt")])
    assert rc == 0
    for name in ("path.txt", "dry.wav", "hierarchical.wav", "oracle.wav", "splice.wav",
                 "static.wav", "image7.csv", "report.txt"):
        shutil.copy(os.path.join(tmp, name), os.path.join(out_dir, name))
    with open(os.path.join(out_dir, "run.cfg"), "w") as fh:
        fh.write(cfg.replace("{tmp}", "{dir}"))
    print("cli fixtures written")


if __name__ == "__main__":
    import sys as _sys
    if "--source-only" in _sys.argv:
        source_modulation_case()
    elif "--static-only" in _sys.argv:
        static_cases()
    elif "--cli-only" in _sys.argv:
        cli_cases()
    else:
        cli_cases()
        static_cases()
        kernel_cases()
        render_cases()
        source_modulation_case()
