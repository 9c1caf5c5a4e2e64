"""Hierarchical moving-image-source synthesis -- the drop-in API.

Mirrors reference synth.py (SynthesisConfig :43-91, DelayStreams :94-119,
prepare_streams :273-288, synthesize :194-258, render :291-294,
select_images :261-270, cost_report :302-331, BudgetError :39-40) and
reference.py:116-130 (full_rate_moving_oracle).  Same validation and
ValueError behaviour; numpy in, float64 numpy out.

Differences, all opt-in through new SynthesisConfig fields:
  tiers      ((max_order, N), ...) any number of hierarchical rates; the
             reference's (order_split, decimation) is the 2-tier default.
  modulate   "receiver" (default) on both engines; "source" (the reference's
             validation switch) on the exact path, one branch pass per image.
  precision  "fp64": the exact engine (reference arithmetic and summation
             order, bit-faithful); "fp32": the fused B200 fast path
             (max error ~1e-6 of the output peak); "auto" (default): fp32
             when the dry signal is float32, fp64 otherwise.
A moving receiver is accepted as a (T, 3) array in place of the mic.
`workers` is accepted and ignored (the GPU schedules itself).
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib, engine
from ._dev import require_cuda
from .farrow import as_filter
from .room import as_arrays, as_mic, image_count, image_table

SUMMATION_BLOCK = 32


class BudgetError(RuntimeError):
    """Raised when a requested render exceeds the configured evaluation cap."""


@dataclass(frozen=True)
class SynthesisConfig:
    audio_rate: float = 16000.0
    order_split: int = 1
    decimation: int = 3200
    max_order: int = 3
    t60: float = None
    sound_speed: float = 343.0
    d_min: float = 0.05
    summation: str = "pairwise"
    modulate: str = "receiver"
    workers: int = 1
    eval_budget: float = 2.0e9
    tiers: tuple = None
    precision: str = "auto"

    def __post_init__(self):
        if self.audio_rate <= 0:
            raise ValueError("audio_rate must be > 0")
        if self.decimation < 1 or int(self.decimation) != self.decimation:
            raise ValueError("decimation must be a positive integer")
        if self.order_split < 0:
            raise ValueError("order_split must be >= 0")
        if self.max_order < 0:
            raise ValueError("max_order must be >= 0")
        if self.t60 is not None and self.t60 <= 0:
            raise ValueError("t60 must be > 0 when set")
        if self.sound_speed <= 0:
            raise ValueError("sound_speed must be > 0")
        if self.d_min <= 0:
            raise ValueError("d_min must be > 0")
        if self.summation != "pairwise":
            raise ValueError("summation policy must be 'pairwise'")
        if self.modulate not in ("receiver", "source"):
            raise ValueError("modulate must be 'receiver' or 'source'")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.eval_budget <= 0:
            raise ValueError("eval_budget must be > 0")
        if self.precision not in ("auto", "fp32", "fp64"):
            raise ValueError("precision must be 'auto', 'fp32' or 'fp64'")
        if self.tiers is not None:
            tiers = tuple((int(a), int(b)) for a, b in self.tiers)
            engine._validate_tiers(tiers, self.max_order)
            object.__setattr__(self, "tiers", tiers)

    def tier_table(self) -> tuple:
        """((max_order, N), ...): explicit tiers, else the reference's split
        (orders <= order_split at full rate, the rest decimated by N)."""
        if self.tiers is not None:
            return self.tiers
        if self.order_split >= self.max_order:
            return ((self.max_order, 1),)
        return ((self.order_split, 1), (self.max_order, int(self.decimation)))


def _canonical_index(specs, room, max_order) -> np.ndarray:
    """Positions of `specs` (ImageSourceSpec list) in the canonical order."""
    t = image_table(room.dims, room.wall_reflection, max_order)
    lat = t.lattice[0].cpu().numpy()
    par = t.parity[0].cpu().numpy()
    where = {(tuple(lat[i]), tuple(par[i])): i for i in range(lat.shape[0])}
    idx = []
    for sp in specs:
        k = (tuple(int(v) for v in sp.lattice), tuple(int(bool(v)) for v in sp.parity))
        if k not in where:
            raise ValueError("image spec beyond max_order")
        idx.append(where[k])
    idx = np.asarray(idx, dtype=np.int64)
    return np.sort(idx)  # merge_streams restores canonical order (synth.py:161-179)


class DelayStreams:
    """Per-image distance tracks plus the specs they belong to (reference
    synth.py:94-119): rate, specs, d (S, T) metres at `rate`, eval_count,
    tau(cfg), amplitude(cfg), image_count().

    Built by low_order_distances / high_order_distances / merge_streams or
    directly like the reference's dataclass; `d` may be a numpy array or a
    CUDA float64 tensor (the stream builders keep it on the device and
    materialise the numpy view only when `.d` is read).
    """

    def __init__(self, rate, specs, d, eval_count=0):
        self.rate = float(rate)
        self._specs = list(specs)
        self._d = d
        self.eval_count = int(eval_count)

    @property
    def specs(self):
        return self._specs

    def image_count(self):
        return len(self._specs)

    @property
    def d(self) -> np.ndarray:
        if isinstance(self._d, torch.Tensor):
            self._d = self._d.cpu().numpy()
        return self._d

    def d_dev(self, device=None) -> torch.Tensor:
        """(S, T) float64 tracks on the device."""
        if isinstance(self._d, torch.Tensor) and self._d.is_cuda:
            return self._d
        from ._dev import to_dev
        return to_dev(np.asarray(self._d, dtype=np.float64), torch.float64, require_cuda(device))

    def beta_dev(self, device=None) -> torch.Tensor:
        from ._dev import to_dev
        return to_dev(np.array([sp.beta for sp in self.specs], dtype=np.float64), torch.float64,
                      require_cuda(device))

    def tau(self, cfg):
        return self.rate * self.d / cfg.sound_speed

    def amplitude(self, cfg):
        beta = np.array([s.beta for s in self.specs])
        return beta[:, None] / (4.0 * np.pi * np.maximum(self.d, cfg.d_min))


class GeometryStreams(DelayStreams):
    """prepare_streams' result: the tracks of one render held by the engine
    (coarse tier tracks and interpolation records on the device); `specs`
    and `d` are materialised only when read."""

    def __init__(self, geometry, rate, room, max_order, index):
        self.geometry = geometry
        self.rate = float(rate)
        self._room = room
        self._max_order = max_order
        self._index = index
        self._specs = None
        self._d = None
        self.eval_count = geometry.eval_count[0] if geometry is not None else 0

    @property
    def specs(self):
        if self._specs is None:
            from .room import enumerate_images
            full = enumerate_images(self._room, self._max_order)
            self._specs = [full[i] for i in self._index] if self._index is not None else full
        return self._specs

    def image_count(self):
        return 0 if self.geometry is None else int(self.geometry.n_img[0])

    @property
    def d(self) -> np.ndarray:
        if self._d is None:
            self._d = materialize_tracks(self.geometry)
        return self._d

    def d_dev(self, device=None) -> torch.Tensor:
        return materialize_tracks_dev(self.geometry)

    def beta_dev(self, device=None) -> torch.Tensor:
        g = self.geometry
        S = int(g.n_img[0])
        return g.images[int(g.img_off[0]):int(g.img_off[0]) + S].view(torch.float64)[:, 3]


# ---------------------------------------------------------------------------
# stream builders (reference synth.py:122-179): materialised per-image tracks
def _mic_pos(mic):
    return np.asarray(mic.pos if hasattr(mic, "pos") else mic, dtype=np.float64)


def low_order_distances(images, traj, mic, room) -> DelayStreams:
    """Exact per-sample distances of `images` along `traj` (reference
    synth.py:122-130), one libmvb distance pass; eval_count = S * T."""
    from . import kernels
    if not images:
        return DelayStreams(traj.rate, [], np.zeros((0, len(traj))))
    offset, sign, _, _ = as_arrays(images, room)
    dev = require_cuda()
    d = kernels.distance_streams(torch.from_numpy(offset).to(dev), sign, _mic_pos(mic),
                                 traj.positions)
    return DelayStreams(traj.rate, list(images), d, eval_count=d.numel())


def high_order_distances(images, traj_coarse, mic, room, out_len, factor) -> DelayStreams:
    """Distances on the coarse path, band-limit upsampled by `factor` to
    out_len samples (reference synth.py:133-158): factor 1 truncates or
    hold-extends; eval_count counts the coarse evaluations."""
    from . import kernels
    from ._dev import ptr, stream_handle
    from .trajectory import phase_table
    out_len, factor = int(out_len), int(factor)
    if not images:
        return DelayStreams(traj_coarse.rate * factor, [], np.zeros((0, out_len)))
    offset, sign, _, _ = as_arrays(images, room)
    dev = require_cuda()
    coarse = kernels.distance_streams(torch.from_numpy(offset).to(dev), sign, _mic_pos(mic),
                                      traj_coarse.positions)
    S, K = coarse.shape
    if factor == 1:
        d = coarse[:, :out_len]
        if K < out_len:
            d = torch.cat([d, d[:, -1:].expand(S, out_len - K)], dim=1)
        d = d.contiguous()
    else:
        tab = torch.from_numpy(np.array(phase_table(factor))).to(dev)
        d = torch.empty(S, out_len, dtype=torch.float64, device=dev)
        _lib.call("mvb_upsample_streams", ptr(coarse), S, K, ptr(tab), factor, tab.shape[1],
                  out_len, ptr(d), stream_handle(dev))
    return DelayStreams(traj_coarse.rate * factor, list(images), d, eval_count=coarse.numel())


def merge_streams(low: DelayStreams, high: DelayStreams) -> DelayStreams:
    """Union of two stream sets, rows restored to enumeration order
    (reference synth.py:161-179; same errors, an empty side returns the
    other unchanged)."""
    if low.image_count() == 0:
        return high
    if high.image_count() == 0:
        return low
    if low.rate != high.rate:
        raise ValueError("stream rates differ")
    da, db = low.d_dev(), high.d_dev()
    if da.shape[1] != db.shape[1]:
        raise ValueError("stream lengths differ")
    specs = list(low.specs) + list(high.specs)
    order = sorted(range(len(specs)), key=lambda i: specs[i])
    d = torch.cat([da, db], dim=0)[torch.as_tensor(order, device=da.device)]
    return DelayStreams(low.rate, [specs[i] for i in order], d,
                        eval_count=low.eval_count + high.eval_count)


def materialize_tracks(geom) -> np.ndarray:
    """(S, T) fp64 tracks of job 0 in canonical order (numpy)."""
    if geom is None:
        return np.zeros((0, 0))
    return materialize_tracks_dev(geom).cpu().numpy()


def materialize_tracks_dev(geom) -> torch.Tensor:
    """(S, T) fp64 tracks of job 0 in canonical order, computed on the GPU
    with the reference kernels (distance_streams / upsample_stream)."""
    from . import _lib
    from ._dev import ptr, stream_handle
    dev = geom.dev
    S, T = int(geom.n_img[0]), int(geom.T[0])
    img = geom.images[int(geom.img_off[0]):int(geom.img_off[0]) + S]
    f64 = img.view(torch.float64)
    i32 = img[:, 6:7].view(torch.int32)
    factor = i32[:, 0].cpu().numpy()
    coarse_off = img[:, 7].cpu().numpy()
    K = i32[:, 1].cpu().numpy()
    out = torch.empty(S, T, dtype=torch.float64, device=dev)
    st = stream_handle(dev)
    full = np.nonzero(factor == 1)[0]
    if full.size:
        sel = torch.as_tensor(full, device=dev)
        off = f64[sel, 0:3].contiguous()
        sg = img[sel, 4:6].view(torch.float32)[:, 0:3].to(torch.float64).contiguous()
        res = torch.empty(full.size, T, dtype=torch.float64, device=dev)
        if geom.moving[0]:
            raise NotImplementedError("materialising tracks of a moving receiver")
        mic = geom.paths[int(geom.mic_off[0])].contiguous()
        pos = geom.paths[int(geom.pos_off[0]):int(geom.pos_off[0]) + T].contiguous()
        _lib.call("mvb_distance_streams", ptr(off), ptr(sg), ptr(mic), ptr(pos), full.size, T,
                  ptr(res), st)
        out[sel] = res
    from .trajectory import phase_table
    for N in sorted(set(factor.tolist()) - {1}):
        rows = np.nonzero(factor == N)[0]
        tab = torch.from_numpy(np.array(phase_table(int(N)))).to(dev)
        k = int(K[rows[0]])
        idx = torch.as_tensor(coarse_off[rows], device=dev)[:, None] + torch.arange(k, device=dev)
        coarse = geom.coarse[idx].contiguous()
        res = torch.empty(rows.size, T, dtype=torch.float64, device=dev)
        _lib.call("mvb_upsample_streams", ptr(coarse), rows.size, k, ptr(tab), int(N), 65, T,
                  ptr(res), st)
        out[torch.as_tensor(rows, device=dev)] = res
    return out


def _check_receiver(mic, room, T):
    m = mic.pos if hasattr(mic, "pos") else np.asarray(mic, dtype=np.float64)
    if m.ndim == 1:
        as_mic(m).require_inside(room)
        return m
    if m.shape != (T, 3):
        raise ValueError("a moving receiver must be a (T, 3) path")
    if not (np.all(m > 0) and np.all(m < room.dims)):
        raise ValueError("mic path must stay strictly inside the room")
    return m


def select_images(room, traj, mic, cfg):
    """Canonical image indices kept for a render (t60 cull at the start
    position, reference synth.py:261-270); None = all images."""
    if cfg.t60 is None:
        return None
    from .kernels import distance_streams
    t = image_table(room.dims, room.wall_reflection, cfg.max_order)
    m = np.asarray(mic if not hasattr(mic, "pos") else mic.pos, dtype=np.float64)
    m0 = m if m.ndim == 1 else m[0]
    d = distance_streams(t.offset[0], t.sign[0], torch.tensor(np.array(m0), device=t.offset.device),
                         torch.tensor(np.array(traj.positions[:1]), device=t.offset.device))[:, 0]
    keep = (d <= cfg.sound_speed * cfg.t60).nonzero().squeeze(1).cpu().numpy()
    return keep.astype(np.int64)


def prepare_streams(traj, room, mic, cfg, images=None) -> DelayStreams:
    """Device tracks of every image (reference synth.py:273-288), for any
    tier table."""
    if traj.rate != cfg.audio_rate:
        raise ValueError("trajectory rate must equal the audio rate")
    m = _check_receiver(mic, room, len(traj))
    if images is not None:
        index = _canonical_index(images, room, cfg.max_order) if len(images) else np.zeros(0, np.int64)
    else:
        index = select_images(room, traj, m, cfg)
    if index is not None and index.size == 0:
        return GeometryStreams(None, traj.rate, room, cfg.max_order, index)
    job = engine.Job(s=None, pos=traj.positions, mic=m, dims=room.dims, walls=room.wall_reflection,
                     max_order=cfg.max_order, tiers=cfg.tier_table(), rate=traj.rate,
                     c=cfg.sound_speed, d_min=cfg.d_min, image_index=index)
    geom = engine.Geometry([job])
    return GeometryStreams(geom, traj.rate, room, cfg.max_order, index)


def _precision(s, cfg) -> str:
    if cfg.precision != "auto":
        return cfg.precision
    dt = s.dtype if hasattr(s, "dtype") else np.asarray(s).dtype
    return "fp32" if dt in (np.float32, torch.float32) else "fp64"


def _check_signal(s):
    a = s.detach().cpu().numpy() if isinstance(s, torch.Tensor) else np.asarray(s)
    if a.ndim != 1 or a.size == 0:
        raise ValueError("input must be a nonempty 1-D signal")
    if not np.all(np.isfinite(a)):
        raise ValueError("input must be finite")
    return a


def synthesize(s, streams: DelayStreams, f, cfg) -> np.ndarray:
    """Render s through the moving image set (reference synth.py:194-258).
    Output length len(s) + ceil(max delay) + L, float64.

    prepare_streams' engine-held tracks render on the fused engine (fp32 or
    the exact fp64 one, `cfg.precision`); materialised track sets (the
    stream builders, or a DelayStreams built by hand) and modulate="source"
    render on the exact fp64 track path, the reference's own algorithm."""
    a = _check_signal(s)
    filt = as_filter(f)
    if streams.image_count() == 0:
        return np.zeros(a.size + filt.branch_len)
    geom = getattr(streams, "geometry", None)
    if cfg.modulate == "source" or geom is None:
        return _synthesize_tracks(a, streams, filt, cfg)
    prec = _precision(a, cfg)
    res = engine.render(geom, [a], filt, precision=prec)
    from ._staging import d2h
    return d2h(res.job(0), np.float64)


def _synthesize_tracks(x, streams, f, cfg) -> np.ndarray:
    """Exact fp64 synthesis from (S, T) tracks on the device, reference
    synth.py:211-258 step for step: hold-extend the tracks to the output
    length, tau/amplitude per sample, one branch pass (kernels.branch_filter)
    and one accumulate_images call per 32-image block, pairwise block merge.
    modulate="source" (synth.py:228-242, the reference's validation switch)
    applies the gain at emission time instead: one branch pass per image of
    its gain-modulated input.  Materialises (S, out_len) tracks like the
    reference, so it is meant for validation-size renders."""
    from . import kernels
    dev = require_cuda()
    d = streams.d_dev(dev)
    S, T = d.shape
    xs = torch.from_numpy(np.array(x, dtype=np.float64)).to(dev)
    tau_max = streams.rate * float(d.max().item()) / cfg.sound_speed
    out_len = x.size + int(np.ceil(tau_max)) + f.branch_len
    d_ext = torch.cat([d, d[:, -1:].expand(S, out_len - T)], dim=1) if T < out_len else d[:, :out_len]
    d_ext = d_ext.contiguous()
    # divide by a device tensor: torch turns `tensor / python scalar` into a
    # multiply by the reciprocal, which is not the reference's rounding
    c = torch.tensor(cfg.sound_speed, dtype=torch.float64, device=dev)
    tau = (streams.rate * d_ext) / c
    beta = streams.beta_dev(dev)
    amp = beta[:, None] / (4.0 * np.pi * torch.clamp_min(d_ext, cfg.d_min))
    branches = torch.from_numpy(np.array(f.branches)).to(dev)
    buffers = []
    if cfg.modulate == "source":
        ones = torch.ones(1, out_len, dtype=torch.float64, device=dev)
        for b0 in range(0, S, SUMMATION_BLOCK):
            buf = torch.zeros(out_len, dtype=torch.float64, device=dev)
            for i in range(b0, min(b0 + SUMMATION_BLOCK, S)):
                v = kernels.branch_filter((xs * amp[i, :x.size]).contiguous(), branches)
                kernels.accumulate_images(buf, v, tau[i:i + 1], ones, f.branch_len,
                                          f.nominal_delay)
            buffers.append(buf)
    else:
        v = kernels.branch_filter(xs, branches)
        for b0 in range(0, S, SUMMATION_BLOCK):
            b1 = min(b0 + SUMMATION_BLOCK, S)
            buf = torch.zeros(out_len, dtype=torch.float64, device=dev)
            kernels.accumulate_images(buf, v, tau[b0:b1].contiguous(), amp[b0:b1].contiguous(),
                                      f.branch_len, f.nominal_delay)
            buffers.append(buf)
    while len(buffers) > 1:  # synth.py:182-191
        merged = [buffers[k] + buffers[k + 1] for k in range(0, len(buffers) - 1, 2)]
        if len(buffers) % 2:
            merged.append(buffers[-1])
        buffers = merged
    return buffers[0].cpu().numpy()


_PLANS: dict = {}  # render(): the one cached RenderPlan, keyed by structure
_SEEN: list = [None]  # structure key of the previous render() call


def release_plans() -> None:
    """Drop render()'s cached CUDA-graph plan (and the device memory it holds)."""
    _PLANS.clear()
    _SEEN[0] = None


def _plan_render(a, traj, room, m, f, cfg):
    """render() through a cached RenderPlan when the same structure is seen
    twice in a row (loops over signals / paths); None when not applicable."""
    import os
    if os.environ.get("MVB_PLAN_CACHE", "1") == "0" or cfg.modulate != "receiver" \
            or cfg.t60 is not None:
        return None
    from .plan import RenderPlan, structure_key
    prec = _precision(a, cfg)
    job = engine.Job(s=a, pos=traj.positions, mic=m, dims=room.dims, walls=room.wall_reflection,
                     max_order=cfg.max_order, tiers=cfg.tier_table(), rate=traj.rate,
                     c=cfg.sound_speed, d_min=cfg.d_min)
    key = structure_key([job], f, prec)
    plan = _PLANS.get(key)
    if plan is None:
        if _SEEN[0] != key:
            _SEEN[0] = key
            return None
        _PLANS.clear()
        plan = _PLANS[key] = RenderPlan([job], f, precision=prec)
    from ._staging import d2h
    return d2h(plan.run([job]).job(0), np.float64)


def render(s, traj, room, mic, f, cfg) -> np.ndarray:
    """End-to-end: trajectory in, reverberant moving-source audio out.
    Repeated calls with the same structure (shapes, room, orders, tiers,
    filter, precision) replay a cached CUDA-graph plan from the second
    repeat on (plan.RenderPlan; `release_plans()` frees it, environment
    MVB_PLAN_CACHE=0 disables it)."""
    a = _check_signal(s)
    if traj.rate != cfg.audio_rate:
        raise ValueError("trajectory rate must equal the audio rate")
    m = _check_receiver(mic, room, len(traj))
    y = _plan_render(a, traj, room, m, as_filter(f), cfg)
    if y is not None:
        return y
    return synthesize(s, prepare_streams(traj, room, mic, cfg), f, cfg)


def full_rate_moving_oracle(s, traj, room, mic, f, cfg):
    """Every image's distance at every sample (reference.py:116-130)."""
    evals = image_count(cfg.max_order) * len(traj)
    if evals > cfg.eval_budget:
        raise BudgetError(f"oracle render needs {evals:.3g} distance evaluations, "
                          f"budget is {cfg.eval_budget:.3g}")
    return render(s, traj, room, mic, f, replace(cfg, decimation=1, tiers=((cfg.max_order, 1),)))


def _count_order_leq(k):
    return 1 + sum(4 * o * o + 2 for o in range(1, k + 1))


def cost_report(cfg, images, duration):
    """Distance-evaluation counts, brute force vs hierarchical (reference
    synth.py:302-331), for any tier table."""
    n = int(round(duration * cfg.audio_rate))
    tiers = cfg.tier_table()
    if isinstance(images, int):
        total = images
        per_tier, prev, left = [], -1, images
        for mo, N in tiers:
            c = min(left, _count_order_leq(mo) - (_count_order_leq(prev) if prev >= 0 else 0))
            per_tier.append((c, N))
            left -= c
            prev = mo
        if left > 0:
            per_tier[-1] = (per_tier[-1][0] + left, per_tier[-1][1])
    else:
        total = len(images)
        per_tier, prev = [], -1
        for mo, N in tiers:
            per_tier.append((sum(1 for sp in images if prev < sp.order <= mo), N))
            prev = mo
    low = sum(c for c, N in per_tier if N == 1)
    high = total - low
    hier = sum(c * (n if N == 1 else -(-n // N)) for c, N in per_tier)
    high_hier = sum(c * -(-n // N) for c, N in per_tier if N != 1)
    naive = total * n
    return {
        "images_total": total,
        "images_low": low,
        "images_high": high,
        "samples": n,
        "naive_evals": naive,
        "hierarchical_evals": hier,
        "reduction_ratio": naive / hier if hier else float("inf"),
        "high_order_reduction": (high * n / high_hier) if high_hier else float("inf"),
    }


# ----------------------------------------------------------------------------
# batched, device-resident entry points (benchmarks, multi-scene workloads)


def scene_jobs(scenes, channels=None) -> list:
    """workloads.Scene list -> engine.Job list (one job per (scene, mic))."""
    jobs = []
    for q, sc in enumerate(scenes):
        chans = range(len(sc.mics)) if channels is None else channels
        for ch in chans:
            jobs.append(engine.Job(s=sc.s, pos=sc.pos, mic=sc.mics[ch], dims=sc.dims, walls=sc.walls,
                                   max_order=sc.max_order, tiers=sc.tiers, rate=sc.rate,
                                   signal_key=("scene", q), path_key=("scene", q)))
    return jobs


def job_footprint(jb, fd_taps: int = 64) -> int:
    """Estimated device bytes of one job in a render: coarse tracks (8 B)
    and interval records (48 B) per decimated image per coarse sample, the
    image records (96 B, plus the delay-sorted copy per 16384-sample
    segment), branch records (32 B per padded input row), paths and output."""
    T = int(jb.pos.shape[0]) if hasattr(jb.pos, "shape") else len(jb.pos)
    n_sig = T if jb.s is None else (int(jb.s.numel()) if isinstance(jb.s, torch.Tensor)
                                    else int(np.size(jb.s)))
    moving = len(getattr(jb.mic, "shape", np.shape(jb.mic))) > 1
    prev, inter, imgs = -1, 0, 0
    for mo, N in jb.tiers:
        cnt = image_count(int(mo)) - (image_count(prev) if prev >= 0 else 0)
        if jb.image_index is not None:
            cnt = int(np.sum((np.asarray(jb.image_index) >= (image_count(prev) if prev >= 0 else 0))
                             & (np.asarray(jb.image_index) < image_count(int(mo)))))
        imgs += cnt
        if int(N) > 1:
            inter += cnt * -(-T // int(N))
        prev = int(mo)
    n_seg = -(-T // engine.SEG_LEN)
    reach = 2 * (int(jb.max_order) + 2) * float(np.max(jb.dims)) * float(jb.rate) / float(jb.c)
    return int(56 * inter + 96 * imgs * (1 + n_seg) + 8 * imgs * n_seg
               + 32 * (n_sig + 2 * reach + fd_taps) + 24 * T * (1 + moving) + 8 * (n_sig + reach))


def _memory_groups(jobs, budget: int, fd_taps: int) -> list:
    """Consecutive job groups whose estimated footprints fit `budget`."""
    groups, cur, used = [], [], 0
    for j, jb in enumerate(jobs):
        b = job_footprint(jb, fd_taps)
        if cur and used + b > budget:
            groups.append(cur)
            cur, used = [], 0
        cur.append(j)
        used += b
    if cur:
        groups.append(cur)
    return groups


def shard_batches(jobs, shard, budget: int, fd_taps: int) -> tuple:
    """(sub-batch groups, the jobs this rank renders).  The groups are cut
    from the UNSHARDED jobs: a shard's footprint is rank-specific (delay
    bands equalise cost, not image count), so groups cut after sharding
    could differ between ranks and mismatch their collectives (every group
    all-reduces its track maxima)."""
    groups = _memory_groups(jobs, budget, fd_taps)
    if shard is not None and int(shard[1]) > 1:
        from . import parallel
        jobs = parallel.shard_jobs(jobs, int(shard[0]), int(shard[1]), parallel.shard_kind(shard))
    return groups, jobs


def render_jobs(jobs, f, precision="fp32", shard=None, signals=None, timing=None,
                inputs_ready=None, dmax_hook=None, max_batch_bytes=None):
    """Geometry + render of a job batch; returns engine.RenderResult
    (device output, per-job offsets/lengths, update count, launches).
    `inputs_ready` (optional CUDA event): the jobs' device tensors are final
    once it completes -- lets planning overlap earlier work on the stream.
    `shard=(rank, world)`: render the image shard of `rank` of every job
    (parallel.image_shard: per-tier delay bands; all per-image work divides
    by world); `shard=(rank, world, "time")`: its output window
    (parallel.time_window: all images, 1/world of the samples),
    with out_len from the batch-wide track maximum (all-reduce MAX over
    the ranks, or `dmax_hook` when given) so the ranks' outputs sum to the
    full render.  Batches whose estimated device footprint exceeds
    `max_batch_bytes` (default: 40% of the GPU's memory, identical on every
    rank) render as consecutive sub-batches, results concatenated."""
    if max_batch_bytes is None:
        from ._dev import require_cuda
        dev = require_cuda()
        max_batch_bytes = int(0.4 * torch.cuda.get_device_properties(dev).total_memory)
    groups, jobs = shard_batches(jobs, shard, int(max_batch_bytes), int(as_filter(f).branch_len))
    if shard is not None and int(shard[1]) > 1:
        if precision == "fp64":
            raise ValueError("the exact fp64 engine runs replicas only (its summation order "
                             "spans all images)")
        from . import parallel
        if dmax_hook is None:
            dmax_hook = parallel.allreduce_max
    sig = signals if signals is not None else [jb.s for jb in jobs]
    keys = [engine._key(jb.signal_key, jb.s) for jb in jobs]
    parts = []
    for g in groups:
        sub = [jobs[j] for j in g]
        launches0 = _lib.launch_count()
        geom = engine.Geometry(sub, inputs_ready=inputs_ready, dmax_hook=dmax_hook)
        res = engine.render(geom, [sig[j] for j in g], f, precision=precision,
                            signal_keys=[keys[j] for j in g], timing=timing)
        geom.release()  # everything reading the staged paths is enqueued
        res.launches = _lib.launch_count() - launches0  # libmvb kernels, geometry + render
        parts.append(res)
    return parts[0] if len(parts) == 1 else engine.RenderResult.concat(parts)
