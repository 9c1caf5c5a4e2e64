"""Seeded synthetic scenes for the five BASELINE.json configurations.

Host-side input preparation only (numpy).  The reference has no datasets
for this path (SURVEY.md 8c "Datasets"); every config is white Gaussian dry
signal plus an analytic or seeded source path.  c1/c2 paths restate the
reference's own `generate` kinds (trajectory.py:354-389: line with pinned
start/direction, circle about the room centre); c3-c5 use the generators
SURVEY.md 8d prescribes (random-waypoint piecewise-linear, billiard line,
translating 8-mic circle), which the reference lacks.

    scenes = make_scenes("c3")            # full size
    scenes = make_scenes("c3", duration=0.1, max_order=8)   # reduced
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    rate: float
    duration: float
    max_order: int
    fd_taps: int
    tiers: tuple  # ((max_order, N), ...) ascending
    dtype: str  # "f64" | "f32" : dry-signal / output precision
    n_scenes: int = 1
    n_channels: int = 1
    seed: int = 0
    note: str = ""


WORKLOADS = {
    "c1": Workload("c1", 16000.0, 2.0, 3, 32, ((1, 1), (3, 32)), "f64", seed=1,
                   note="6x4x3 m beta .85, line (1,1,1.5)->(5,3,1.5), mic (3,2,1.2)"),
    "c2": Workload("c2", 16000.0, 4.0, 10, 32, ((2, 1), (5, 16), (10, 128)), "f32", seed=2,
                   note="6x4x3 m beta .85, r=1 circle about (3,2,1.5) at 0.5 rev/s, mic (1.5,1,1.2)"),
    "c3": Workload("c3", 48000.0, 10.0, 20, 64, ((2, 1), (8, 32), (20, 256)), "f32", seed=3,
                   note="20x15x8 m beta .9, random-waypoint 1-5 m/s, mic at centre"),
    "c4": Workload("c4", 16000.0, 4.0, 12, 32, ((2, 1), (12, 64)), "f32", n_scenes=256, seed=4,
                   note="256 random rooms, billiard line 0.5-3 m/s, random fixed mic"),
    "c5": Workload("c5", 48000.0, 8.0, 15, 64, ((2, 1), (7, 32), (15, 256)), "f32",
                   n_channels=8, seed=5,
                   note="10x8x4 m, waypoint 2 m/s, 8-mic r=5 cm circle translating 1 m/s"),
}


@dataclass
class Scene:
    """One render job: dry signal, source path, receiver(s), room."""

    s: np.ndarray  # (T,) float64 or float32
    pos: np.ndarray  # (T,3) float64 source path at the audio rate
    mics: list  # per channel: (3,) fixed or (T,3) moving receiver path
    dims: np.ndarray  # (3,)
    walls: np.ndarray  # (6,) ordered (-x,+x,-y,+y,-z,+z)
    rate: float
    max_order: int
    tiers: tuple
    fd_taps: int
    meta: dict = field(default_factory=dict)

    @property
    def T(self) -> int:
        return int(self.pos.shape[0])


def _n_samples(duration: float, rate: float) -> int:
    return max(2, int(round(duration * rate)))


def line_path(start, direction, speed, duration, rate):
    """Constant-velocity line (trajectory.py:354-365 arithmetic)."""
    n = _n_samples(duration, rate)
    t = np.arange(n) / rate
    d = np.asarray(direction, dtype=np.float64)
    d = d / np.linalg.norm(d)
    start = np.asarray(start, dtype=np.float64)
    return start[None, :] + d[None, :] * (speed * t)[:, None]


def circle_path(dims, freq, speed, duration, rate):
    """Horizontal circle about the room centre (trajectory.py:378-389)."""
    n = _n_samples(duration, rate)
    t = np.arange(n) / rate
    centre = np.asarray(dims, dtype=np.float64) / 2.0
    radius = speed / (2 * np.pi * freq)
    ph = 2 * np.pi * freq * t
    disp = np.stack([radius * np.cos(ph), radius * np.sin(ph), np.zeros(n)], axis=1)
    return centre + disp


def waypoint_path(rng, dims, margin, speed_lo, speed_hi, duration, rate):
    """Piecewise-linear path through uniform waypoints inside a wall margin,
    constant speed per segment drawn from U[speed_lo, speed_hi]."""
    dims = np.asarray(dims, dtype=np.float64)
    n = _n_samples(duration, rate)
    t = np.arange(n) / rate
    pts = [rng.uniform(margin, dims - margin)]
    ends = [0.0]
    while ends[-1] <= t[-1]:
        q = rng.uniform(margin, dims - margin)
        v = rng.uniform(speed_lo, speed_hi)
        seg = np.linalg.norm(q - pts[-1])
        pts.append(q)
        ends.append(ends[-1] + max(seg, 1e-9) / v)
    pts = np.array(pts)
    ends = np.array(ends)
    k = np.clip(np.searchsorted(ends, t, side="right") - 1, 0, len(ends) - 2)
    frac = (t - ends[k]) / (ends[k + 1] - ends[k])
    return pts[k] + (pts[k + 1] - pts[k]) * frac[:, None]


def billiard_path(start, direction, speed, lo, hi, duration, rate):
    """Straight motion with specular reflection inside the box [lo, hi]
    (a 4 s line at <= 3 m/s cannot stay straight in a 3 m room)."""
    n = _n_samples(duration, rate)
    t = np.arange(n) / rate
    d = np.asarray(direction, dtype=np.float64)
    d = d / np.linalg.norm(d)
    free = np.asarray(start, np.float64)[None, :] + d[None, :] * (speed * t)[:, None]
    lo = np.asarray(lo, np.float64)
    w = np.asarray(hi, np.float64) - lo
    u = np.mod(free - lo, 2 * w)
    return lo + np.where(u <= w, u, 2 * w - u)


def _dry(rng, n, dtype):
    x = rng.standard_normal(n)
    return x if dtype == "f64" else x.astype(np.float32)


def make_scenes(name: str, duration: float | None = None, max_order: int | None = None,
                n_scenes: int | None = None, n_channels: int | None = None,
                tiers: tuple | None = None, seed: int | None = None) -> list:
    """Build the seeded scenes of a config; optional overrides give the
    reduced-size parity cases (same generators, same seeds unless `seed`)."""
    w = WORKLOADS[name]
    if seed is not None:
        w = replace(w, seed=int(seed))
    if duration is not None:
        w = replace(w, duration=duration)
    if max_order is not None:
        w = replace(w, max_order=max_order)
    if tiers is not None:
        w = replace(w, tiers=tuple(tiers))
    elif max_order is not None:
        # clip the tier table to the reduced order
        tl = [(min(mo, max_order), N) for mo, N in w.tiers]
        out = []
        for mo, N in tl:
            if not out or mo > out[-1][0]:
                out.append((mo, N))
        w = replace(w, tiers=tuple(out))
    rate = w.rate
    T = _n_samples(w.duration, rate)
    rng = np.random.default_rng(w.seed)
    scenes = []
    if name == "c1":
        dims = np.array([6.0, 4.0, 3.0])
        pos = line_path((1.0, 1.0, 1.5), (2.0, 1.0, 0.0), np.sqrt(5.0), w.duration, rate)
        scenes.append(Scene(_dry(rng, T, w.dtype), pos, [np.array([3.0, 2.0, 1.2])], dims,
                            np.full(6, 0.85), rate, w.max_order, w.tiers, w.fd_taps))
    elif name == "c2":
        dims = np.array([6.0, 4.0, 3.0])
        pos = circle_path(dims, 0.5, np.pi, w.duration, rate)
        scenes.append(Scene(_dry(rng, T, w.dtype), pos, [np.array([1.5, 1.0, 1.2])], dims,
                            np.full(6, 0.85), rate, w.max_order, w.tiers, w.fd_taps))
    elif name == "c3":
        dims = np.array([20.0, 15.0, 8.0])
        pos = waypoint_path(rng, dims, 1.0, 1.0, 5.0, w.duration, rate)
        s = _dry(rng, T, w.dtype)
        scenes.append(Scene(s, pos, [dims / 2.0], dims, np.full(6, 0.9), rate, w.max_order,
                            w.tiers, w.fd_taps))
    elif name == "c4":
        count = w.n_scenes if n_scenes is None else n_scenes
        for k in range(count):
            r = np.random.default_rng(w.seed * 1000 + k)
            dims = np.array([r.uniform(3, 10), r.uniform(3, 8), r.uniform(2.5, 4)])
            walls = r.uniform(0.6, 0.95, size=6)
            lo, hi = np.full(3, 0.5), dims - 0.5
            start = r.uniform(lo, hi)
            direction = r.normal(size=3)
            speed = r.uniform(0.5, 3.0)
            pos = billiard_path(start, direction, speed, lo, hi, w.duration, rate)
            mic = r.uniform(lo, hi)
            scenes.append(Scene(_dry(r, T, w.dtype), pos, [mic], dims, walls, rate,
                                w.max_order, w.tiers, w.fd_taps, meta={"scene": k}))
    elif name == "c5":
        dims = np.array([10.0, 8.0, 4.0])
        walls = np.array([0.7, 0.75, 0.8, 0.85, 0.6, 0.9])
        pos = waypoint_path(rng, dims, 1.0, 2.0, 2.0, w.duration, rate)
        s = _dry(rng, T, w.dtype)
        count = w.n_channels if n_channels is None else n_channels
        t = np.arange(T) / rate
        centre = np.stack([1.5 + 1.0 * t, np.full(T, 4.0), np.full(T, 1.5)], axis=1)
        mics = []
        for k in range(count):
            a = 2 * np.pi * k / 8
            mics.append(centre + 0.05 * np.array([np.cos(a), np.sin(a), 0.0])[None, :])
        scenes.append(Scene(s, pos, mics, dims, walls, rate, w.max_order, w.tiers, w.fd_taps))
    else:
        raise KeyError(name)
    for sc in scenes:
        sc.meta.setdefault("workload", name)
        sc.meta["dtype"] = w.dtype
    return scenes


def updates(scene: Scene, n_images: int, out_len: int) -> int:
    """Image x output-sample updates of one scene (SURVEY.md 8d unit)."""
    return int(n_images) * int(out_len) * len(scene.mics)
