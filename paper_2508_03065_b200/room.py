"""Shoebox rooms and the image-source lattice.

Same values and API as reference room.py (Room :27-56, MicPosition :59-79,
ImageSourceSpec :82-95, enumerate_images :108-143, as_arrays :175-187,
image_distance :159-165).  The enumeration itself runs on the GPU
(libmvb mvb_enumerate: one thread per image, canonical order) and returns
the reference's spec list; `image_table` returns the same lattice as device
arrays for the fused renderer without a host round trip.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._dev import ptr, require_cuda, stream_handle, to_dev


def _vec3(v, name):
    a = np.asarray(v, dtype=np.float64)
    if a.shape != (3,):
        raise ValueError(f"{name} must be a 3-vector, got shape {a.shape}")
    if not np.all(np.isfinite(a)):
        raise ValueError(f"{name} must be finite")
    return a


@dataclass(frozen=True)
class Room:
    """dims (Lx, Ly, Lz) > 0; wall_reflection 6 values in (0, 1] ordered
    (-x, +x, -y, +y, -z, +z) or one scalar."""

    dims: np.ndarray
    wall_reflection: np.ndarray

    def __post_init__(self):
        dims = _vec3(self.dims, "dims")
        walls = np.asarray(self.wall_reflection, dtype=np.float64)
        if walls.shape == ():
            walls = np.full(6, float(walls))
        if walls.shape != (6,):
            raise ValueError("wall_reflection needs 6 values (or one scalar)")
        if not np.all(dims > 0):
            raise ValueError("room dims must be strictly positive")
        if not (np.all(walls > 0) and np.all(walls <= 1)):
            raise ValueError("wall reflections must lie in (0, 1]")
        dims = dims.copy()
        walls = walls.copy()
        dims.flags.writeable = False
        walls.flags.writeable = False
        object.__setattr__(self, "dims", dims)
        object.__setattr__(self, "wall_reflection", walls)

    def contains(self, pos, margin=0.0):
        p = np.asarray(pos, dtype=np.float64)
        return bool(np.all(p > margin) and np.all(p < self.dims - margin))


@dataclass(frozen=True)
class MicPosition:
    """Fixed receiver, strictly inside the room when used."""

    pos: np.ndarray

    def __post_init__(self):
        p = _vec3(self.pos, "mic pos").copy()
        p.flags.writeable = False
        object.__setattr__(self, "pos", p)

    def require_inside(self, room):
        if not room.contains(self.pos):
            raise ValueError("mic position must be strictly inside the room")


def as_mic(value):
    if isinstance(value, MicPosition):
        return value
    return MicPosition(pos=np.asarray(value, dtype=np.float64))


@dataclass(frozen=True, order=True)
class ImageSourceSpec:
    """order, lattice (per-axis n), parity (per-axis flip), beta; field
    order gives the canonical sort (order, lattice, parity)."""

    order: int
    lattice: tuple
    parity: tuple
    beta: float


@dataclass
class ImageTable:
    """Canonical-order lattice of n_rooms rooms as device tensors."""

    offset: torch.Tensor  # (R, S, 3) f64
    sign: torch.Tensor  # (R, S, 3) f64
    beta: torch.Tensor  # (R, S) f64
    order: torch.Tensor  # (R, S) int32
    lattice: torch.Tensor  # (R, S, 3) int32
    parity: torch.Tensor  # (R, S, 3) int32

    @property
    def count(self) -> int:
        return int(self.order.shape[1])


def image_count(max_order: int) -> int:
    """Images with reflection order <= max_order (4 o^2 + 2 per order o)."""
    if max_order < 0:
        raise ValueError("max_order must be >= 0")
    return _lib.image_count(max_order)


def image_table(dims, walls, max_order: int, device=None) -> ImageTable:
    """GPU enumeration for one room (dims (3,), walls (6,)) or a batch
    (dims (R,3), walls (R,6)) of rooms sharing max_order."""
    if max_order < 0:
        raise ValueError("max_order must be >= 0")
    dev = require_cuda(device)
    d = to_dev(np.atleast_2d(np.asarray(dims, dtype=np.float64)), torch.float64, dev)
    w = np.asarray(walls, dtype=np.float64)
    if w.ndim == 0:
        w = np.full(6, float(w))
    w = to_dev(np.atleast_2d(w), torch.float64, dev)
    R = d.shape[0]
    if w.shape != (R, 6) or d.shape != (R, 3):
        raise ValueError("dims (R,3) and walls (R,6) expected")
    S = image_count(max_order)
    f64 = dict(dtype=torch.float64, device=dev)
    i32 = dict(dtype=torch.int32, device=dev)
    t = ImageTable(torch.empty(R, S, 3, **f64), torch.empty(R, S, 3, **f64), torch.empty(R, S, **f64),
                   torch.empty(R, S, **i32), torch.empty(R, S, 3, **i32), torch.empty(R, S, 3, **i32))
    _lib.call("mvb_enumerate", ptr(d), ptr(w), R, int(max_order), ptr(t.lattice), ptr(t.parity),
              ptr(t.order), ptr(t.beta), ptr(t.offset), ptr(t.sign), stream_handle(dev))
    return t


def enumerate_images(room: Room, max_order: int):
    """All images of total reflection order <= max_order in canonical order
    (reference room.py:108-143), enumerated on the GPU."""
    if max_order < 0:
        raise ValueError("max_order must be >= 0")
    t = image_table(room.dims, room.wall_reflection, max_order)
    order = t.order[0].cpu().numpy()
    lat = t.lattice[0].cpu().numpy()
    par = t.parity[0].cpu().numpy()
    beta = t.beta[0].cpu().numpy()
    return [ImageSourceSpec(order=int(order[i]), lattice=tuple(int(v) for v in lat[i]),
                            parity=tuple(bool(v) for v in par[i]), beta=float(beta[i]))
            for i in range(order.shape[0])]


def attenuation(beta, distance):
    """Spherical-spreading gain beta / (4 pi d) (reference room.py:168-172)."""
    if distance <= 0:
        raise ValueError("attenuation requires distance > 0 (clamp first)")
    return beta / (4.0 * np.pi * distance)


def as_arrays(specs, room):
    """(offset (S,3), sign (S,3), beta (S,), order (S,)) as numpy, in list
    order (reference room.py:175-187)."""
    lat = np.array([s.lattice for s in specs], dtype=np.float64).reshape(-1, 3)
    par = np.array([s.parity for s in specs], dtype=bool).reshape(-1, 3)
    offset = 2.0 * lat * room.dims
    sign = np.where(par, -1.0, 1.0)
    beta = np.array([s.beta for s in specs], dtype=np.float64)
    order = np.array([s.order for s in specs], dtype=np.int64)
    return offset, sign, beta, order


def image_position(spec, source_pos, room):
    src = np.asarray(source_pos, dtype=np.float64)
    lat = np.asarray(spec.lattice, dtype=np.float64)
    flip = np.where(np.asarray(spec.parity), -1.0, 1.0)
    return 2.0 * lat * room.dims + flip * src


def image_distance(spec, source_pos, mic, room):
    return float(np.linalg.norm(image_position(spec, source_pos, room) - as_mic(mic).pos))


def estimate_image_count(room, t60, c=343.0) -> int:
    """Lattice points m (room-centred source and mic) with path length
    |(m_x Lx, m_y Ly, m_z Lz)| <= c * t60: the cost-budget estimate of
    reference room.py:190-209 (not an enumeration)."""
    if t60 <= 0:
        raise ValueError("t60 must be > 0")
    r = c * t60
    lx, ly, lz = (float(v) for v in room.dims)
    mx = np.arange(-int(r // lx), int(r // lx) + 1, dtype=np.float64)
    my = np.arange(-int(r // ly), int(r // ly) + 1, dtype=np.float64)
    rest = r * r - (mx[:, None] * lx) ** 2 - (my[None, :] * ly) ** 2
    inside = rest >= 0.0
    half = np.floor(np.sqrt(np.where(inside, rest, 0.0)) / lz)
    return int(np.sum(np.where(inside, 2.0 * half + 1.0, 0.0)))
