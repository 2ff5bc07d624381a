"""Particle data model on the device (mirrors the reference's particles.py).

``ParticleBuffer`` keeps the reference's structure-of-arrays field names
(particles.py:54-164) but every field is a ``torch.Tensor`` -- on a CUDA
device for the force path, or on the CPU for construction and inspection.
The layout the kernels consume (packed double4 positions in cell/cluster
order) is built from these SoA arrays by the containers; this class is the
API-level state a caller owns.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np
import torch

from .errors import ScenarioError

OWNED = 0
HALO = 1
DUMMY = 2


class Ownership(IntEnum):
    OWNED = OWNED
    HALO = HALO
    DUMMY = DUMMY


def default_device() -> torch.device:
    return torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")


def _vec3(v) -> np.ndarray:
    arr = np.asarray(v, dtype=np.float64)
    if arr.shape != (3,):
        raise ValueError(f"expected a 3-vector, got shape {arr.shape}")
    return arr.copy()


@dataclass
class Particle:
    """A single particle with its integration state (particles.py:35-51)."""

    id: int
    position: np.ndarray
    velocity: np.ndarray = field(default_factory=lambda: np.zeros(3))
    force: np.ndarray = field(default_factory=lambda: np.zeros(3))
    old_force: np.ndarray = field(default_factory=lambda: np.zeros(3))
    ownership: Ownership = Ownership.OWNED

    def __post_init__(self):
        self.position = _vec3(self.position)
        self.velocity = _vec3(self.velocity)
        self.force = _vec3(self.force)
        self.old_force = _vec3(self.old_force)
        self.ownership = Ownership(self.ownership)


FLOAT_FIELDS = (
    "pos_x", "pos_y", "pos_z",
    "vel_x", "vel_y", "vel_z",
    "force_x", "force_y", "force_z",
    "old_force_x", "old_force_y", "old_force_z",
)
ALL_FIELDS = FLOAT_FIELDS + ("id", "ownership")


class ParticleBuffer:
    """Structure-of-arrays particle storage on one device.

    Every field is a contiguous 1-D tensor of identical length: float64 for
    the twelve kinematic fields, int64 ``id`` and int8 ``ownership``.
    """

    _FLOAT_FIELDS = FLOAT_FIELDS

    def __init__(self, **fields):
        n = None
        for name in ALL_FIELDS:
            if name not in fields:
                raise TypeError(f"missing field {name!r}")
        for name in ALL_FIELDS:
            t = fields[name]
            if not isinstance(t, torch.Tensor):
                t = torch.as_tensor(np.asarray(t))
            want = torch.float64 if name in FLOAT_FIELDS else (
                torch.int64 if name == "id" else torch.int8)
            if t.dtype != want:
                t = t.to(want)
            if n is None:
                n = t.shape[0]
            elif t.shape[0] != n:
                raise ValueError(f"property array {name!r} has mismatched length")
            setattr(self, name, t)
        self.extra: dict = {}

    # ------------------------------------------------------------ creation
    @classmethod
    def empty(cls, n: int, device=None) -> "ParticleBuffer":
        device = torch.device(device) if device is not None else default_device()
        # one zeroed allocation, one row per float field (one fill launch)
        block = torch.zeros((len(FLOAT_FIELDS), n), dtype=torch.float64, device=device)
        kw = {name: block[k] for k, name in enumerate(FLOAT_FIELDS)}
        kw["id"] = torch.zeros(n, dtype=torch.int64, device=device)
        kw["ownership"] = torch.full((n,), OWNED, dtype=torch.int8, device=device)
        return cls(**kw)

    @classmethod
    def from_positions(cls, positions, ids=None, ownership=None, device=None) -> "ParticleBuffer":
        pos = torch.as_tensor(np.asarray(positions, dtype=np.float64)).reshape(-1, 3)
        buf = cls.empty(pos.shape[0], device=device)
        dev = buf.pos_x.device
        buf.pos_x.copy_(pos[:, 0].to(dev))
        buf.pos_y.copy_(pos[:, 1].to(dev))
        buf.pos_z.copy_(pos[:, 2].to(dev))
        if ids is None:
            buf.id.copy_(torch.arange(pos.shape[0], dtype=torch.int64, device=dev))
        else:
            buf.id.copy_(torch.as_tensor(np.asarray(ids, dtype=np.int64)).to(dev))
        if ownership is not None:
            buf.ownership.copy_(torch.as_tensor(np.asarray(ownership, dtype=np.int8)).to(dev))
        return buf

    @classmethod
    def from_host(cls, host, device=None, fields=ALL_FIELDS) -> "ParticleBuffer":
        """Copy a SoA buffer with the reference's field names (numpy or torch)
        to the device.  Only ``fields`` are transferred (missing or None
        fields start as zeros / OWNED); pinned torch tensors copy async."""
        device = torch.device(device) if device is not None else default_device()
        n = len(getattr(host, "pos_x"))
        out = cls.empty(n, device=device)
        for name in fields:
            arr = getattr(host, name, None)
            if arr is None:
                continue
            t = arr if isinstance(arr, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(arr))
            getattr(out, name).copy_(t, non_blocking=t.device.type == "cpu" and t.is_pinned())
        if "id" not in fields or getattr(host, "id", None) is None:
            out.id.copy_(torch.arange(n, dtype=torch.int64, device=device))
        return out

    # ------------------------------------------------------------- queries
    def __len__(self) -> int:
        return int(self.pos_x.shape[0])

    @property
    def device(self) -> torch.device:
        return self.pos_x.device

    @property
    def real_count(self) -> int:
        return self.ownership_counts()[1]

    @property
    def has_dummies(self) -> bool:
        return self.ownership_counts()[1] < len(self)

    def ownership_counts(self) -> tuple[int, int]:
        """(owned, non-dummy) entry counts (particles.py:111-123), cached."""
        cached = self.__dict__.get("_counts")
        if cached is None:
            own = self.ownership
            cached = (int((own == OWNED).sum()), int((own != DUMMY).sum()))
            self.__dict__["_counts"] = cached
        return cached

    def self_pair_slots(self, newton3: bool) -> int:
        """Real pair slots of this buffer against itself (particles.py:125-143)."""
        key = "_self_slots_n3" if newton3 else "_self_slots"
        cached = self.__dict__.get(key)
        if cached is None:
            own = self.ownership
            owned = own == OWNED
            nondummy = (own != DUMMY).to(torch.int64)
            total = int(nondummy.sum())
            if newton3:
                after = total - torch.cumsum(nondummy, 0)
                cached = int(after[owned].sum())
            else:
                cached = int(owned.sum()) * max(total - 1, 0)
            self.__dict__[key] = cached
        return cached

    def invalidate_counts(self) -> None:
        for k in ("_counts", "_self_slots_n3", "_self_slots"):
            self.__dict__.pop(k, None)

    def positions(self) -> torch.Tensor:
        """(N, 3) copy of the positions."""
        return torch.stack([self.pos_x, self.pos_y, self.pos_z], dim=1)

    def forces(self) -> torch.Tensor:
        return torch.stack([self.force_x, self.force_y, self.force_z], dim=1)

    def velocities(self) -> torch.Tensor:
        return torch.stack([self.vel_x, self.vel_y, self.vel_z], dim=1)

    # ------------------------------------------------------------- slicing
    def view(self, start: int, stop: int) -> "ParticleBuffer":
        """Zero-copy slice sharing memory with this buffer."""
        return ParticleBuffer(**{name: getattr(self, name)[start:stop] for name in ALL_FIELDS})

    def take(self, indices) -> "ParticleBuffer":
        idx = torch.as_tensor(indices, device=self.device, dtype=torch.int64)
        return ParticleBuffer(**{name: getattr(self, name)[idx] for name in ALL_FIELDS})

    def copy(self) -> "ParticleBuffer":
        return ParticleBuffer(**{name: getattr(self, name).clone() for name in ALL_FIELDS})

    def to(self, device) -> "ParticleBuffer":
        return ParticleBuffer(**{name: getattr(self, name).to(device) for name in ALL_FIELDS})

    def numpy(self) -> dict:
        return {name: getattr(self, name).cpu().numpy() for name in ALL_FIELDS}


def concat_buffers(first: ParticleBuffer, second: ParticleBuffer) -> ParticleBuffer:
    return ParticleBuffer(**{name: torch.cat([getattr(first, name), getattr(second, name)])
                             for name in ALL_FIELDS})


def soa_from_particles(particles: list[Particle], device=None) -> ParticleBuffer:
    """Pack a particle list into an SoA buffer, preserving order (particles.py:175-186)."""
    n = len(particles)
    arrs = {name: np.zeros(n) for name in FLOAT_FIELDS}
    ids = np.zeros(n, dtype=np.int64)
    own = np.zeros(n, dtype=np.int8)
    for k, p in enumerate(particles):
        arrs["pos_x"][k], arrs["pos_y"][k], arrs["pos_z"][k] = p.position
        arrs["vel_x"][k], arrs["vel_y"][k], arrs["vel_z"][k] = p.velocity
        arrs["force_x"][k], arrs["force_y"][k], arrs["force_z"][k] = p.force
        arrs["old_force_x"][k], arrs["old_force_y"][k], arrs["old_force_z"][k] = p.old_force
        ids[k] = p.id
        own[k] = int(p.ownership)
    device = torch.device(device) if device is not None else default_device()
    kw = {k: torch.from_numpy(v).to(device) for k, v in arrs.items()}
    kw["id"] = torch.from_numpy(ids).to(device)
    kw["ownership"] = torch.from_numpy(own).to(device)
    return ParticleBuffer(**kw)


def particles_from_soa(buf: ParticleBuffer) -> list[Particle]:
    h = buf.numpy()
    out = []
    for k in range(len(buf)):
        out.append(Particle(
            id=int(h["id"][k]),
            position=np.array([h["pos_x"][k], h["pos_y"][k], h["pos_z"][k]]),
            velocity=np.array([h["vel_x"][k], h["vel_y"][k], h["vel_z"][k]]),
            force=np.array([h["force_x"][k], h["force_y"][k], h["force_z"][k]]),
            old_force=np.array([h["old_force_x"][k], h["old_force_y"][k], h["old_force_z"][k]]),
            ownership=Ownership(int(h["ownership"][k])),
        ))
    return out


def generate_cube_lattice(origin, counts, spacing: float, velocity=(0.0, 0.0, 0.0),
                          id_start: int = 0) -> list[Particle]:
    """Regular x-fastest lattice (particles.py:205-231)."""
    counts = tuple(int(c) for c in counts)
    if any(c < 1 for c in counts):
        raise ScenarioError(f"lattice counts must all be >= 1, got {counts}")
    if spacing <= 0:
        raise ScenarioError(f"lattice spacing must be positive, got {spacing}")
    origin = _vec3(origin)
    v0 = _vec3(velocity)
    out = []
    pid = id_start
    for kz in range(counts[2]):
        for ky in range(counts[1]):
            for kx in range(counts[0]):
                pos = origin + spacing * np.array([kx, ky, kz], dtype=np.float64)
                out.append(Particle(id=pid, position=pos, velocity=v0))
                pid += 1
    return out


def lattice_positions(origin, counts, spacing: float) -> np.ndarray:
    """Vectorised generate_cube_lattice positions, identical values and order."""
    origin = _vec3(origin)
    nx, ny, nz = (int(c) for c in counts)
    kz, ky, kx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    k = np.stack([kx.ravel(), ky.ravel(), kz.ravel()], axis=1).astype(np.float64)
    return origin + spacing * k
