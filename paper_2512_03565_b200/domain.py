"""Simulation box, LJ parameters, boundaries and periodic images on the device.

Mirrors the reference's domain.py (20-144).  ``build_halo`` and
``apply_boundaries`` run as CUDA kernels (K9 / K11) through the C ABI.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _native as N
from .errors import ScenarioError, SimulationDivergedError
from .particles import HALO, OWNED, ParticleBuffer


class BoundaryKind(Enum):
    REFLECTIVE = "reflective"
    PERIODIC = "periodic"


@dataclass(frozen=True)
class SimulationBox:
    """Axis-aligned box with a per-axis boundary condition (domain.py:20-42)."""

    min: np.ndarray
    max: np.ndarray
    boundary: tuple

    def __post_init__(self):
        object.__setattr__(self, "min", np.asarray(self.min, dtype=np.float64))
        object.__setattr__(self, "max", np.asarray(self.max, dtype=np.float64))
        b = tuple(BoundaryKind(getattr(x, "value", x)) for x in self.boundary)
        object.__setattr__(self, "boundary", b)
        if not np.all(self.max > self.min):
            raise ScenarioError(f"box max {self.max} must exceed min {self.min} on every axis")

    @property
    def lengths(self) -> np.ndarray:
        return self.max - self.min

    @property
    def periodic_axes(self) -> list[int]:
        return [k for k, b in enumerate(self.boundary) if b is BoundaryKind.PERIODIC]

    @classmethod
    def cube(cls, length: float, periodic: bool = True, origin: float = 0.0) -> "SimulationBox":
        kind = BoundaryKind.PERIODIC if periodic else BoundaryKind.REFLECTIVE
        return cls(np.full(3, origin), np.full(3, origin + length), (kind,) * 3)


@dataclass(frozen=True)
class LJParams:
    """Lennard-Jones interaction and integration parameters (domain.py:45-66)."""

    epsilon: float = 1.0
    sigma: float = 1.0
    cutoff: float = 2.5
    skin: float = 0.5
    mass: float = 1.0
    dt: float = 0.001

    def __post_init__(self):
        for name in ("epsilon", "sigma", "cutoff", "mass", "dt"):
            if getattr(self, name) <= 0:
                raise ScenarioError(f"{name} must be strictly positive")
        if self.skin < 0:
            raise ScenarioError("skin must be non-negative")

    @property
    def interaction_length(self) -> float:
        """Cutoff plus skin: the neighbor-structure design length."""
        return self.cutoff + self.skin


def as_box(box) -> SimulationBox:
    """Accept the reference's SimulationBox (duck-typed) as well as ours."""
    if isinstance(box, SimulationBox):
        return box
    return SimulationBox(box.min, box.max, tuple(b.value for b in box.boundary))


def apply_boundaries(buf: ParticleBuffer, box) -> None:
    """Wrap / mirror escaped particles in place (domain.py:69-94), on the device."""
    box = as_box(box)
    if len(buf) == 0:
        return
    flag = torch.zeros(1, dtype=torch.int32, device=buf.device)
    N.call("lmd_apply_boundaries", N.make_box(box), len(buf), N.ptr(buf.pos_x), N.ptr(buf.pos_y),
           N.ptr(buf.pos_z), N.ptr(buf.vel_x), N.ptr(buf.vel_y), N.ptr(buf.vel_z), N.ptr(flag),
           N.stream())
    if int(flag.item()):
        raise SimulationDivergedError("particle more than one box length outside the box")


def build_halo(buf: ParticleBuffer, box, margin: float) -> ParticleBuffer:
    """Periodic images of owned particles within ``margin`` of a face (domain.py:97-144).

    Images carry HALO ownership and their owner's id; ``extra['owner']`` holds
    the owner's index in ``buf`` and ``extra['shift']`` the shift code so the
    images can be refreshed from moved owners without re-deriving them.
    Image order is (owner, shift combination) rather than the reference's
    (shift combination, owner); containers re-sort images by cell anyway.
    """
    box = as_box(box)
    dev = buf.device
    n = len(buf)
    if not box.periodic_axes or n == 0:
        out = ParticleBuffer.empty(0, device=dev)
        out.extra["owner"] = torch.zeros(0, dtype=torch.int32, device=dev)
        out.extra["shift"] = torch.zeros(0, dtype=torch.int8, device=dev)
        return out
    cb = N.make_box(box)
    s = N.stream()
    count = torch.empty(n, dtype=torch.int32, device=dev)
    N.call("lmd_halo_count", cb, float(margin), n, N.ptr(buf.pos_x), N.ptr(buf.pos_y),
           N.ptr(buf.pos_z), N.ptr(buf.ownership), N.ptr(count), s)
    offset = torch.empty(n, dtype=torch.int32, device=dev)
    tb = N.load().lmd_scan_temp_bytes(n)
    temp = torch.empty(max(tb, 1), dtype=torch.uint8, device=dev)
    N.call("lmd_exclusive_scan_i32", n, N.ptr(count), N.ptr(offset), N.ptr(temp), tb, s)
    total = int((offset[-1] + count[-1]).item())
    out = ParticleBuffer.empty(total, device=dev)
    owner = torch.empty(total, dtype=torch.int32, device=dev)
    shift = torch.empty(total, dtype=torch.int8, device=dev)
    if total:
        N.call("lmd_halo_emit", cb, float(margin), n, N.ptr(buf.pos_x), N.ptr(buf.pos_y),
               N.ptr(buf.pos_z), N.ptr(buf.ownership), N.ptr(offset), N.ptr(out.pos_x),
               N.ptr(out.pos_y), N.ptr(out.pos_z), N.ptr(owner), N.ptr(shift), s)
        out.id.copy_(buf.id[owner.long()])
    out.ownership.fill_(HALO)
    out.extra["owner"] = owner
    out.extra["shift"] = shift
    return out


__all__ = ["BoundaryKind", "SimulationBox", "LJParams", "apply_boundaries", "build_halo",
           "as_box", "OWNED"]
