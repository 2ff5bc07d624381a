"""Velocity-Verlet (kick-drift-kick) on the device (integrator.py:21-48).

One elementwise CUDA kernel per half step (K11), numpy-identical arithmetic.
"""

from __future__ import annotations

import torch

from . import _native as N
from .errors import SimulationDivergedError
from .particles import ParticleBuffer

PRE_FORCE = "pre-force"
POST_FORCE = "post-force"
POST_THEN_PRE = "post-then-pre"   # this step's second half + the next step's first, one pass


def velocity_verlet_step(buf: ParticleBuffer, params, phase: str, check: bool = True) -> None:
    """Advance one half of a velocity-Verlet step in place.

    ``check=False`` skips the host read of the non-finite flag (no sync);
    the flag accumulates in ``buf.extra['nonfinite']`` for a later check.
    """
    if phase == PRE_FORCE:
        code = 0
    elif phase == POST_FORCE:
        code = 1
    elif phase == POST_THEN_PRE:
        code = 2
    else:
        raise ValueError(f"unknown integration phase {phase!r}")
    flag = buf.extra.get("nonfinite")
    if flag is None or flag.device != buf.device:
        flag = torch.zeros(1, dtype=torch.int32, device=buf.device)
        buf.extra["nonfinite"] = flag
    if len(buf):
        N.call("lmd_verlet_step", len(buf), code, float(params.dt), float(params.mass),
               N.ptr(buf.pos_x), N.ptr(buf.pos_y), N.ptr(buf.pos_z), N.ptr(buf.vel_x),
               N.ptr(buf.vel_y), N.ptr(buf.vel_z), N.ptr(buf.force_x), N.ptr(buf.force_y),
               N.ptr(buf.force_z), N.ptr(buf.old_force_x), N.ptr(buf.old_force_y),
               N.ptr(buf.old_force_z), N.ptr(flag), N.stream())
    if check and int(flag.item()):
        flag.zero_()
        raise SimulationDivergedError("non-finite particle state")
