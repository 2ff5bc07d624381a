"""Packed schedule execution on the device (executor.py:24-171 of the reference).

``pack_schedule`` flattens a ``Schedule`` into offset arrays over the two
backing buffers (owned-side, halo-side) exactly as the reference does, and
additionally keeps each unit's color and base so the device can run
same-color bases concurrently (traversals.py:1-6).  ``execute_packed`` runs
every unit with ``lmd_execute_packed`` -- one launch per color, one warp per
base, units of a base in order -- and returns the reference's statistics:
invocations = sum ceil(ni/a) * ceil(nj/b), lane slots = invocations * V,
useful = the pack-time count, pairs from the kernel.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .errors import ConfigurationError, ParticleOverlapError
from .kernels import KernelStats, as_pattern, validate_vector_width


@dataclass
class PackedSchedule:
    i_offset: np.ndarray
    i_length: np.ndarray
    j_offset: np.ndarray
    j_length: np.ndarray
    j_in_halo: np.ndarray
    newton3: np.ndarray
    same_buffer: np.ndarray
    useful_total: int
    color: np.ndarray = field(default=None)
    base: np.ndarray = field(default=None)


def pack_schedule(sched) -> PackedSchedule:
    """Flatten work units into offset arrays; count useful lanes once (executor.py:38-69)."""
    n = len(sched.units)
    i_off = np.empty(n, dtype=np.int64)
    i_len = np.empty(n, dtype=np.int64)
    j_off = np.empty(n, dtype=np.int64)
    j_len = np.empty(n, dtype=np.int64)
    j_halo = np.empty(n, dtype=np.bool_)
    n3 = np.empty(n, dtype=np.bool_)
    same = np.empty(n, dtype=np.bool_)
    color = np.empty(n, dtype=np.int64)
    base = np.empty(n, dtype=np.int64)
    useful = 0
    for k, u in enumerate(sched.units):
        iw, io, il = u.i_buffer.backing_slot
        jw, jo, jl = u.j_buffer.backing_slot
        if iw != 0:
            raise ConfigurationError("i-buffer must come from the owned backing")
        i_off[k], i_len[k], j_off[k], j_len[k] = io, il, jo, jl
        j_halo[k] = bool(jw)
        n3[k] = u.newton3
        same[k] = u.same_buffer
        color[k] = u.color
        base[k] = u.base_index
        if u.same_buffer:
            useful += u.i_buffer.self_pair_slots(u.newton3)
        else:
            useful += u.i_buffer.ownership_counts()[0] * u.j_buffer.ownership_counts()[1]
    return PackedSchedule(i_off, i_len, j_off, j_len, j_halo, n3, same, useful, color, base)


def _pos4(buf, dev) -> torch.Tensor:
    own = buf.ownership.to(torch.float64)
    return torch.stack([buf.pos_x, buf.pos_y, buf.pos_z, own], dim=1).to(dev).contiguous()


def execute_packed(packed: PackedSchedule, owned_backing, halo_backing, params, pattern,
                   vector_width: int) -> KernelStats:
    """Run every packed unit on the GPU; forces accumulate (+=) into the backings."""
    validate_vector_width(vector_width)
    pattern = as_pattern(pattern)
    a, b = pattern.shape(vector_width)
    n = len(packed.i_offset)
    inv = int((-(-packed.i_length // a) * -(-packed.j_length // b)).sum()) if n else 0
    dev = owned_backing.device
    if n == 0:
        return KernelStats(0, 0, packed.useful_total, 0)
    # group units by (color, base); an unannotated pack runs as one base
    color = packed.color if packed.color is not None else np.zeros(n, dtype=np.int64)
    base = packed.base if packed.base is not None else np.zeros(n, dtype=np.int64)
    order = np.lexsort((np.arange(n), base, color))        # color, base, then unit order
    cb = np.stack([color[order], base[order]], axis=1)
    new_base = np.ones(n, dtype=bool)
    new_base[1:] = np.any(cb[1:] != cb[:-1], axis=1)
    base_start = np.append(np.nonzero(new_base)[0], n).astype(np.int64)
    base_color = color[order][new_base]
    colors = np.unique(base_color)
    color_base_start = np.searchsorted(base_color, np.append(colors, colors[-1] + 1)).astype(
        np.int64)
    t = lambda x, dt: torch.as_tensor(np.ascontiguousarray(x), dtype=dt, device=dev)  # noqa
    arrays = [t(packed.i_offset, torch.int64), t(packed.i_length, torch.int64),
              t(packed.j_offset, torch.int64), t(packed.j_length, torch.int64),
              t(packed.j_in_halo, torch.uint8), t(packed.newton3, torch.uint8),
              t(packed.same_buffer, torch.uint8)]
    bu = t(order, torch.int64)
    bs = t(base_start, torch.int64)
    own4 = _pos4(owned_backing, dev)
    halo4 = _pos4(halo_backing, dev) if len(halo_backing) else torch.zeros((1, 4),
                                                                            dtype=torch.float64,
                                                                            device=dev)
    hfx = halo_backing.force_x if len(halo_backing) else torch.zeros(1, dtype=torch.float64,
                                                                    device=dev)
    hfy = halo_backing.force_y if len(halo_backing) else hfx
    hfz = halo_backing.force_z if len(halo_backing) else hfx
    for f in (owned_backing.force_x, owned_backing.force_y, owned_backing.force_z):
        if not f.is_contiguous():
            raise ConfigurationError("backing forces must be contiguous device arrays")
    stats_t = N.new_stats(dev)
    cbs = (N.C.c_int64 * len(color_base_start))(*color_base_start.tolist())
    N.call("lmd_execute_packed", n, *[N.ptr(x) for x in arrays], len(colors), cbs, N.ptr(bu),
           N.ptr(bs), pattern.code, N.make_lj(params), N.ptr(own4), N.ptr(halo4),
           N.ptr(owned_backing.force_x), N.ptr(owned_backing.force_y),
           N.ptr(owned_backing.force_z), N.ptr(hfx), N.ptr(hfy), N.ptr(hfz), N.ptr(stats_t),
           N.stream())
    st = N.read_stats(stats_t)
    if st.overlap:
        raise ParticleOverlapError("zero distance between interacting particles")
    return KernelStats(inv, inv * vector_width, packed.useful_total, int(st.pair_interactions))
