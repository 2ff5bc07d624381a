"""Lennard-Jones pair functor on the B200: patterns, statistics, kernels.

Mirrors the reference's kernels.py (40-424).  The four register-fill
patterns (interaction orders) are realised as warp lane mappings at the GPU's
natural width of 32 lanes: lane l of a fill holds the pair
(i_off(l), j_off(l)) of ``_lane_templates`` (kernels.py:250-265) with
(a, b) = (1, 32), (32, 1), (2, 16), (16, 2).  The caller's ``vector_width``
keeps its reference meaning for the lane statistics, which are geometric
(kernels.py:416-423, executor.py:165-171) and reproduced exactly.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import _native as N
from .errors import ConfigurationError, ParticleOverlapError
from .particles import ParticleBuffer


class PatternKind(Enum):
    """Register-fill order: how many distinct i- and j-particles per fill."""

    ONE_BY_V = "one_by_v"
    V_BY_ONE = "v_by_one"
    TWO_BY_HALF = "two_by_half"
    HALF_BY_TWO = "half_by_two"

    def shape(self, vector_width: int) -> tuple[int, int]:
        """(a, b) with a * b == vector_width (kernels.py:48-56)."""
        half = vector_width // 2
        return {
            PatternKind.ONE_BY_V: (1, vector_width),
            PatternKind.V_BY_ONE: (vector_width, 1),
            PatternKind.TWO_BY_HALF: (2, half),
            PatternKind.HALF_BY_TWO: (half, 2),
        }[self]

    @property
    def code(self) -> int:
        return _PATTERN_CODES[self]


_PATTERN_CODES = {PatternKind.ONE_BY_V: N.ONE_BY_V, PatternKind.V_BY_ONE: N.V_BY_ONE,
                  PatternKind.TWO_BY_HALF: N.TWO_BY_HALF, PatternKind.HALF_BY_TWO: N.HALF_BY_TWO}

PATTERN_ORDER = (
    PatternKind.ONE_BY_V,
    PatternKind.V_BY_ONE,
    PatternKind.TWO_BY_HALF,
    PatternKind.HALF_BY_TWO,
)

GPU_LANES = 32


def as_pattern(pattern) -> PatternKind:
    if isinstance(pattern, PatternKind):
        return pattern
    value = pattern if isinstance(pattern, str) else getattr(pattern, "value", None)
    if isinstance(value, str):
        try:
            return PatternKind(value)
        except ValueError:
            pass
    raise ConfigurationError(f"unknown pattern {pattern!r}")


@dataclass
class KernelStats:
    """Lane-slot accounting (kernels.py:67-89), plus energy/virial (extension).

    ``epot`` and ``virial`` are filled only when the force phase is asked for
    them; they do not take part in equality, so stats compare exactly as the
    reference's do.
    """

    kernel_invocations: int = 0
    lane_slots: int = 0
    useful_interactions: int = 0
    pair_interactions: int = 0
    epot: float = field(default=0.0, compare=False)
    virial: float = field(default=0.0, compare=False)

    @property
    def blank_lanes(self) -> int:
        return self.lane_slots - self.useful_interactions

    def merge(self, other: "KernelStats") -> None:
        self.kernel_invocations += other.kernel_invocations
        self.lane_slots += other.lane_slots
        self.useful_interactions += other.useful_interactions
        self.pair_interactions += other.pair_interactions
        self.epot += other.epot
        self.virial += other.virial


def validate_vector_width(vector_width: int) -> None:
    if not isinstance(vector_width, (int, np.integer)) or vector_width < 4 or (
            vector_width & (vector_width - 1)) != 0:
        raise ConfigurationError(
            f"vector width must be a power of two >= 4, got {vector_width}")


def blanks_expected(pattern: PatternKind, n_i: int, n_j: int, vector_width: int) -> int:
    """Closed-form blank lanes of the chunked double loop (kernels.py:98-109)."""
    if n_i < 0 or n_j < 0:
        raise ConfigurationError("buffer sizes must be non-negative")
    validate_vector_width(vector_width)
    a, b = as_pattern(pattern).shape(vector_width)
    return math.ceil(n_i / a) * math.ceil(n_j / b) * a * b - n_i * n_j


def lj_pair_force(displacement, params) -> np.ndarray:
    """Single-pair force on i for ``displacement = r_i - r_j`` (kernels.py:112-126)."""
    d = np.asarray(displacement, dtype=np.float64)
    r2 = float(d @ d)
    if r2 == 0.0:
        raise ParticleOverlapError("zero distance between interacting particles")
    if r2 >= params.cutoff * params.cutoff:
        return np.zeros(3)
    s2 = params.sigma * params.sigma / r2
    s6 = s2 * s2 * s2
    return (24.0 * params.epsilon) * (2.0 * s6 * s6 - s6) / r2 * d


# ------------------------------------------------------------ device plumbing
class _DeviceView:
    """A ParticleBuffer (ours, on CUDA, or any host SoA buffer with the
    reference's field names) presented as pos4 + SoA force tensors."""

    def __init__(self, buf, device):
        self.src = buf
        self.host = not (isinstance(buf, ParticleBuffer) and buf.device.type == "cuda")
        if self.host:
            self.dev = ParticleBuffer.from_host(buf, device=device)
        else:
            self.dev = buf
        n = len(self.dev)
        self.n = n
        self.pos4 = torch.empty((n, 4), dtype=torch.float64, device=device)
        if n:
            d = self.dev
            N.call("lmd_gather_pos4", n, None, N.ptr(d.pos_x), N.ptr(d.pos_y), N.ptr(d.pos_z),
                   N.ptr(d.ownership), 0.0, N.ptr(self.pos4), N.stream())

    def write_back(self):
        if not self.host or self.n == 0:
            return
        for name in ("force_x", "force_y", "force_z"):
            dst = getattr(self.src, name)
            val = getattr(self.dev, name)
            if isinstance(dst, torch.Tensor):
                dst.copy_(val)   # direct device -> (pinned) host DMA
            else:
                torch.from_numpy(dst).copy_(val)


def _device_for(*bufs) -> torch.device:
    for b in bufs:
        if isinstance(b, ParticleBuffer) and b.device.type == "cuda":
            return b.device
    if not torch.cuda.is_available():
        raise N.NativeLibraryError("the B200 force path needs a CUDA device (no CPU fallback)")
    return torch.device("cuda")


def _sweep(i_buf, j_buf, params, newton3, same_buffer, pattern, energy=False):
    dev = _device_for(i_buf, j_buf)
    vi = _DeviceView(i_buf, dev)
    vj = vi if same_buffer else _DeviceView(j_buf, dev)
    stats_t = N.new_stats(dev)
    counts = torch.zeros(6, dtype=torch.int64, device=dev)
    s = N.stream()
    if vi.n:
        N.call("lmd_buffer_counts", vi.n, N.ptr(vi.pos4), N.ptr(counts[:3]), s)
    if vj.n and not same_buffer:
        N.call("lmd_buffer_counts", vj.n, N.ptr(vj.pos4), N.ptr(counts[3:]), s)
    ev = None
    flags = N.FLAG_ENERGY if energy else 0
    if vi.n and vj.n:
        slots = N.load().lmd_pair_sweep_ev_slots(vi.n, pattern.code)
        ev = torch.empty(2 * slots, dtype=torch.float64, device=dev)
        di, dj = vi.dev, vj.dev
        N.call("lmd_pair_sweep", vi.n, N.ptr(vi.pos4), vj.n, N.ptr(vj.pos4), int(same_buffer),
               int(newton3), pattern.code, flags, N.make_lj(params),
               N.ptr(di.force_x), N.ptr(di.force_y), N.ptr(di.force_z),
               N.ptr(dj.force_x), N.ptr(dj.force_y), N.ptr(dj.force_z), N.ptr(ev),
               N.ptr(stats_t), s)
    st = N.read_stats(stats_t)
    c = counts.cpu().tolist()
    if st.overlap:
        vi.write_back()
        if not same_buffer:
            vj.write_back()
        raise ParticleOverlapError("zero distance between interacting particles")
    vi.write_back()
    if not same_buffer:
        vj.write_back()
    if same_buffer:
        useful = c[2] if newton3 else c[0] * max(c[1] - 1, 0)
    else:
        useful = c[0] * c[4]
    return st, useful, vi.n, vj.n


def compute_pair_vectorized(i_buf, j_buf, params, newton3: bool, same_buffer: bool, pattern,
                            vector_width: int, lane_sim: bool = False,
                            energy: bool = False) -> KernelStats:
    """Accumulate pair forces under a register-fill pattern on the GPU; return stats.

    Semantics of kernels.py:377-424: forces accumulate (+=); ``same_buffer``
    requires the identical buffer object; Newton3 writes the reaction into
    the j buffer.  ``lane_sim`` is accepted for API compatibility: the GPU
    lanes execute the same fills the interpreter materialises, and the
    statistics are the same closed forms either way.
    """
    validate_vector_width(vector_width)
    if not isinstance(pattern, PatternKind):
        pattern = as_pattern(pattern)
    if same_buffer and i_buf is not j_buf:
        raise ConfigurationError("same_buffer requires the identical buffer object")
    st, useful, ni, nj = _sweep(i_buf, j_buf, params, newton3, same_buffer, pattern, energy)
    a, b = pattern.shape(vector_width)
    inv = -(-ni // a) * -(-nj // b)
    return KernelStats(kernel_invocations=inv, lane_slots=inv * vector_width,
                       useful_interactions=useful, pair_interactions=int(st.pair_interactions),
                       epot=st.epot, virial=st.virial)


def compute_pair_scalar(i_buf, j_buf, params, newton3: bool, same_buffer: bool,
                        energy: bool = False) -> KernelStats:
    """The reference's scalar path (kernels.py:129-194), executed on the GPU.

    Same pair semantics as the vectorized functor; a scalar loop has no blank
    lanes, so ``lane_slots == useful_interactions`` and no invocations are
    counted beyond the examined slots.
    """
    if same_buffer and i_buf is not j_buf:
        raise ConfigurationError("same_buffer requires the identical buffer object")
    st, useful, _, _ = _sweep(i_buf, j_buf, params, newton3, same_buffer,
                              PatternKind.V_BY_ONE, energy)
    return KernelStats(kernel_invocations=0, lane_slots=useful, useful_interactions=useful,
                       pair_interactions=int(st.pair_interactions), epot=st.epot,
                       virial=st.virial)
