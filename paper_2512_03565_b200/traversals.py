"""Traversal kinds and the reference's host-side work-unit schedules.

On the device a traversal is a kernel, not a list of units: the linked-cell
kernels walk every owned cell's 27-cell shell (Newton3 off) or the colored
cell-pair bases (Newton3 on), the Verlet-list and cluster-list kernels walk
their lists.  For API compatibility and for checking the coloring contract
this module still materialises the reference's ordered, colored unit lists
(traversals.py:108-305) from a container's occupancy on the host.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _native as N
from .errors import ConfigurationError


class TraversalKind(Enum):
    LC_C01 = "lc_c01"
    LC_C08 = "lc_c08"
    LC_C18 = "lc_c18"
    VCL = "vcl"
    VL = "vl"          # extension: plain Verlet lists with a skin


TRAVERSAL_ORDER = (TraversalKind.LC_C01, TraversalKind.LC_C08, TraversalKind.LC_C18,
                   TraversalKind.VCL, TraversalKind.VL)

_CODES = {TraversalKind.LC_C01: N.LC_C01, TraversalKind.LC_C08: N.LC_C08,
          TraversalKind.LC_C18: N.LC_C18, TraversalKind.VCL: N.VCL, TraversalKind.VL: N.VL}


def as_traversal(kind) -> TraversalKind:
    if isinstance(kind, TraversalKind):
        return kind
    value = getattr(kind, "value", kind)
    try:
        return TraversalKind(value)
    except ValueError as exc:
        raise ConfigurationError(f"unknown traversal {kind!r}") from exc


def traversal_code(kind) -> int:
    return _CODES[as_traversal(kind)]


@dataclass(slots=True)
class WorkUnit:
    """One i-buffer x j-buffer task (traversals.py:51-68)."""

    i_buffer: object
    j_buffer: object
    same_buffer: bool
    color: int
    base_index: int
    newton3: bool
    i_index: int
    j_index: int


@dataclass(frozen=True)
class Schedule:
    kind: TraversalKind
    newton3: bool
    units: tuple
    n_colors: int


# 13 forward directions (strictly positive x-fastest offset) and all 27, in
# itertools.product order (traversals.py:79-84)
FORWARD_DIRS = tuple(d for d in itertools.product((-1, 0, 1), repeat=3)
                     if (d[2], d[1], d[0]) > (0, 0, 0))
ALL_DIRS = tuple(itertools.product((-1, 0, 1), repeat=3))


def c08_ranks(d) -> tuple[int, int]:
    """In-block ranks of the two cells of a pair along d (traversals.py:94-105)."""
    lo = [max(-c, 0) for c in d]
    hi = [max(c, 0) for c in d]
    return 4 * lo[0] + 2 * lo[1] + lo[2], 4 * hi[0] + 2 * hi[1] + hi[2]
