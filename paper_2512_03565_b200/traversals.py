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


# ---------------------------------------------------------------- schedules
def _lin_to_xyz(lin: np.ndarray, tdims) -> tuple:
    tx, ty, _ = (int(t) for t in tdims)
    return lin % tx, (lin // tx) % ty, lin // (tx * ty)


class _CellInfo:
    """Host copy of a linked-cell container's cell tables."""

    def __init__(self, cont):
        self.cont = cont
        self.tdims = np.asarray(cont.total_dims, dtype=np.int64)
        self.oc = cont._o_count.cpu().numpy().astype(np.int64)
        self.hc = cont._h_count.cpu().numpy().astype(np.int64)
        self.occ = np.zeros(len(self.oc), dtype=np.uint8)          # containers.py:93-94
        self.occ[self.hc > 0] = 2
        self.occ[self.oc > 0] = 1
        self.owned = np.nonzero(self.oc)[0].astype(np.int64)
        self.halo = np.nonzero(self.hc)[0].astype(np.int64)
        self._views: dict = {}

    def buf(self, lin: int):
        v = self._views.get(lin)
        if v is None:
            v = self.cont.buffer_at(int(lin))
            self._views[lin] = v
        return v


def _pair_units(units, ci: _CellInfo, a, b, a_halo, b_halo, newton3, color, base):
    """_emit_pair (traversals.py:152-165): halo pairs one-sided (owned side i),
    owned pairs once with Newton3 or both orders without."""
    if a_halo or b_halo:
        if a_halo:
            a, b = b, a
        units.append(WorkUnit(ci.buf(a), ci.buf(b), False, color, base, False, a, b))
    elif newton3:
        units.append(WorkUnit(ci.buf(a), ci.buf(b), False, color, base, True, a, b))
    else:
        units.append(WorkUnit(ci.buf(a), ci.buf(b), False, color, base, False, a, b))
        units.append(WorkUnit(ci.buf(b), ci.buf(a), False, color, base, False, b, a))


def _forward_pairs(ci: _CellInfo):
    """Occupied adjacent cell pairs, each once from its lower-index anchor,
    halo-halo skipped (traversals.py:125-149).  The anchor list repeats a
    cell that holds both owned particles and images, as the reference's
    concatenation does."""
    anchors = np.concatenate([ci.owned, ci.halo])
    if anchors.size == 0:
        return
    x, y, z = _lin_to_xyz(anchors, ci.tdims)
    tx, ty, tz = (int(t) for t in ci.tdims)
    a_halo = ci.occ[anchors] == 2
    for d in FORWARD_DIRS:
        nx, ny, nz = x + d[0], y + d[1], z + d[2]
        inside = (nx >= 0) & (nx < tx) & (ny >= 0) & (ny < ty) & (nz >= 0) & (nz < tz)
        nlin = np.where(inside, nx + tx * (ny + ty * nz), 0)
        st = ci.occ[nlin]
        keep = inside & (st != 0) & ~(a_halo & (st == 2))
        if keep.any():
            yield anchors[keep], nlin[keep], a_halo[keep], st[keep] == 2, d


def _sorted_schedule(kind, newton3, units, n_colors) -> Schedule:
    units.sort(key=lambda u: u.color)          # stable: traversals.py:168-170
    return Schedule(kind, newton3, tuple(units), n_colors)


def _schedule_lc(cont, kind: TraversalKind, newton3: bool) -> Schedule:
    ci = _CellInfo(cont)
    units: list = []
    tx, ty, _ = (int(t) for t in ci.tdims)
    if kind is TraversalKind.LC_C01:             # traversals.py:173-187
        x, y, z = _lin_to_xyz(ci.owned, ci.tdims)
        for d in ALL_DIRS:
            nlin = (x + d[0]) + tx * ((y + d[1]) + ty * (z + d[2]))
            hit = ci.occ[nlin] != 0
            for a, b in zip(ci.owned[hit].tolist(), nlin[hit].tolist()):
                units.append(WorkUnit(ci.buf(a), ci.buf(b), a == b, 0, a, False, a, b))
        return _sorted_schedule(kind, False, units, 1)
    x, y, z = _lin_to_xyz(ci.owned, ci.tdims)
    if kind is TraversalKind.LC_C18:
        colors = (x % 3) + 3 * (y % 3) + 9 * (z % 2)
    else:
        colors = (x % 2) + 2 * (y % 2) + 4 * (z % 2)
    for c, col in zip(ci.owned.tolist(), colors.tolist()):
        units.append(WorkUnit(ci.buf(c), ci.buf(c), True, col, c, newton3, c, c))
    for anchors, nbrs, ah, bh, d in _forward_pairs(ci):
        axc, ayc, azc = _lin_to_xyz(anchors, ci.tdims)
        if kind is TraversalKind.LC_C18:         # traversals.py:190-211
            cols = (axc % 3) + 3 * (ayc % 3) + 9 * (azc % 2)
            bases = anchors
            swap = False
        else:                                    # traversals.py:214-241
            bx = axc + min(d[0], 0)
            by = ayc + min(d[1], 0)
            bz = azc + min(d[2], 0)
            bases = bx + tx * (by + ty * bz)
            cols = np.mod(bx, 2) + 2 * np.mod(by, 2) + 4 * np.mod(bz, 2)
            r1, r2 = c08_ranks(d)
            swap = r2 < r1
        for a, b, a_h, b_h, col, base in zip(anchors.tolist(), nbrs.tolist(), ah.tolist(),
                                             bh.tolist(), cols.tolist(), bases.tolist()):
            if swap:
                a, b, a_h, b_h = b, a, b_h, a_h
            _pair_units(units, ci, a, b, a_h, b_h, newton3, col, base)
    return _sorted_schedule(kind, newton3, units, 18 if kind is TraversalKind.LC_C18 else 8)


def greedy_base_colors(n: int, lists) -> tuple[list, int]:
    """Smallest free color per base so equal-color write sets are disjoint
    (traversals.py:269-287)."""
    writes = [set([k]) | set(lists[k]) for k in range(n)]
    writers: dict = {}
    for k, ws in enumerate(writes):
        for z in ws:
            writers.setdefault(z, []).append(k)
    colors = [-1] * n
    for k in range(n):
        taken = {colors[o] for z in writes[k] for o in writers[z] if o != k and colors[o] >= 0}
        c = 0
        while c in taken:
            c += 1
        colors[k] = c
    return colors, (max(colors) + 1 if colors else 1)


def _schedule_vcl(cont, newton3: bool) -> Schedule:
    """traversals.py:244-266 on the device cluster container."""
    lists = cont.neighbor_lists[newton3]
    links = cont.halo_links
    n = cont.n_clusters
    M = cont.cluster_size
    colors, n_colors = greedy_base_colors(n, lists) if newton3 else ([0] * n, 1)
    own, hal = cont.kernel_backings()
    units: list = []

    def view(backing, which, k):
        v = backing.view(k * M, (k + 1) * M)
        v.backing_slot = (which, k * M, M)
        return v

    for k in range(n):
        b = view(own, 0, k)
        col = colors[k]
        units.append(WorkUnit(b, b, True, col, k, newton3, k, k))
        for z in lists[k]:
            units.append(WorkUnit(b, view(own, 0, z), False, col, k, newton3, k, z))
        for h in links[k]:
            units.append(WorkUnit(b, view(hal, 1, h), False, col, k, False, k, n + h))
    return _sorted_schedule(TraversalKind.VCL, newton3, units, n_colors)


def schedule(container, kind, newton3: bool) -> Schedule:
    """Ordered, colored work units of one force phase (traversals.py:108-122)."""
    kind = as_traversal(kind)
    ck = getattr(container, "kind", None)
    if kind is TraversalKind.VCL:
        if ck != "vcl":
            raise ConfigurationError("vcl traversal requires the cluster container")
        return _schedule_vcl(container, newton3)
    if kind is TraversalKind.VL:
        raise ConfigurationError("verlet lists are executed by their container, not a schedule")
    if ck != "lc":
        raise ConfigurationError(f"{kind.value} traversal requires linked cells")
    if kind is TraversalKind.LC_C01 and newton3:
        raise ConfigurationError("lc_c01 cannot exploit Newton's third law")
    return _schedule_lc(container, kind, newton3)


def verify_coloring(sched: Schedule) -> bool:
    """Same color => disjoint write sets across bases (traversals.py:290-305)."""
    owner: dict = {}
    for u in sched.units:
        for buf in ((u.i_buffer, u.j_buffer) if u.newton3 else (u.i_buffer,)):
            key = (u.color, id(buf))
            if owner.setdefault(key, u.base_index) != u.base_index:
                return False
    return True
