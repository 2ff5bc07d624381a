"""Verlet cluster lists on the device (VerletClusterContainer, containers.py:302-479).

Clusters follow the reference exactly: x-y columns of side rc + skin, each
column sorted by z (``np.lexsort((z, col))``) and chunked into M-slot
clusters, the last one dummy-padded with its dummies parked at the AABB
minimum.  Cluster pairs are those whose AABB gap^2 <= (rc+skin)^2, found by a
binned search (K6) instead of the reference's dense O(C^2) matrix.  Halo
clusters and halo links are re-derived on every ``refresh`` as the reference
does; the owned lists stay fixed between rebuilds.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .containers import _check_all_owned, device_soa, needs_rebuild_buffer
from .domain import as_box, build_halo
from .errors import ConfigurationError, ParticleOverlapError
from .kernels import KernelStats, as_pattern, validate_vector_width
from .particles import HALO, OWNED, ParticleBuffer

REBUILD_PERIOD_DEFAULT = 20


@dataclass
class Cluster:
    """Fixed-size particle group (containers.py:201-213), as a host view."""

    cluster_id: int
    buffer: object
    aabb_min: np.ndarray
    aabb_max: np.ndarray
    n_real: int

    @property
    def size(self) -> int:
        return len(self.buffer)


class _Clustered:
    """Device clustering of one particle set (owned or halo)."""

    def __init__(self, n, M, dev):
        self.n = n
        self.M = M
        self.ncl = 0
        self.order = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        self.slot = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        self.ckey = torch.empty(max(n, 1), dtype=torch.int32, device=dev)


def _cluster(x, y, z, box, col, width, M, dev) -> _Clustered:
    n = int(x.shape[0])
    out = _Clustered(n, M, dev)
    if n == 0:
        return out
    L = N.load()
    tb = int(L.lmd_vcl_temp_bytes(n))
    temp = torch.empty(max(tb, 1), dtype=torch.uint8, device=dev)
    i32 = lambda: torch.empty(n, dtype=torch.int32, device=dev)  # noqa: E731
    colkey, ckey2, tmp_idx, sorted_key = i32(), i32(), i32(), i32()
    zkey = torch.empty(n, dtype=torch.int64, device=dev)
    zkey2 = torch.empty(n, dtype=torch.int64, device=dev)
    s = N.stream()
    N.call("lmd_vcl_order", n, N.ptr(x), N.ptr(y), N.ptr(z), float(box.min[0]), float(box.min[1]),
           float(col), int(width), N.ptr(colkey), N.ptr(ckey2), N.ptr(zkey), N.ptr(zkey2),
           N.ptr(tmp_idx), N.ptr(out.order), N.ptr(sorted_key), N.ptr(temp), tb, s)
    flag, run_id, run_start, run_nclu, run_coff = i32(), i32(), i32(), i32(), i32()
    ncl = N.I64_out()
    N.call("lmd_vcl_chunk", n, M, N.ptr(sorted_key), N.ptr(flag), N.ptr(run_id), N.ptr(run_start),
           N.ptr(run_nclu), N.ptr(run_coff), N.ptr(out.slot), N.ptr(out.ckey), ncl, N.ptr(temp),
           tb, s)
    out.ncl = int(ncl.value)
    out.ckey = out.ckey[: out.ncl].contiguous()
    return out


class VerletClusterContainer:
    """Cluster-list container on the GPU: owned clusters plus per-refresh halo clusters."""

    kind = "vcl"

    def __init__(self, box, params, cluster_size: int,
                 rebuild_period: int = REBUILD_PERIOD_DEFAULT, device=None):
        if cluster_size < 2:
            raise ConfigurationError(f"cluster size must be >= 2, got {cluster_size}")
        self.box = as_box(box)
        self.params = params
        self.cluster_size = int(cluster_size)
        self.rebuild_period = rebuild_period
        self.column_length = params.interaction_length
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu"))
        L = self.box.lengths
        self.width = int(L[0] / self.column_length) + 4            # containers.py:340
        self.height = int(L[1] / self.column_length) + 4
        self.tsize = self.width * self.height
        self.reference_positions = None
        self.steps_since_rebuild = 0
        self.structure_version = 0
        # interaction orders as warp lane templates (lmd_force_vcl_order; an
        # order aligned with the cluster size runs as the stream kernel, whose
        # mapping it is; "strict": the lane-template kernel even then);
        # False: the packed stream kernel for every order (the cluster-aligned
        # M x 32/M mapping with hit compaction, the fastest one on the GPU)
        self.order_kernels = type(self).ORDER_KERNELS
        # stream kernel: cutoff tests in FP32 with an error band, exact FP64
        # decision for the pairs that pass (same pairs; the FP64 pipe is the
        # scarce one)
        self.fp32_tests = True
        self._pos4f = None
        self._own = None
        self._stats_cache: dict = {}

    ORDER_KERNELS = True   # default of ``order_kernels`` for new containers

    # ------------------------------------------------------------ protocol
    def needs_rebuild(self, owned) -> bool:
        d = device_soa(owned)
        return needs_rebuild_buffer(d, self.reference_positions, self.params.skin,
                             self.steps_since_rebuild, self.rebuild_period)

    def _table(self, cl: _Clustered, dev):
        tbeg = torch.zeros(self.tsize, dtype=torch.int32, device=dev)
        tend = torch.zeros(self.tsize, dtype=torch.int32, device=dev)
        N.call("lmd_vcl_column_table", cl.ncl, N.ptr(cl.ckey), N.ptr(tbeg), N.ptr(tend),
               self.tsize, N.stream())
        return tbeg, tend

    def _lists(self, a_min, a_max, b_min, b_max, tbeg, tend, exclude_self, want_n3, dev):
        ncl = self._own.ncl
        rl = self.params.interaction_length
        limit = rl * rl                                   # containers.py:291
        count = torch.zeros(max(ncl, 1), dtype=torch.int32, device=dev)
        n3 = torch.zeros(max(ncl, 1), dtype=torch.int32, device=dev) if want_n3 else None
        s = N.stream()
        N.call("lmd_vcl_pairs", ncl, N.ptr(self._own.ckey), N.ptr(a_min), N.ptr(a_max),
               N.ptr(b_min), N.ptr(b_max), N.ptr(tbeg), N.ptr(tend), self.width, self.tsize,
               int(exclude_self), float(rl), float(limit), N.ptr(count), N.ptr(n3), None, None, s)
        c64 = count[:ncl].to(torch.int64)
        off = torch.zeros(max(ncl, 1), dtype=torch.int64, device=dev)
        if ncl > 1:
            off[1:ncl] = torch.cumsum(c64, 0)[:-1]
        total = int(c64.sum().item()) if ncl else 0
        lst = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
        if total:
            N.call("lmd_vcl_pairs", ncl, N.ptr(self._own.ckey), N.ptr(a_min), N.ptr(a_max),
                   N.ptr(b_min), N.ptr(b_max), N.ptr(tbeg), N.ptr(tend), self.width, self.tsize,
                   int(exclude_self), float(rl), float(limit), N.ptr(count), None, N.ptr(off),
                   N.ptr(lst), s)
        return count, n3, off, lst

    def rebuild(self, owned, halo=None) -> None:
        """``halo`` is accepted for protocol uniformity; images enter at refresh."""
        d = device_soa(owned)
        _check_all_owned(d)
        dev = d.device
        M = self.cluster_size
        self._own = _cluster(d.pos_x, d.pos_y, d.pos_z, self.box, self.column_length, self.width,
                             M, dev)
        self._owned_pos4 = torch.empty((max(self._own.ncl * M, 1), 4), dtype=torch.float64,
                                       device=dev)
        ncl = self._own.ncl
        self._amin = torch.empty((max(ncl, 1), 3), dtype=torch.float64, device=dev)
        self._amax = torch.empty((max(ncl, 1), 3), dtype=torch.float64, device=dev)
        self._load_owned(d)
        self._tbeg, self._tend = self._table(self._own, dev)
        self._count, self._n3count, self._off, self._list = self._lists(
            self._amin, self._amax, self._amin, self._amax, self._tbeg, self._tend, True, True,
            dev)
        self.reference_positions = d.positions().clone()
        self.steps_since_rebuild = 0
        self.structure_version += 1
        self._stats_cache.clear()
        self._halo_ready = False

    def _load_owned(self, d) -> None:
        M = self.cluster_size
        N.call("lmd_vcl_backing", self._own.n, self._own.ncl, M, N.ptr(self._own.order),
               N.ptr(self._own.slot), N.ptr(d.pos_x), N.ptr(d.pos_y), N.ptr(d.pos_z),
               float(OWNED), N.ptr(self._owned_pos4), N.ptr(self._amin), N.ptr(self._amax),
               N.stream())

    def refresh(self, owned, halo=None) -> None:
        """Reload positions into the clusters, recompute the AABBs (dummies
        re-parked) and re-derive the halo clusters and links (containers.py:431-469)."""
        if self._own is None:
            raise ConfigurationError("cluster container has not been rebuilt")
        d = device_soa(owned)
        dev = d.device
        M = self.cluster_size
        self._load_owned(d)
        if halo is None:
            halo = build_halo(d, self.box, self.params.interaction_length)
        h = device_soa(halo, dev)
        self._hal = _cluster(h.pos_x, h.pos_y, h.pos_z, self.box, self.column_length, self.width,
                             M, dev)
        nh = self._hal.ncl
        ncl = self._own.ncl
        self._pos4 = torch.empty(((ncl + nh) * M + 1, 4), dtype=torch.float64, device=dev)
        self._pos4[: ncl * M] = self._owned_pos4[: ncl * M]
        self._hmin = torch.empty((max(nh, 1), 3), dtype=torch.float64, device=dev)
        self._hmax = torch.empty((max(nh, 1), 3), dtype=torch.float64, device=dev)
        if nh:
            N.call("lmd_vcl_backing", self._hal.n, nh, M, N.ptr(self._hal.order),
                   N.ptr(self._hal.slot), N.ptr(h.pos_x), N.ptr(h.pos_y), N.ptr(h.pos_z),
                   float(HALO), N.ptr(self._pos4[ncl * M:]), N.ptr(self._hmin), N.ptr(self._hmax),
                   N.stream())
            htb, hte = self._table(self._hal, dev)
            self._hcount, _, self._hoff, self._hlist = self._lists(
                self._amin, self._amax, self._hmin, self._hmax, htb, hte, False, False, dev)
        else:
            self._hcount = torch.zeros(max(ncl, 1), dtype=torch.int32, device=dev)
            self._hoff = torch.zeros(max(ncl, 1), dtype=torch.int64, device=dev)
            self._hlist = torch.zeros(1, dtype=torch.int32, device=dev)
        n = self._own.ncl * M
        self._fx = torch.zeros(max(n, 1), dtype=torch.float64, device=dev)
        self._fy = torch.zeros(max(n, 1), dtype=torch.float64, device=dev)
        self._fz = torch.zeros(max(n, 1), dtype=torch.float64, device=dev)
        self.structure_version += 1
        self._stats_cache.clear()
        self._halo_ready = True

    # --------------------------------------------------------------- views
    def kernel_backings(self):
        """(owned, halo) padded backings as device views (containers.py:471-473)."""
        M = self.cluster_size
        n = self._own.ncl * M
        nh = self._hal.ncl * M if self._halo_ready else 0
        dev = self._pos4.device

        def mk(a, b, fx, fy, fz):
            p = self._pos4[a:b]
            z = torch.zeros(b - a, dtype=torch.float64, device=dev)
            return ParticleBuffer(pos_x=p[:, 0], pos_y=p[:, 1], pos_z=p[:, 2], vel_x=z, vel_y=z,
                                  vel_z=z, force_x=fx, force_y=fy, force_z=fz, old_force_x=z,
                                  old_force_y=z, old_force_z=z,
                                  id=torch.full((b - a,), -1, dtype=torch.int64, device=dev),
                                  ownership=p[:, 3].to(torch.int8))
        if not hasattr(self, "_hfx") or self._hfx.shape[0] != max(nh, 1):
            self._hfx = torch.zeros(max(nh, 1), dtype=torch.float64, device=dev)
            self._hfy = torch.zeros(max(nh, 1), dtype=torch.float64, device=dev)
            self._hfz = torch.zeros(max(nh, 1), dtype=torch.float64, device=dev)
        return (mk(0, n, self._fx[:n], self._fy[:n], self._fz[:n]),
                mk(n, n + nh, self._hfx[:nh], self._hfy[:nh], self._hfz[:nh]))

    @property
    def n_clusters(self) -> int:
        return self._own.ncl if self._own else 0

    @property
    def neighbor_lists(self) -> dict:
        """{newton3: list of neighbour-id lists} as in containers.py:421-426 (host copy)."""
        off = self._off.cpu().numpy()
        cnt = self._count.cpu().numpy()
        lst = self._list.cpu().numpy()
        full = [lst[off[k]:off[k] + cnt[k]].tolist() for k in range(self.n_clusters)]
        return {False: full, True: [[z for z in zs if z > k] for k, zs in enumerate(full)]}

    @property
    def halo_links(self) -> list:
        off = self._hoff.cpu().numpy()
        cnt = self._hcount.cpu().numpy()
        lst = self._hlist.cpu().numpy()
        return [lst[off[k]:off[k] + cnt[k]].tolist() for k in range(self.n_clusters)]

    def structure(self) -> dict:
        """perm / slots / real counts / AABBs / padded positions (host copies)."""
        M = self.cluster_size
        ncl = self.n_clusters
        slots = self._own.slot[: self._own.n].cpu().numpy().astype(np.int64)
        counts = np.bincount(slots // M, minlength=ncl)
        return dict(perm=self._own.order[: self._own.n].cpu().numpy().astype(np.int64),
                    slots=slots, counts=counts,
                    aabb_min=self._amin[:ncl].cpu().numpy(), aabb_max=self._amax[:ncl].cpu().numpy(),
                    padded=self._owned_pos4[: ncl * M, :3].cpu().numpy())

    # ---------------------------------------------------------------- force
    def launch_force(self, energy: bool = False, stats_t=None, ev_t=None, pattern=None):
        """Force kernel over the cluster lists.  With ``pattern`` (and
        ``order_kernels``) the interaction order is the warp's lane template
        (lmd_force_vcl_order); without, the packed stream kernel."""
        if not self._halo_ready:
            raise ConfigurationError("cluster container has not been refreshed")
        dev = self._pos4.device
        if stats_t is None:
            stats_t = N.new_stats(dev)
        else:
            stats_t.zero_()
        ncl = self._own.ncl
        if ev_t is None:
            ev_t = torch.empty(2 * max(int(N.load().lmd_vcl_ev_slots(ncl)), 1),
                               dtype=torch.float64, device=dev)
        # an order whose i-side is exactly one cluster (A = M: v_by_one at
        # M = 32, half_by_two at 16, two_by_half at 2, one_by_v at 1) IS the
        # stream kernel's M x 32/M mapping, which also compacts hits
        aligned = (pattern is not None and
                   as_pattern(pattern).shape(32)[0] == self.cluster_size)
        if (pattern is not None and self.order_kernels and self.cluster_size <= 32
                and not (aligned and self.order_kernels != "strict")):
            N.call("lmd_force_vcl_order", ncl, self.cluster_size, as_pattern(pattern).code,
                   N.FLAG_ENERGY if energy else 0, N.make_lj(self.params), N.ptr(self._pos4),
                   N.ptr(self._off), N.ptr(self._count), N.ptr(self._list), N.ptr(self._hoff),
                   N.ptr(self._hcount), N.ptr(self._hlist), N.ptr(self._amin),
                   N.ptr(self._amax), N.ptr(self._hmin), N.ptr(self._hmax), N.ptr(self._fx),
                   N.ptr(self._fy), N.ptr(self._fz), N.ptr(ev_t), N.ptr(stats_t), N.stream())
            return stats_t
        nrec = int(self._pos4.shape[0])
        if self._pos4f is None or self._pos4f.shape[0] < nrec:
            self._pos4f = torch.empty((nrec, 4), dtype=torch.float32, device=dev)
        # coordinates of owned particles, images and parked dummies stay within
        # the box grown by the interaction length (plus mid-step drift)
        max_abs = float(max(np.abs(self.box.min).max(), np.abs(self.box.max).max())) + \
            2.0 * float(self.params.interaction_length) + 1.0
        N.call("lmd_force_vcl", ncl, self.cluster_size, N.FLAG_ENERGY if energy else 0,
               N.make_lj(self.params), N.ptr(self._pos4), N.ptr(self._off), N.ptr(self._count),
               N.ptr(self._list), N.ptr(self._hoff), N.ptr(self._hcount), N.ptr(self._hlist),
               N.ptr(self._fx), N.ptr(self._fy), N.ptr(self._fz), N.ptr(ev_t), N.ptr(stats_t),
               nrec, N.ptr(self._pos4f) if self.fp32_tests else None, max_abs, N.stream())
        return stats_t

    def vcl_stats(self, newton3: bool, pattern, V: int):
        key = (self.structure_version, bool(newton3), pattern, V)
        hit = self._stats_cache.get(key)
        if hit is None:
            a, b = pattern.shape(V)
            t = N.new_stats(self._pos4.device)
            nclt = int(self._pos4.shape[0]) // self.cluster_size
            nd = torch.empty(max(nclt, 1), dtype=torch.int32, device=self._pos4.device)
            N.call("lmd_vcl_stats", self._own.ncl, self.cluster_size, int(newton3), a, b, V,
                   N.ptr(self._pos4), N.ptr(self._off), N.ptr(self._count), N.ptr(self._n3count),
                   N.ptr(self._list), N.ptr(self._hoff), N.ptr(self._hcount), N.ptr(self._hlist),
                   nclt, N.ptr(nd), N.ptr(t), N.stream())
            st = N.read_stats(t)
            hit = (int(st.kernel_invocations), int(st.lane_slots), int(st.useful_interactions))
            self._stats_cache[key] = hit
        return hit

    def compute_forces(self, traversal, newton3: bool, pattern, vector_width: int,
                       energy: bool = False) -> KernelStats:
        from .traversals import TraversalKind, as_traversal
        validate_vector_width(vector_width)
        if as_traversal(traversal) is not TraversalKind.VCL:
            raise ConfigurationError(f"{traversal} traversal requires linked cells")
        pattern = as_pattern(pattern)
        inv, slots, useful = self.vcl_stats(newton3, pattern, vector_width)
        st = N.read_stats(self.launch_force(energy, pattern=pattern))
        if st.overlap:
            raise ParticleOverlapError("zero distance between interacting particles")
        pairs = int(st.pair_interactions)
        if newton3:
            oh = int(st.pairs_owned_halo)
            pairs = (pairs - oh) // 2 + oh
        return KernelStats(kernel_invocations=inv, lane_slots=slots, useful_interactions=useful,
                           pair_interactions=pairs, epot=st.epot, virial=st.virial)

    def collect_forces(self, owned) -> None:
        d = device_soa(owned)
        n = self._own.n
        if n:
            N.call("lmd_vcl_collect", n, N.ptr(self._own.order), N.ptr(self._own.slot),
                   N.ptr(self._fx), N.ptr(self._fy), N.ptr(self._fz), N.ptr(d.force_x),
                   N.ptr(d.force_y), N.ptr(d.force_z), N.stream())
        if d is not owned:
            for name in ("force_x", "force_y", "force_z"):
                dst = getattr(owned, name)
                val = getattr(d, name)
                if isinstance(dst, torch.Tensor):
                    dst.copy_(val)   # direct device -> (pinned) host DMA
                else:
                    torch.from_numpy(dst).copy_(val)


# ------------------------------------------------------- standalone cluster API
def build_clusters(buf, size: int, column_length: float | None = None) -> list:
    """Group particles into clusters of exactly ``size`` entries
    (containers.py:216-247), on the device: x-y columns of ``column_length``
    (default: the particles' x/y span over floor(sqrt(n / size)) columns,
    slightly widened), each column ordered by z (a stable lexsort as two
    stable device sorts), chunked into ``size``; a column's last chunk is
    padded with DUMMY entries parked at its bounding-box minimum.  Returns
    :class:`Cluster` objects whose buffers are device ParticleBuffers."""
    import math
    if size < 2:
        raise ConfigurationError(f"cluster size must be >= 2, got {size}")
    d = device_soa(buf)
    n = len(d)
    if n == 0:
        return []
    x, y, z = d.pos_x, d.pos_y, d.pos_z
    xmin, ymin = x.min(), y.min()
    if column_length is None:
        span = max(float((x.max() - xmin).item()), float((y.max() - ymin).item()), 1e-12)
        column_length = span * (1.0 + 1e-9) / max(1, int(math.sqrt(n / size)))
    col_x = torch.floor((x - xmin) / column_length).to(torch.int64)
    col_y = torch.floor((y - ymin) / column_length).to(torch.int64)
    col = col_x + col_y * (col_x.max() + 1)
    # np.lexsort((z, col)): stable by z, then stable by col
    o1 = torch.sort(z, stable=True).indices
    order = o1[torch.sort(col[o1], stable=True).indices]
    scol = col[order]
    starts = torch.nonzero(torch.diff(scol)).flatten() + 1
    bounds = [0] + starts.tolist() + [n]
    clusters = []
    cid = 0
    for b in range(len(bounds) - 1):
        lo, hi = bounds[b], bounds[b + 1]
        for s0 in range(lo, hi, size):
            clusters.append(_make_cluster(cid, d, order[s0:min(s0 + size, hi)], size))
            cid += 1
    return clusters


def _make_cluster(cid: int, src, members, size: int) -> Cluster:
    """containers.py:250-268 on device buffers."""
    n_real = int(members.shape[0])
    cb = ParticleBuffer.empty(size, device=src.device)
    for name in tuple(ParticleBuffer._FLOAT_FIELDS) + ("id", "ownership"):
        getattr(cb, name)[:n_real] = getattr(src, name)[members]
    pos = torch.stack([cb.pos_x[:n_real], cb.pos_y[:n_real], cb.pos_z[:n_real]], dim=1)
    amin = pos.min(dim=0).values
    amax = pos.max(dim=0).values
    if n_real < size:
        cb.pos_x[n_real:] = amin[0]
        cb.pos_y[n_real:] = amin[1]
        cb.pos_z[n_real:] = amin[2]
        cb.id[n_real:] = -1
        cb.ownership[n_real:] = 2   # DUMMY
    return Cluster(cid, cb, amin.cpu().numpy(), amax.cpu().numpy(), n_real)


def build_cluster_neighbor_lists(clusters: list, interaction_length: float,
                                 newton3: bool) -> list:
    """Neighbour cluster ids per cluster by bounding-box distance
    (containers.py:271-299): d2 = sum of squared per-axis gaps, listed iff
    d2 <= interaction_length^2; with ``newton3`` each unordered pair once
    (the lower id keeps it), else in both lists; never self.  The gap
    expression is evaluated on the device in the reference's order, in
    blocks of rows (the reference's dense C x C matrix, without the
    memory)."""
    n = len(clusters)
    if n == 0:
        return []
    dev = torch.device("cuda") if torch.cuda.is_available() else None
    if dev is None:
        raise ConfigurationError("build_cluster_neighbor_lists needs a CUDA device")
    mins = torch.as_tensor(np.stack([c.aabb_min for c in clusters]), dtype=torch.float64,
                           device=dev)
    maxs = torch.as_tensor(np.stack([c.aabb_max for c in clusters]), dtype=torch.float64,
                           device=dev)
    limit = interaction_length * interaction_length
    ids = torch.arange(n, device=dev)
    lists = []
    block = 2048
    for r0 in range(0, n, block):
        a0, a1 = mins[r0:r0 + block, None, :], maxs[r0:r0 + block, None, :]
        gap = torch.clamp(torch.maximum(a0 - maxs[None, :, :], mins[None, :, :] - a1), min=0.0)
        g2 = gap * gap
        d2 = (g2[..., 0] + g2[..., 1]) + g2[..., 2]
        close = d2 <= limit
        rows = ids[r0:r0 + block, None]
        keep = close & ((ids[None, :] > rows) if newton3 else (ids[None, :] != rows))
        for row in keep.cpu().numpy():
            lists.append([int(z) for z in np.nonzero(row)[0]])
    return lists
