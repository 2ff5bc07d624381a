"""Neighbor identification on the device: linked cells (and, in sibling
modules, Verlet lists and Verlet cluster lists).

Mirrors the reference's containers.py (23-198).  The container keeps a
cell-sorted backing of the owned particles followed by the sorted periodic
images, packed as double4 {x, y, z, ownership} in HBM, with per-cell
(start, count) tables in the ring-padded grid.  Binning and sorting are
CUDA kernels (K1: bit-exact cell index, CUB stable radix sort); the force
sweep is K2 (``lmd_force_lc``).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from .domain import SimulationBox, as_box, build_halo
from .errors import ConfigurationError, DegenerateDomainError
from .kernels import KernelStats, PatternKind, as_pattern, validate_vector_width
from .particles import HALO, OWNED, ParticleBuffer

REBUILD_PERIOD_DEFAULT = 20


def needs_rebuild(positions, reference_positions, skin: float, steps_since_rebuild: int,
                  period: int = REBUILD_PERIOD_DEFAULT) -> bool:
    """True when any particle moved at least skin/2 or the period elapsed
    (containers.py:23-38).  Works on torch tensors (any device) or arrays."""
    if steps_since_rebuild >= period:
        return True
    if reference_positions is None or tuple(reference_positions.shape) != tuple(positions.shape):
        return True
    if isinstance(positions, torch.Tensor):
        ref = reference_positions
        if not isinstance(ref, torch.Tensor):
            ref = torch.as_tensor(np.asarray(ref), device=positions.device)
        if positions.shape[0] == 0:
            return False
        d = positions - ref
        sq = d * d
        disp2 = (sq[:, 0] + sq[:, 1]) + sq[:, 2]
        return bool((disp2.max() >= (0.5 * skin) ** 2).item())
    positions = np.asarray(positions)
    disp2 = ((positions - np.asarray(reference_positions)) ** 2).sum(axis=1)
    if disp2.size == 0:
        return False
    return bool(disp2.max() >= (0.5 * skin) ** 2)


def needs_rebuild_buffer(buf: ParticleBuffer, reference_positions, skin: float,
                         steps_since_rebuild: int, period: int) -> bool:
    """needs_rebuild for a device buffer: one fused max-displacement kernel
    and one 8-byte read instead of stacking the positions."""
    if steps_since_rebuild >= period:
        return True
    n = len(buf)
    if reference_positions is None or tuple(reference_positions.shape) != (n, 3):
        return True
    if n == 0:
        return False
    if skin <= 0.0:            # any displacement >= 0: no need to look
        return True
    out = torch.empty(1, dtype=torch.float64, device=buf.device)
    N.call("lmd_max_displacement2", n, N.ptr(buf.pos_x), N.ptr(buf.pos_y), N.ptr(buf.pos_z),
           N.ptr(reference_positions), N.ptr(out), N.stream())
    return bool(out.item() >= (0.5 * skin) ** 2)


def max_particles_per_cell(buf: ParticleBuffer, box, cell_size: float) -> int:
    """Peak owned-particle occupancy on a reference grid (containers.py:41-53)."""
    box = as_box(box)
    dims = np.maximum((box.lengths / cell_size).astype(np.int64), 1)
    own = buf.ownership
    owned = own == OWNED
    if not bool(owned.any()):
        return 0
    idx = []
    for axis, pos in enumerate((buf.pos_x, buf.pos_y, buf.pos_z)):
        scaled = (pos[owned] - float(box.min[axis])) / float(box.lengths[axis] / dims[axis])
        idx.append(torch.clamp(scaled.to(torch.int64), 0, int(dims[axis]) - 1))
    lin = idx[0] + int(dims[0]) * (idx[1] + int(dims[1]) * idx[2])
    return int(torch.bincount(lin).max().item())


def _grid(box: SimulationBox, length: float) -> N.Grid:
    g = N.Grid()
    b = N.make_box(box)
    status = N.load().lmd_grid_init(C.byref(b), float(length), C.byref(g))
    if status == N.ERR_DEGENERATE:
        raise DegenerateDomainError(
            f"box {box.lengths} smaller than cutoff+skin {length} on some axis")
    if status:
        raise ConfigurationError(f"cell grid for box {box.lengths} / {length} is too large")
    return g


class _Sorter:
    """Reusable scratch for binning n particles (CUB temp sized once)."""

    def __init__(self, device):
        self.device = device
        self.cap = -1
        self.temp = None
        self.temp_bytes = 0

    def ensure(self, n: int):
        if n > self.cap:
            cap = max(n, 1)
            self.temp_bytes = int(N.load().lmd_sort_temp_bytes(cap))
            self.temp = torch.empty(max(self.temp_bytes, 1), dtype=torch.uint8, device=self.device)
            self.cell = torch.empty(cap, dtype=torch.int32, device=self.device)
            self.cell_sorted = torch.empty(cap, dtype=torch.int32, device=self.device)
            self.iota = torch.empty(cap, dtype=torch.int32, device=self.device)
            self.cap = cap

    def bin(self, grid: N.Grid, ring: int, x, y, z, base: int, start, count):
        n = x.shape[0]
        self.ensure(n)
        perm = torch.empty(n, dtype=torch.int32, device=self.device)
        s = N.stream()
        N.call("lmd_cell_index", grid, ring, n, N.ptr(x), N.ptr(y), N.ptr(z), N.ptr(self.cell), s)
        N.call("lmd_sort_by_cell", n, grid.ncell, N.ptr(self.cell), N.ptr(self.cell_sorted),
               N.ptr(perm), N.ptr(self.iota), N.ptr(self.temp), self.temp_bytes, s)
        N.call("lmd_cell_ranges", n, grid.ncell, base, N.ptr(self.cell_sorted), N.ptr(start),
               N.ptr(count), s)
        return perm


def device_soa(buf, device=None) -> ParticleBuffer:
    """The caller's buffer on the device (zero-copy for our CUDA buffers)."""
    if isinstance(buf, ParticleBuffer) and buf.device.type == "cuda":
        return buf
    if device is None:
        if not torch.cuda.is_available():
            raise N.NativeLibraryError("the B200 force path needs a CUDA device")
        device = torch.device("cuda")
    # the force path reads positions and ownership only (H2D 25 B / particle)
    return ParticleBuffer.from_host(buf, device=device,
                                    fields=("pos_x", "pos_y", "pos_z", "ownership"))


def _check_all_owned(buf: ParticleBuffer) -> None:
    if len(buf) and bool((buf.ownership != OWNED).any()):
        raise ConfigurationError(
            "device containers take an all-OWNED particle buffer (halo images are derived)")


class LinkedCellsContainer:
    """Uniform cell grid with a one-cell halo ring (containers.py:61-198), on the GPU."""

    kind = "lc"

    def __init__(self, box, params, rebuild_period: int = REBUILD_PERIOD_DEFAULT, device=None):
        self.box = as_box(box)
        self.params = params
        self.rebuild_period = rebuild_period
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu"))
        length = params.interaction_length
        self.grid = _grid(self.box, length)
        g = self.grid
        self.dims = np.array(list(g.dims), dtype=np.int64)
        self.cell_length = np.array(list(g.cell_len), dtype=np.float64)
        self.total_dims = self.dims + 2
        self._n_total = int(g.ncell)
        self.reference_positions = None
        self.steps_since_rebuild = 0
        self.structure_version = 0
        self.n_owned = 0
        self.n_halo = 0
        self._perm = None
        self._sorter = None
        self._stats_cache: dict = {}
        self._tables_ready = False
        # Newton3 on lc_c08/lc_c18: "colored" dual-write passes, or "full_shell"
        # Newton3 on lc_c08/lc_c18: "full_shell" evaluates every pair from both
        # sides with the reference's Newton3 pair bookkeeping; "colored" runs
        # the dual-write color passes.  Both are deterministic; the full shell
        # measured 2-3.5x faster at 1M particles and 6-20x at 8,000
        # (tools/n3_modes.py).
        self.n3_mode = "full_shell"
        # thread per particle over consecutive cell-sorted particles
        # (lmd_force_lc_particles) for the orders with a >= 16 distinct i per
        # fill -- N x 1: 1.83 -> 0.78 ms, N/2 x 2: 1.08 -> 0.89 ms at 1M; the
        # 1 x N and 2 x N/2 orders stay warp per cell (lmd_force_lc), where a
        # warp per one or two particles is 2x slower.  False: warp per cell
        self.thread_per_particle = True
        self._max_cell = 1

    # ------------------------------------------------------------ geometry
    def linear_index(self, coords: np.ndarray) -> np.ndarray:
        tx, ty, _ = self.total_dims
        return coords[..., 0] + tx * (coords[..., 1] + ty * coords[..., 2])

    def cell_coords(self, buf, clip_ring: bool) -> np.ndarray:
        """Ring-padded cell coordinates per entry (containers.py:104-115), via K1."""
        d = device_soa(buf, self.device if self.device.type == "cuda" else None)
        n = len(d)
        cell = torch.empty(n, dtype=torch.int32, device=d.device)
        if n:
            N.call("lmd_cell_index", self.grid, int(clip_ring), n, N.ptr(d.pos_x),
                   N.ptr(d.pos_y), N.ptr(d.pos_z), N.ptr(cell), N.stream())
        lin = cell.cpu().numpy().astype(np.int64)
        tx, ty, _ = self.total_dims
        return np.stack([lin % tx, (lin // tx) % ty, lin // (tx * ty)], axis=1)

    def cell_index(self, buf, clip_ring: bool = False) -> torch.Tensor:
        d = device_soa(buf)
        cell = torch.empty(len(d), dtype=torch.int32, device=d.device)
        if len(d):
            N.call("lmd_cell_index", self.grid, int(clip_ring), len(d), N.ptr(d.pos_x),
                   N.ptr(d.pos_y), N.ptr(d.pos_z), N.ptr(cell), N.stream())
        return cell

    # ------------------------------------------------------------ protocol
    def needs_rebuild(self, owned) -> bool:
        d = device_soa(owned)
        return needs_rebuild_buffer(d, self.reference_positions, self.params.skin,
                             self.steps_since_rebuild, self.rebuild_period)

    def _alloc_tables(self, dev):
        nc = self._n_total
        self._o_start = torch.empty(nc, dtype=torch.int32, device=dev)
        self._o_count = torch.empty(nc, dtype=torch.int32, device=dev)
        self._h_start = torch.zeros(nc, dtype=torch.int32, device=dev)
        self._h_count = torch.zeros(nc, dtype=torch.int32, device=dev)
        self._start = torch.empty(nc, dtype=torch.int32, device=dev)
        self._count = torch.empty(nc, dtype=torch.int32, device=dev)
        self._dup = torch.zeros(nc, dtype=torch.uint8, device=dev)

    def rebuild(self, owned, halo=None) -> None:
        """``halo`` is accepted for protocol uniformity; images enter at refresh."""
        d = device_soa(owned)
        dev = d.device
        if self._sorter is None or self._sorter.device != dev:
            self._sorter = _Sorter(dev)
            self._alloc_tables(dev)
        n = len(d)
        self.n_owned = n
        self._perm = self._sorter.bin(self.grid, 0, d.pos_x, d.pos_y, d.pos_z, 0,
                                      self._o_start, self._o_count)
        self._cell_of = self._sorter.cell_sorted[:n].clone()   # rebuild-time cell per slot
        if n:
            # one host read for the ownership check and the peak occupancy
            bad, peak = torch.stack([(d.ownership != OWNED).any().to(torch.int32),
                                     self._o_count.max()]).tolist()
            if bad:
                raise ConfigurationError(
                    "device containers take an all-OWNED particle buffer (halo images are "
                    "derived)")
            self._max_cell = max(1, int(peak))
        else:
            self._max_cell = 1
        self.reference_positions = d.positions().clone()
        self.steps_since_rebuild = 0
        self.structure_version += 1
        self._stats_cache.clear()
        self._tables_ready = False

    def refresh(self, owned, halo=None) -> None:
        """Reload positions, zero forces and re-bin the halo images (containers.py:141-172).

        ``halo=None`` derives the periodic images on the device (K9)."""
        d = device_soa(owned)
        if self._perm is None:
            raise ConfigurationError("container has not been rebuilt")
        if len(d) != self.n_owned:
            raise ConfigurationError("owned particle count changed without a rebuild")
        dev = d.device
        if halo is None:
            halo = build_halo(d, self.box, self.params.interaction_length)
        h = device_soa(halo, dev)
        nh = len(h)
        n = self.n_owned
        if nh or self.n_halo:
            self.structure_version += 1
            self._stats_cache.clear()
        self.n_halo = nh
        self._pos4 = torch.empty((n + nh, 4), dtype=torch.float64, device=dev)
        self._fx = torch.zeros(n + nh, dtype=torch.float64, device=dev)
        self._fy = torch.zeros(n + nh, dtype=torch.float64, device=dev)
        self._fz = torch.zeros(n + nh, dtype=torch.float64, device=dev)
        s = N.stream()
        if n:
            N.call("lmd_gather_pos4", n, N.ptr(self._perm), N.ptr(d.pos_x), N.ptr(d.pos_y),
                   N.ptr(d.pos_z), None, float(OWNED), N.ptr(self._pos4), s)
        if nh:
            hperm = self._sorter.bin(self.grid, 1, h.pos_x, h.pos_y, h.pos_z, n,
                                     self._h_start, self._h_count)
            N.call("lmd_gather_pos4", nh, N.ptr(hperm), N.ptr(h.pos_x), N.ptr(h.pos_y),
                   N.ptr(h.pos_z), None, float(HALO), N.ptr(self._pos4[n:]), s)
            owner = h.extra.get("owner")
            shift = h.extra.get("shift")
            hp = hperm.long()
            self._halo_owner = owner[hp].contiguous() if owner is not None else None
            self._halo_shift = shift[hp].contiguous() if shift is not None else None
            self._halo_ids = h.id[hp]
        else:
            self._h_start.zero_()
            self._h_count.zero_()
            self._halo_owner = None
            self._halo_shift = None
            self._halo_ids = torch.zeros(0, dtype=torch.int64, device=dev)
        N.call("lmd_merge_cell_tables", self._n_total, N.ptr(self._o_start), N.ptr(self._o_count),
               N.ptr(self._h_start), N.ptr(self._h_count), N.ptr(self._start), N.ptr(self._count),
               N.ptr(self._dup), s)
        self._tables_ready = True

    def refresh_positions(self, owned) -> None:
        """Between rebuilds: reload owned positions into their rebuild-time cells
        and move the images with their owners (no re-binning, no host sync)."""
        d = device_soa(owned)
        n, nh = self.n_owned, self.n_halo
        s = N.stream()
        N.call("lmd_gather_pos4", n, N.ptr(self._perm), N.ptr(d.pos_x), N.ptr(d.pos_y),
               N.ptr(d.pos_z), None, float(OWNED), N.ptr(self._pos4), s)
        if nh:
            if self._halo_owner is None:
                raise ConfigurationError("halo images were supplied without owner indices")
            N.call("lmd_halo_refresh_pos4", N.make_box(self.box), nh, N.ptr(self._halo_owner),
                   N.ptr(self._halo_shift), N.ptr(d.pos_x), N.ptr(d.pos_y), N.ptr(d.pos_z),
                   N.ptr(self._pos4[n:]), s)

    def kernel_backings(self) -> tuple[ParticleBuffer, ParticleBuffer]:
        """(owned-side, halo-side) backings in sorted order (device views)."""
        n = self.n_owned
        return self._backing_view(0, n), self._backing_view(n, n + self.n_halo)

    def _backing_view(self, a: int, b: int) -> ParticleBuffer:
        p = self._pos4[a:b]
        m = b - a
        dev = self._pos4.device
        z = torch.zeros(m, dtype=torch.float64, device=dev)
        n = self.n_owned
        ids = self._halo_ids[a - n:b - n] if a >= n else self._perm[a:b].long()
        return ParticleBuffer(pos_x=p[:, 0], pos_y=p[:, 1], pos_z=p[:, 2], vel_x=z, vel_y=z,
                              vel_z=z, force_x=self._fx[a:b], force_y=self._fy[a:b],
                              force_z=self._fz[a:b], old_force_x=z, old_force_y=z, old_force_z=z,
                              id=ids, ownership=p[:, 3].to(torch.int8))

    def collect_forces(self, owned) -> None:
        """Scatter sorted forces back to the caller's order (containers.py:186-189)."""
        d = device_soa(owned)
        n = self.n_owned
        if n:
            N.call("lmd_scatter_forces", n, N.ptr(self._perm), N.ptr(self._fx), N.ptr(self._fy),
                   N.ptr(self._fz), N.ptr(d.force_x), N.ptr(d.force_y), N.ptr(d.force_z),
                   N.stream())
        if d is not owned:
            for name in ("force_x", "force_y", "force_z"):
                dst = getattr(owned, name)
                val = getattr(d, name)
                if isinstance(dst, torch.Tensor):
                    dst.copy_(val)   # direct device -> (pinned) host DMA
                else:
                    torch.from_numpy(dst).copy_(val)

    # --------------------------------------------------------------- views
    @property
    def occupancy(self) -> np.ndarray:
        oc = self._o_count.cpu().numpy()
        hc = self._h_count.cpu().numpy()
        occ = np.zeros(self._n_total, dtype=np.uint8)
        occ[hc > 0] = 2
        occ[oc > 0] = 1
        return occ

    @property
    def owned_occupied(self) -> np.ndarray:
        return np.nonzero(self._o_count.cpu().numpy())[0].astype(np.int64)

    @property
    def halo_occupied(self) -> np.ndarray:
        return np.nonzero(self._h_count.cpu().numpy())[0].astype(np.int64)

    def buffer_at(self, linear: int) -> ParticleBuffer:
        oc = int(self._o_count[linear])
        if oc:
            s = int(self._o_start[linear])
            v = self._backing_view(s, s + oc)
        else:
            hc = int(self._h_count[linear])
            if hc == 0:
                raise KeyError(f"cell {linear} is empty")
            s = int(self._h_start[linear])
            v = self._backing_view(s, s + hc)
        v.backing_slot = (0 if oc else 1, s - (0 if oc else self.n_owned), len(v))
        return v

    # ---------------------------------------------------------------- force
    def _lc_stats(self, traversal: int, newton3: bool, pattern: PatternKind, V: int):
        key = (self.structure_version, traversal, bool(newton3), pattern, V)
        hit = self._stats_cache.get(key)
        if hit is not None:
            return hit
        a, b = pattern.shape(V)
        t = N.new_stats(self._pos4.device)
        N.call("lmd_lc_stats", self.grid, traversal, int(newton3), a, b, V, N.ptr(self._o_count),
               N.ptr(self._h_count), N.ptr(t), N.stream())
        st = N.read_stats(t)
        hit = (int(st.kernel_invocations), int(st.lane_slots), int(st.useful_interactions))
        self._stats_cache[key] = hit
        return hit

    def _uses_tpi(self, pattern) -> bool:
        return bool(self.thread_per_particle) and pattern.shape(32)[0] >= 16

    def gpu_lane_stats(self, pattern, traversal=N.LC_C01, newton3: bool = False):
        """Physical lane use of the kernel that executes this configuration
        (the GPU analogue of the reference's lane statistics):
        (lane_steps, active_lanes) = 32 x warp fill steps executed, and the
        lanes of those steps holding a real (i, j) candidate.  Exact by
        construction: warp per cell sweeps ceil(nC/A) x ceil(nD/B) fills per
        occupied (C, D) at width 32 -- the reference's c01 formula at V = 32;
        thread per particle runs, per warp of a consecutive particles and per
        neighbour offset, ceil(n/b) steps for the largest neighbour cell n of
        those particles.  Colored Newton3 passes are not covered."""
        pattern = as_pattern(pattern)
        if self.uses_colored_n3(traversal, newton3):
            raise ConfigurationError("lane statistics cover the full-shell kernels")
        _, _, useful = self._lc_stats(N.LC_C01, False, pattern, 32)
        if self._uses_tpi(pattern):
            n = self.n_owned
            a, b = pattern.shape(32)
            t0, t1 = int(self.total_dims[0]), int(self.total_dims[1])
            offs = torch.tensor([(d // 9 - 1) + t0 * ((d // 3) % 3 - 1 + t1 * (d % 3 - 1))
                                 for d in range(27)], dtype=torch.int64, device=self._pos4.device)
            cells = self._cell_of.long()
            pad = (-n) % a
            per = (self._count.long()[cells[:, None] + offs[None, :]] + b - 1) // b  # (n, 27)
            if pad:
                per = torch.cat([per, torch.zeros((pad, 27), dtype=per.dtype, device=per.device)])
            steps = int(per.view(-1, a, 27).amax(dim=1).sum().item())
            return 32 * steps, useful
        _, slots, _ = self._lc_stats(N.LC_C01, False, pattern, 32)
        return slots, useful

    def uses_colored_n3(self, traversal, newton3: bool) -> bool:
        return bool(newton3) and traversal in (N.LC_C08, N.LC_C18) and self.n3_mode == "colored"

    def launch_force(self, pattern, energy: bool = False, stats_t=None, ev_t=None,
                     traversal=N.LC_C01, newton3: bool = False):
        """Launch the force phase on the current stream without synchronising;
        returns the device stats tensor (pair counts, overlap flag, energy).

        Newton3 on lc_c08 / lc_c18 runs, with n3_mode="colored", the colored
        dual-write traversal (lmd_force_lc_n3: one launch per color,
        deterministic); otherwise the 27-cell full shell (lmd_force_lc).  Both weight cells that hold owned
        particles and images the way the reference's duplicated anchor units
        do (traversals.py:133)."""
        if not self._tables_ready:
            raise ConfigurationError("container has not been refreshed")
        pattern = as_pattern(pattern)
        dev = self._pos4.device
        if stats_t is None:
            stats_t = N.new_stats(dev)
        else:
            stats_t.zero_()
        if self.uses_colored_n3(traversal, newton3):
            if ev_t is None or ev_t.numel() < 2 * int(N.load().lmd_lc_n3_ev_slots(self.grid)):
                slots = int(N.load().lmd_lc_n3_ev_slots(self.grid))
                ev_t = torch.empty(2 * slots, dtype=torch.float64, device=dev)
            N.call("lmd_force_lc_n3", self.grid, N.make_lj(self.params), traversal, pattern.code,
                   N.FLAG_ENERGY if energy else 0, N.ptr(self._pos4), self.n_owned,
                   N.ptr(self._start), N.ptr(self._count), N.ptr(self._o_count),
                   N.ptr(self._h_count), N.ptr(self._dup), self._max_cell, N.ptr(self._fx),
                   N.ptr(self._fy), N.ptr(self._fz), N.ptr(ev_t), N.ptr(stats_t), N.stream())
            return stats_t
        dup = None if traversal == N.LC_C01 else N.ptr(self._dup)
        if self._uses_tpi(pattern):
            slots = int(N.load().lmd_lc_tpi_ev_slots(self.n_owned, pattern.code))
            if ev_t is None or ev_t.numel() < 2 * slots:
                ev_t = torch.empty(2 * max(slots, 1), dtype=torch.float64, device=dev)
            N.call("lmd_force_lc_particles", self.grid, N.make_lj(self.params), pattern.code,
                   N.FLAG_ENERGY if energy else 0, N.ptr(self._pos4), self.n_owned,
                   N.ptr(self._cell_of), N.ptr(self._start), N.ptr(self._count), dup,
                   N.ptr(self._fx), N.ptr(self._fy), N.ptr(self._fz), N.ptr(ev_t),
                   N.ptr(stats_t), N.stream())
            return stats_t
        if ev_t is None:
            slots = int(N.load().lmd_lc_ev_slots(self.grid))
            ev_t = torch.empty(2 * slots, dtype=torch.float64, device=dev)
        N.call("lmd_force_lc", self.grid, N.make_lj(self.params), pattern.code,
               N.FLAG_ENERGY if energy else 0, N.ptr(self._pos4), N.ptr(self._start),
               N.ptr(self._count), dup, N.ptr(self._fx), N.ptr(self._fy), N.ptr(self._fz),
               N.ptr(ev_t), N.ptr(stats_t), N.stream())
        return stats_t

    def compute_forces(self, traversal, newton3: bool, pattern, vector_width: int,
                       energy: bool = False) -> KernelStats:
        """Execute one force phase over the current structure; forces are
        written into the sorted backing (collect_forces scatters them)."""
        from .traversals import traversal_code
        validate_vector_width(vector_width)
        pattern = as_pattern(pattern)
        code = traversal_code(traversal)
        if code not in (N.LC_C01, N.LC_C08, N.LC_C18):
            raise ConfigurationError(f"{traversal} traversal requires linked cells")
        if code == N.LC_C01 and newton3:
            raise ConfigurationError("lc_c01 cannot exploit Newton's third law")
        inv, slots, useful = self._lc_stats(code, newton3, pattern, vector_width)
        st = N.read_stats(self.launch_force(pattern, energy, traversal=code, newton3=newton3))
        once = self.uses_colored_n3(code, newton3)
        return self.finish_stats(st, newton3 and not once, inv, slots, useful)

    @staticmethod
    def finish_stats(st, newton3, inv, slots, useful) -> KernelStats:
        """KernelStats from a device stats record; ``newton3`` converts ordered
        full-shell pair counts to the reference's Newton3 convention."""
        from .errors import ParticleOverlapError
        if st.overlap:
            raise ParticleOverlapError("zero distance between interacting particles")
        pairs = int(st.pair_interactions)
        if newton3:
            oh = int(st.pairs_owned_halo)
            pairs = (pairs - oh) // 2 + oh
        return KernelStats(kernel_invocations=inv, lane_slots=slots, useful_interactions=useful,
                           pair_interactions=pairs, epot=st.epot, virial=st.virial)
