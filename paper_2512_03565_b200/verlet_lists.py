"""Verlet lists with a skin on the device (north-star extension; the reference
excludes them).

The container follows the reference's container protocol (driver.py:179-208):
``needs_rebuild`` (displacement >= skin/2 or the rebuild period),
``rebuild`` (bin + images + lists), ``refresh`` (between rebuilds: reload
positions into the rebuild-time order and move the images with their owners
-- no re-binning, no host synchronisation), ``collect_forces``.  Lists are
built by K3 on the rc+skin cell grid and laid out per interaction order
(see csrc/vl.cu); the force kernel K4 gathers 32-byte pos4 records.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as N
from .containers import _Sorter, _grid, device_soa, needs_rebuild_buffer
from .domain import as_box, build_halo
from .errors import ConfigurationError, ParticleOverlapError
from .kernels import KernelStats, as_pattern, validate_vector_width
from .particles import HALO, OWNED

VL_REBUILD_PERIOD_DEFAULT = 10   # BASELINE config 2: lists rebuilt every 10 steps
SENTINEL_POSITION = 1.0e30


class VerletListContainer:
    kind = "vl"

    def __init__(self, box, params, rebuild_period: int = VL_REBUILD_PERIOD_DEFAULT, device=None):
        self.box = as_box(box)
        self.params = params
        self.rebuild_period = rebuild_period
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu"))
        self.grid = _grid(self.box, params.interaction_length)
        g = self.grid
        self.dims = np.array(list(g.dims), dtype=np.int64)
        self.total_dims = self.dims + 2
        self.reference_positions = None
        self.steps_since_rebuild = 0
        self.structure_version = 0
        self.n_owned = 0
        self.n_halo = 0
        self._sorter = None
        self._lists: dict = {}
        self._counts: dict = {}
        self._stats_cache: dict = {}
        self._max_seen: dict = {}
        self.knobs = 0        # extra lmd_force_vl flags
        # gathers: SoA x, y, z (three 64-bit loads, rows 128-B aligned) in a
        # bank-conflict-aware entry order (bank_rounds: -1 off, 0 lane-local
        # Latin-square order, >= 1 warp-cooperative with that many proposal
        # rounds per step; csrc/vl.cu vl_bank_local_kernel / vl_bank_kernel)
        # use_soa=False: 256-bit pos4 records in ascending order
        self.use_soa = True
        # lane-local bank order on staged lists: force 196 -> 167 us at 1M for a
        # 0.27 ms pass per list build
        self.bank_rounds = 0
        # staged lists (v_by_one, full lists): groups of staged_group owned
        # particles copy their candidate runs into shared memory (TMA) and
        # gather there; groups needing more than staged_capacity rows gather
        # from global memory.  0 = off.
        self.staged_group = 128
        self._staging: dict = {}
        # staged lists with every group staged store 16-bit local rows
        self.index16 = True
        # Newton3: "full_list" runs the full lists with the reference's Newton3
        # pair bookkeeping (no atomics, deterministic); "half_list" runs half
        # lists with FP64 atomics on the j side
        self.n3_mode = "full_list"
        self._collected_into = None
        # segmented staged lists (csrc/vls.cu): the default for v_by_one full
        # lists (N3 off, or Newton3 by bookkeeping).  Entries whose build-time
        # distance is below rc + inner_skin form the inner segment, which
        # alone covers every pair while no particle moved inner_skin / 2 since
        # the build (decided on the device from the refresh's displacement)
        self.segmented = True
        self.inner_skin = 0.1
        # adaptive: when the last epoch ended with a displacement of at least
        # inner_skin (the outer segment ran for most of its steps), the next
        # lists are built as one segment (cheaper to run in full than two
        # padded segments); decided at each rebuild from the displacement
        # refresh_and_check last read
        self.adaptive_inner = True
        self._last_disp2 = None
        self._inner_eff = self.inner_skin
        # a container built for one force computation (driver.force_phase):
        # rebuild loads the (x, y, z) rows only -- no pos4 / SoA copies and no
        # snapshots of the build-time state (positions never change)
        self.one_shot = False
        self._vls: dict = {}
        self._vls_plan = None
        self._vls_cap = None
        self._vls_ev = None
        self._disp = None          # (2,) int64: bit patterns of max |dr|^2, per slot
        self._disp_slot = -1       # slot of the last fused refresh (-1: unknown)
        self._pos4_stale = False

    # ------------------------------------------------------------ protocol
    def needs_rebuild(self, owned) -> bool:
        d = device_soa(owned)
        return needs_rebuild_buffer(d, self.reference_positions, self.params.skin,
                             self.steps_since_rebuild, self.rebuild_period)

    def rebuild(self, owned, halo=None) -> None:
        """Bin the owned particles and their images and drop the lists.

        ``halo=None`` derives the periodic images on the device (K9).  A
        domain decomposition passes its ghost layer instead; later refreshes
        must then pass the ghosts again, in the same order."""
        d = device_soa(owned)
        # the all-OWNED check is read after the halo count's host sync
        not_owned = (d.ownership != OWNED).any() if len(d) else None
        dev = d.device
        nc = int(self.grid.ncell)
        if self._sorter is None or self._sorter.device != dev:
            self._sorter = _Sorter(dev)
            self._o_start = torch.empty(nc, dtype=torch.int32, device=dev)
            self._o_count = torch.empty(nc, dtype=torch.int32, device=dev)
            self._h_start = torch.zeros(nc, dtype=torch.int32, device=dev)
            self._h_count = torch.zeros(nc, dtype=torch.int32, device=dev)
            self._sentinel_row = torch.tensor([SENTINEL_POSITION] * 3 + [2.0],
                                              dtype=torch.float64, device=dev)
        n = len(d)
        self._perm = self._sorter.bin(self.grid, 0, d.pos_x, d.pos_y, d.pos_z, 0,
                                      self._o_start, self._o_count)
        self._external_halo = halo is not None
        if halo is None:
            halo = build_halo(d, self.box, self.params.interaction_length)
        else:
            halo = device_soa(halo, dev)
        if not_owned is not None and bool(not_owned):
            raise ConfigurationError(
                "device containers take an all-OWNED particle buffer (halo images are derived)")
        nh = len(halo)
        self.n_owned, self.n_halo = n, nh
        # combined backing [owned | images | sentinel] as pos4 (32 B records),
        # filled by _load_positions in the rebuild-time order
        self._pos4 = torch.empty((n + nh + 1, 4), dtype=torch.float64, device=dev)
        self._pos4[-1].copy_(self._sentinel_row)
        if nh:
            self._hperm = self._sorter.bin(self.grid, 1, halo.pos_x, halo.pos_y, halo.pos_z, n,
                                           self._h_start, self._h_count)
            if not self._external_halo:
                hp = self._hperm.long()
                self._halo_owner = halo.extra["owner"][hp].contiguous()
                self._halo_shift = halo.extra["shift"][hp].contiguous()
        else:
            self._h_start.zero_()
            self._h_count.zero_()
            self._halo_owner = torch.zeros(0, dtype=torch.int32, device=dev)
            self._halo_shift = torch.zeros(0, dtype=torch.int8, device=dev)
        if self.use_soa:
            self._soa = self._new_soa(n + nh + 1, dev)
        else:
            self._soa = torch.empty((3, 1), dtype=torch.float64, device=dev)
        # (x, y, z) rows for the segmented lists (+2 rows: staged runs are
        # rounded to even lengths)
        self._rows = (torch.zeros((n + nh + 2, 3), dtype=torch.float64, device=dev)
                      if self.segmented else None)
        # every owned slot is written by the force kernel (Newton3 zeroes first)
        self._fx = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        self._fy = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        self._fz = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        # Lists are built lazily per interaction order, always from the
        # rebuild-time positions, whatever the particles did since.  With the
        # segmented lists only the (x, y, z) rows are loaded and snapshot here;
        # the pos4 / SoA copies (the other orders' kernels) follow on demand
        # (_list).  A one-shot container (positions never change) aliases the
        # snapshot.
        lean = self.one_shot and self.segmented
        if self.segmented:
            self._load_rows(d, halo if self._external_halo else None)
            self._build_pos4 = None
            self._build_rows = self._rows if lean else self._rows.clone()
        else:
            self._load_positions(d, halo if self._external_halo else None)
            self._build_pos4 = self._pos4.clone()
            self._build_rows = None
        self._vls.clear()
        self._vls_plan = None
        one_segment = (self.adaptive_inner and self._last_disp2 is not None
                       and self._last_disp2 >= float(self.inner_skin) ** 2)
        self._inner_eff = float(self.params.skin) if one_segment else float(self.inner_skin)
        self._last_disp2 = None
        if self._disp is None or self._disp.device != dev:
            self._disp = torch.zeros(2, dtype=torch.int64, device=dev)
        else:
            self._disp.zero_()
        self._disp_slot = 0
        self._pos4_stale = bool(self.segmented)
        self._lists.clear()
        self._staging.clear()
        self._counts.clear()
        self._stats_cache.clear()
        self.reference_positions = d.positions()     # (a fresh (n, 3) stack)
        self.steps_since_rebuild = 0
        self.structure_version += 1

    def _need_pos4(self) -> bool:
        """Whether a kernel reading the pos4 records may run on these lists
        (the segmented kernels read the SoA rows only)."""
        return not self.segmented or any(k not in self._vls for k in self._lists)

    def _regen_pos4(self) -> None:
        """pos4 and the SoA copies from the current rows (after refreshes
        that only wrote the rows)."""
        n, nh = self.n_owned, self.n_halo
        soa = self.use_soa and self._soa.shape[1] >= n + nh + 1
        N.call("lmd_vls_rows_to_legacy", n + nh, n, N.ptr(self._rows), N.ptr(self._pos4),
               N.ptr(self._soa[0]) if soa else None, N.ptr(self._soa[1]) if soa else None,
               N.ptr(self._soa[2]) if soa else None, N.stream())
        self._pos4_stale = False

    def _load_rows(self, d, ghosts=None, ghost_rows=None, disp: bool = False,
                   which: str = "all") -> None:
        """Current positions into the (x, y, z) rows of the segmented lists;
        with ``disp`` the owned gather also reduces the largest displacement
        since the build into the next displacement slot (on the device)."""
        n, nh = self.n_owned, self.n_halo
        s = N.stream()
        rows = self._rows
        track = disp and self._build_rows is not None
        if n and which != "ghosts":
            dp = None
            slot = 0
            if track:
                slot = 0 if self._disp_slot < 0 else self._disp_slot ^ 1
                dp = self._disp
            # derived periodic images move with their owners in the same launch
            with_images = (which == "all" and nh > 0 and ghost_rows is None and ghosts is None
                           and not self._external_halo)
            N.call("lmd_vls_refresh", n, N.ptr(self._perm), N.ptr(d.pos_x), N.ptr(d.pos_y),
                   N.ptr(d.pos_z), N.ptr(rows), N.ptr(self._build_rows) if dp is not None else None,
                   N.ptr(dp), slot, N.make_box(self.box) if with_images else None,
                   nh if with_images else 0,
                   N.ptr(self._halo_owner) if with_images else None,
                   N.ptr(self._halo_shift) if with_images else None, s)
            if disp:
                self._disp_slot = slot if dp is not None else -1
            if with_images:
                return
        if not nh or which == "owned":
            return
        # an external ghost layer: the ghosts' displacements join the same
        # slot (they decide the inner segment's validity like the owned ones)
        gslot = self._disp_slot if track and self._disp_slot >= 0 else -1
        gdp = self._disp if gslot >= 0 else None
        gbuild = self._build_rows[n:] if gslot >= 0 else None
        if ghost_rows is not None:
            N.call("lmd_vls_gather_rows", nh, N.ptr(self._hperm), N.ptr(ghost_rows),
                   N.ptr(rows[n:]), N.ptr(gbuild), N.ptr(gdp), max(gslot, 0), s)
        elif ghosts is not None:
            N.call("lmd_vls_refresh", nh, N.ptr(self._hperm), N.ptr(ghosts.pos_x),
                   N.ptr(ghosts.pos_y), N.ptr(ghosts.pos_z), N.ptr(rows[n:]), N.ptr(gbuild),
                   N.ptr(gdp), max(gslot, 0), None, 0, None, None, s)
        else:
            N.call("lmd_halo_refresh_rows", N.make_box(self.box), nh, N.ptr(self._halo_owner),
                   N.ptr(self._halo_shift), N.ptr(d.pos_x), N.ptr(d.pos_y), N.ptr(d.pos_z),
                   N.ptr(rows[n:]), s)

    def _load_positions(self, d, ghosts=None, ghost_rows=None, fused: bool = False,
                        which: str = "all") -> None:
        """Current positions into pos4 and the SoA copies, in rebuild-time order:
        owned via the cell permutation; images either moved with their owners
        (shift codes) or, for an external ghost layer, gathered from it.
        ``fused`` (per-step refresh of segmented lists): the owned gather also
        reduces the largest displacement since the build on the device, and
        pos4 is written only when a kernel reading it may run."""
        n, nh = self.n_owned, self.n_halo
        s = N.stream()
        soa = self.use_soa
        if soa:
            if self._soa.shape[1] < n + nh + 1:   # SoA switched on after the rebuild
                self._soa = self._new_soa(n + nh + 1, self._pos4.device)
            sx, sy, sz = self._soa[0], self._soa[1], self._soa[2]
        if self.segmented and self._rows is not None:
            self._load_rows(d, ghosts, ghost_rows, disp=fused, which=which)
        write4 = not (fused and self.segmented) or self._need_pos4()
        if which != "all" and write4:
            raise ConfigurationError("split refreshes serve the segmented lists only")
        if not write4:
            self._pos4_stale = True
            return
        self._pos4_stale = False
        if n:
            if soa:
                N.call("lmd_gather_pos4_soa", n, N.ptr(self._perm), N.ptr(d.pos_x),
                       N.ptr(d.pos_y), N.ptr(d.pos_z), float(OWNED), N.ptr(self._pos4),
                       N.ptr(sx), N.ptr(sy), N.ptr(sz), s)
            else:
                N.call("lmd_gather_pos4", n, N.ptr(self._perm), N.ptr(d.pos_x), N.ptr(d.pos_y),
                       N.ptr(d.pos_z), None, float(OWNED), N.ptr(self._pos4), s)
        if not nh:
            return
        if ghost_rows is not None:
            if soa:
                N.call("lmd_gather_rows_soa", nh, N.ptr(self._hperm), N.ptr(ghost_rows),
                       N.ptr(sx[n:]), N.ptr(sy[n:]), N.ptr(sz[n:]), s)
            N.call("lmd_gather_pos4_rows", nh, N.ptr(self._hperm), N.ptr(ghost_rows), float(HALO),
                   N.ptr(self._pos4[n:]), s)
            return
        if ghosts is not None:
            if soa:
                N.call("lmd_gather_soa", nh, N.ptr(self._hperm), N.ptr(ghosts.pos_x),
                       N.ptr(ghosts.pos_y), N.ptr(ghosts.pos_z), N.ptr(sx[n:]), N.ptr(sy[n:]),
                       N.ptr(sz[n:]), s)
            N.call("lmd_gather_pos4", nh, N.ptr(self._hperm), N.ptr(ghosts.pos_x),
                   N.ptr(ghosts.pos_y), N.ptr(ghosts.pos_z), None, float(HALO),
                   N.ptr(self._pos4[n:]), s)
            return
        box = N.make_box(self.box)
        if soa:
            N.call("lmd_halo_refresh_pos4_soa", box, nh, N.ptr(self._halo_owner),
                   N.ptr(self._halo_shift), N.ptr(d.pos_x), N.ptr(d.pos_y), N.ptr(d.pos_z),
                   N.ptr(self._pos4[n:]), N.ptr(sx[n:]), N.ptr(sy[n:]), N.ptr(sz[n:]), s)
            return
        N.call("lmd_halo_refresh_pos4", box, nh, N.ptr(self._halo_owner), N.ptr(self._halo_shift),
               N.ptr(d.pos_x), N.ptr(d.pos_y), N.ptr(d.pos_z), N.ptr(self._pos4[n:]), s)

    @staticmethod
    def _new_soa(rows: int, dev) -> torch.Tensor:
        """(3, stride) x, y, z rows over the combined backing + sentinel; the
        stride is a multiple of 16 doubles so every row starts on 128 B and
        x[j], y[j], z[j] fall in the same bank pair j & 15 (the bank-aware
        list order relies on it)."""
        stride = (rows + 15) // 16 * 16
        t = torch.empty((3, stride), dtype=torch.float64, device=dev)
        t[:, rows - 1:] = SENTINEL_POSITION
        assert t.data_ptr() % 128 == 0
        return t

    def refresh(self, owned, halo=None) -> None:
        """Reload current positions (rebuild-time order) and move the images
        with their owners; ``halo`` is accepted for protocol compatibility --
        images are derived from the rebuild-time set, which covers every pair
        within the cutoff while displacements stay below skin/2."""
        if self.reference_positions is None:
            raise ConfigurationError("container has not been rebuilt")
        if self._external_halo:
            if halo is None or len(halo) != self.n_halo:
                raise ConfigurationError("refresh needs the same ghost layer as the rebuild")
            if isinstance(halo, torch.Tensor):    # row-major (n_halo, 3) ghost positions
                self._load_positions(device_soa(owned), None, ghost_rows=halo, fused=True)
                return
            self._load_positions(device_soa(owned), device_soa(halo, self._pos4.device),
                                 fused=True)
            return
        self._load_positions(device_soa(owned), fused=True)

    refresh_positions = refresh

    def refresh_and_check(self, owned) -> bool:
        """``needs_rebuild`` and ``refresh`` in one pass for the MD loop: True
        when the period elapsed or a particle moved skin / 2 since the rebuild
        (the caller rebuilds); otherwise the container has been refreshed.
        The displacement is the one the refresh kernel reduces on the device
        while it gathers the rows (the same unfused expression as
        ``lmd_max_displacement2``), so no separate pass over the positions
        runs; one 8-byte read decides."""
        if (self.reference_positions is None or self._external_halo or self._rows is None
                or self._build_rows is None or self.params.skin <= 0.0
                or len(owned) != self.n_owned):
            if self.needs_rebuild(owned):
                return True
            self.refresh(owned)
            return False
        if self.steps_since_rebuild >= self.rebuild_period:
            if self._disp_slot >= 0:   # the epoch's last displacement, for the next lists
                self._last_disp2 = self._disp[self._disp_slot:self._disp_slot + 1].view(
                    torch.float64).item()
            return True
        self.refresh(owned)
        d2 = self._disp[self._disp_slot:self._disp_slot + 1].view(torch.float64).item()
        self._last_disp2 = d2
        return bool(d2 >= (0.5 * self.params.skin) ** 2)

    def refresh_owned(self, owned) -> None:
        """First half of an overlapped refresh with an external ghost layer:
        the owned rows only (the interior groups can run on them)."""
        self._load_positions(device_soa(owned), None, None, fused=True, which="owned")

    def refresh_ghosts(self, owned, ghost_rows) -> None:
        """Second half: the exchanged ghost rows (n_halo, 3)."""
        if ghost_rows is None or len(ghost_rows) != self.n_halo:
            raise ConfigurationError("refresh needs the same ghost layer as the rebuild")
        self._load_positions(device_soa(owned), None, ghost_rows, fused=True, which="ghosts")

    # ----------------------------------------------------------------- lists
    def _count(self, newton3: bool, pattern=None) -> torch.Tensor:
        """Per-particle list lengths (written by the first list build); with
        Newton3 in "full_list" mode, the half-list lengths that the full-list
        build records alongside."""
        key = bool(newton3)
        c = self._counts.get(key)
        if c is None:
            self._list(pattern or as_pattern("v_by_one"), self._list_n3(newton3))
            c = self._counts[key]
        return c

    def _list_n3(self, newton3: bool) -> bool:
        """Whether the lists used for this Newton3 setting are half lists."""
        return bool(newton3) and self.n3_mode == "half_list"

    def _kernel_n3(self, newton3: bool) -> int:
        """lmd_force_vl's newton3 mode: 0 full, 1 half + atomics, 2 full + bookkeeping."""
        if not newton3:
            return 0
        return 1 if self.n3_mode == "half_list" else 2

    def _capacity_guess(self, newton3: bool) -> int:
        """Entries per particle to reserve: the last build's longest list
        (+25 %), else twice the mean-density estimate."""
        seen = self._max_seen.get(bool(newton3))
        if seen is not None:
            return int(seen * 1.25) + 8
        rl = self.params.interaction_length
        vol = float(np.prod(self.box.lengths))
        est = (self.n_owned + self.n_halo) / vol * (4.0 / 3.0) * np.pi * rl ** 3
        if newton3:
            est *= 0.5
        return int(2.0 * est) + 32

    def _bank_for(self) -> int:
        return int(self.bank_rounds) if self.use_soa else -1

    def _staged_for(self, pattern, newton3_list: bool) -> int:
        """Group size of the staged layout for these lists (0: not staged)."""
        if (self.staged_group and self.use_soa and not newton3_list
                and pattern.code == as_pattern("v_by_one").code):
            return int(self.staged_group)
        return 0

    def _list(self, pattern, newton3: bool, bank: int | None = None):
        bank = self._bank_for() if bank is None else bank
        staged = self._staged_for(pattern, bool(newton3))
        key = (pattern.code, bool(newton3), bank, staged)
        hit = self._lists.get(key)
        if hit is not None:
            return hit
        n = self.n_owned
        dev = self._pos4.device
        if staged and n and self.segmented:
            hit = self._vls_lists(key)
            if hit is not None:
                self._lists[key] = hit
                return hit
        if self._build_pos4 is None:
            # first list of another order since the rebuild: pos4 / SoA of the
            # build-time rows
            N.call("lmd_vls_rows_to_legacy", n + self.n_halo, n, N.ptr(self._build_rows),
                   N.ptr(self._pos4), None, None, None, N.stream())
            self._build_pos4 = self._pos4.clone()
            self._pos4_stale = True
        ntiles = int(N.load().lmd_vl_num_tiles(n, pattern.code))
        b_ = pattern.shape(32)[1]
        tile_off = torch.empty(max(ntiles, 1), dtype=torch.int64, device=dev)
        kmax = torch.zeros(max(ntiles, 1), dtype=torch.int32, device=dev)
        count = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        # a full per-particle build also records the half-list lengths
        half = torch.zeros(max(n, 1), dtype=torch.int32, device=dev) if not newton3 else None
        mx = torch.zeros(1, dtype=torch.int32, device=dev)
        rl2 = self.params.interaction_length * self.params.interaction_length
        cap = self._capacity_guess(newton3)
        s = N.stream()
        tables = (N.ptr(self._build_pos4), N.ptr(self._o_start), N.ptr(self._o_count),
                  N.ptr(self._h_start), N.ptr(self._h_count))
        sentinel = self.n_owned + self.n_halo
        if staged and n:
            ngroups = (n + staged - 1) // staged
            groups = torch.empty(ngroups * 128, dtype=torch.int32, device=dev)
            smax = torch.zeros(2, dtype=torch.int32, device=dev)
            capacity = int(N.load().lmd_vl_staged_capacity(staged))
            N.call("lmd_vl_groups", self.grid, n, staged, capacity, *tables,
                   N.ptr(groups), N.ptr(smax), s)
            sentinel = -1
            # 16-bit local rows when every group is staged (one host read)
            sm = smax.tolist()
            bits = 16 if (sm[1] == 0 and self.index16) else 32
        else:
            bits = 32
        chunk = 8 if bits == 16 else 4
        while True:
            steps = (cap + b_ - 1) // b_
            cap_steps = max(chunk, (steps + chunk - 1) // chunk * chunk)
            words = ntiles * cap_steps * 32 * bits // 32
            nbr = torch.empty(max(words, 1), dtype=torch.int32, device=dev)
            if staged and n:
                N.call("lmd_vl_build_staged", self.grid, float(rl2), int(newton3), n, *tables,
                       staged, N.ptr(groups), bits, cap_steps, N.ptr(count),
                       N.ptr(half) if half is not None else None, N.ptr(tile_off),
                       N.ptr(kmax), N.ptr(mx), N.ptr(nbr), s)
            else:
                N.call("lmd_vl_build", self.grid, float(rl2), int(newton3), pattern.code, n,
                       sentinel, *tables, cap_steps, N.ptr(count),
                       N.ptr(half) if half is not None else None, N.ptr(tile_off),
                       N.ptr(kmax), N.ptr(mx), N.ptr(nbr), s)
            longest = int(mx.item()) if n else 0
            if longest <= cap_steps * b_:
                break
            del nbr
            cap = longest
        self._max_seen[bool(newton3)] = longest
        self._counts.setdefault(bool(newton3), count)
        if half is not None and self.n3_mode == "full_list":
            self._counts.setdefault(True, half)
        # lane-local order: 16-bit workspace, staged lists only
        if bank == 0 and not staged:
            bank = -1
        if bank > 0 and bits == 16:
            bank = 0    # the warp-cooperative order is 32-bit only
        if bank >= 0 and n:
            max_steps = min(cap_steps, ((longest + b_ - 1) // b_ + chunk - 1) // chunk * chunk)
            if bank > 0 or max_steps <= 255:
                N.call("lmd_vl_bank_schedule", pattern.code, n, sentinel, int(bank), cap_steps,
                       max_steps, bits, N.ptr(tile_off), N.ptr(kmax), N.ptr(nbr), s)
        if staged and n:
            rows = max(16, (int(sm[0]) + 15) // 16 * 16)
            self._staging[key] = (groups, rows, staged, int(sm[1]), bits)
        hit = (tile_off, kmax, nbr, ntiles * cap_steps * 32)
        self._lists[key] = hit
        return hit

    def _vls_plan_groups(self):
        """Row-aligned groups and their staged runs (one host read: the
        number of groups and the largest staging footprint)."""
        plan = self._vls_plan
        if plan is not None:
            return plan
        dev = self._pos4.device
        lib = N.load()
        g = self.grid
        ncell = int(g.ncell)
        nrows = int(g.tdims[1] * g.tdims[2])
        maxg = int(lib.lmd_vls_max_groups(g, self.n_owned))
        tb = int(lib.lmd_vls_plan_temp_bytes(g))
        plan = {
            "fs_own": torch.empty(ncell, dtype=torch.int32, device=dev),
            "fs_img": torch.empty(ncell, dtype=torch.int32, device=dev),
            "groups": torch.empty(maxg * 64, dtype=torch.int32, device=dev),
            "info": torch.zeros(8, dtype=torch.int32, device=dev),
            "maxg": maxg,
        }
        rg = torch.empty(nrows, dtype=torch.int32, device=dev)
        re = torch.empty(nrows, dtype=torch.int32, device=dev)
        temp = torch.empty(max(tb, 1), dtype=torch.uint8, device=dev)
        N.call("lmd_vls_plan", g, self.n_owned, N.ptr(self._o_start), N.ptr(self._o_count),
               N.ptr(self._h_start), N.ptr(self._h_count), N.ptr(plan["fs_own"]),
               N.ptr(plan["fs_img"]), N.ptr(rg), N.ptr(re), N.ptr(temp), tb, N.ptr(plan["groups"]),
               N.ptr(plan["info"]), N.stream())
        info = plan["info"].tolist()
        plan["rows"] = int(lib.lmd_vls_rows_for(info[0]))
        plan["ngroups"] = info[2]
        self._vls_plan = plan
        return plan

    def _vls_lists(self, key):
        """Segmented staged lists (csrc/vls.cu) for the v_by_one full lists;
        None when a group's staging footprint or a lane's list is too large
        for them (the other staged path then serves)."""
        if self._build_rows is None:
            return None
        plan = self._vls_plan_groups()
        if plan["rows"] == 0:
            return None
        dev = self._pos4.device
        lib = N.load()
        n = self.n_owned
        maxg = plan["maxg"]
        rl = float(self.params.interaction_length)
        rin = min(float(self.params.cutoff) + float(self._inner_eff), rl)
        cap = self._vls_cap
        if cap is None:
            vol = float(np.prod(self.box.lengths))
            est = (self.n_owned + self.n_halo) / vol * (4.0 / 3.0) * np.pi * rl ** 3
            cap = int(min(248, est * 1.5 + 16))
        info = plan["info"]
        s = N.stream()
        ng = plan["ngroups"]
        while True:
            cap = min(248, (cap + 7) // 8 * 8)   # 16-B aligned lane stretches
            cap_chunks = cap // 8 + 2
            nbr = torch.empty(ng * 4 * cap_chunks * 32 * 4, dtype=torch.int32, device=dev)
            segc = torch.empty(ng * 4 * 2, dtype=torch.int32, device=dev)
            slotmap = torch.empty(ng * 128, dtype=torch.uint8, device=dev)
            count = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
            half = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
            info[3:5].zero_()
            N.call("lmd_vls_build", self.grid, rin * rin, rl * rl, n, plan["rows"],
                   N.ptr(self._build_rows), N.ptr(plan["fs_own"]), N.ptr(self._o_count),
                   N.ptr(plan["fs_img"]), N.ptr(self._h_count), N.ptr(plan["groups"]), ng,
                   cap_chunks, cap, 1 if key[2] >= 0 else 0, N.ptr(nbr), N.ptr(segc),
                   N.ptr(slotmap), N.ptr(count), N.ptr(half), N.ptr(info), s)
            chunks_seen, ent_seen = info[3:5].tolist()
            if ent_seen <= cap and chunks_seen <= cap_chunks:
                break
            if ent_seen > 248:
                return None
            cap = ent_seen + 8
        self._vls_cap = min(248, int(ent_seen * 1.2) + 8)
        self._counts.setdefault(False, count)
        if self.n3_mode == "full_list":
            self._counts.setdefault(True, half)
        hit = {"nbr": nbr, "segc": segc, "slotmap": slotmap, "cap_chunks": cap_chunks,
               "plan": plan,
               "total": ng * 4 * cap_chunks * 32 * 8}
        self._vls[key] = hit
        return (None, None, nbr, hit["total"])

    def _vls_outer(self) -> bool:
        """Whether the next segmented launch runs the outer segment too (the
        device decides; this mirrors it for statistics)."""
        if self._disp_slot < 0:
            return True
        d = float(torch.tensor(self._disp[self._disp_slot].item(), dtype=torch.int64)
                  .view(torch.float64).item())
        return d >= self._vls_half_delta2()

    def _vls_half_delta2(self) -> float:
        # (delta / 2)^2 with a relative margin against rounding in the
        # displacement and distance evaluations
        return (0.5 * float(self._inner_eff) * (1.0 - 1e-9)) ** 2

    def gpu_lane_stats(self, pattern, newton3: bool = False):
        """(lane_steps, active_lanes) of the force kernel over the current
        lists: every tile runs kmax/B fill steps on 32 lanes; a lane is
        active when its entry is a real neighbour, not the sentinel pad
        (SURVEY §8f-4).  Exact by construction of the list layout."""
        pattern = as_pattern(pattern)
        tile_off, kmax, _, _ = self._list(pattern, self._list_n3(newton3))
        if tile_off is None:   # segmented lists: chunks of 8 steps per tile segment
            vls = self._vls_for(pattern, newton3)
            ng = vls["plan"]["ngroups"]
            segc = vls["segc"][: 8 * ng].view(-1, 2).long()
            steps = int(segc.sum().item()) * 8
            active = int(self._count(self._list_n3(newton3), pattern)[: self.n_owned].long()
                         .sum().item())
            return 32 * steps, active
        b = pattern.shape(32)[1]
        ntiles = int(N.load().lmd_vl_num_tiles(self.n_owned, pattern.code))
        steps = int((kmax[:ntiles].long() // b).sum().item())
        active = int(self._count(self._list_n3(newton3), pattern)[: self.n_owned].long()
                     .sum().item())
        return 32 * steps, active

    def _key(self, pattern, newton3: bool):
        n3l = self._list_n3(newton3)
        return (pattern.code, n3l, self._bank_for(), self._staged_for(pattern, n3l))

    def _vls_for(self, pattern, newton3: bool):
        return self._vls.get(self._key(as_pattern(pattern), newton3))

    def ensure_lists(self, pattern, newton3: bool) -> bool:
        """Build the lists for this interaction order now (outside any timed
        region); True if they had to be built."""
        pattern = as_pattern(pattern)
        if self._key(pattern, newton3) in self._lists:
            return False
        self._list(pattern, self._list_n3(newton3))
        self._count(newton3, pattern)
        return True

    def list_entries(self, pattern, newton3: bool) -> int:
        """List entries the force kernel reads for `pattern` (padded to whole
        fill steps and 4-step chunks; 4 B each)."""
        pattern = as_pattern(pattern)
        n3l = self._list_n3(newton3)
        tile_off, kmax, _, _ = self._list(pattern, n3l)
        if tile_off is None:
            return self.gpu_lane_stats(pattern, newton3)[0]
        b = pattern.shape(32)[1]
        return int((kmax.long() // b).sum().item()) * 32

    def pairs(self, newton3: bool = False):
        """(id_i, id_j, j_is_image) of every list entry, for exact set checks."""
        pattern = as_pattern("one_by_v")
        tile_off, kmax, nbr, total = self._list(pattern, newton3, bank=-1)
        count = self._count(newton3)[: self.n_owned].long()
        n = self.n_owned
        perm = self._perm.long()
        owner = self._halo_owner.long()
        # ONE_BY_V tiles hold one i each: entries are contiguous per i
        offs = tile_off[:n].long()
        i_idx = torch.repeat_interleave(torch.arange(n, device=count.device), count)
        first = torch.repeat_interleave(torch.cumsum(count, 0) - count, count)
        k = torch.arange(int(count.sum()), device=count.device) - first
        # ONE_BY_V: step s = k // 32 on lane k % 32, lane-chunked by 4 steps
        s_, lane = k // 32, k % 32
        j = nbr[offs[i_idx] + (s_ // 4) * 128 + lane * 4 + s_ % 4].long()
        is_img = j >= n
        jid = torch.empty_like(j)
        jid[~is_img] = perm[j[~is_img]]
        if bool(is_img.any()):
            jid[is_img] = owner[j[is_img] - n]   # owner indices are caller order
        return perm[i_idx], jid, is_img

    # ----------------------------------------------------------------- force
    def _vls_parts(self, plan):
        """Device index lists of the interior groups (no image / ghost rows
        staged: computable before a ghost exchange lands) and the others."""
        parts = plan.get("parts")
        if parts is None:
            ng = plan["ngroups"]
            rec = plan["groups"][: ng * 64].view(ng, 64)
            img_rows = rec[:, 26 + 9:26 + 18].sum(dim=1)   # lengths of the 9 image runs
            ids = torch.arange(ng, dtype=torch.int32, device=rec.device)
            parts = {"interior": ids[img_rows == 0].contiguous(),
                     "boundary": ids[img_rows != 0].contiguous()}
            plan["parts"] = parts
        return parts

    def reduce_ev(self, pattern, newton3: bool, stats_t, ev_t=None) -> None:
        """Energy / virial reduction after launches with ``defer_ev``."""
        vls = self._vls.get(self._key(as_pattern(pattern), newton3))
        N.call("lmd_vls_reduce_ev", vls["plan"]["ngroups"],
               N.ptr(ev_t if ev_t is not None else self._vls_ev), N.ptr(stats_t), N.stream())

    def launch_force(self, pattern, newton3: bool, energy: bool = False, stats_t=None,
                     ev_t=None, out=None, part: str | None = None, zero_stats: bool = True,
                     defer_ev: bool = False):
        """Launch the force kernel without synchronising; returns the device
        stats tensor.  ``out`` (a device ParticleBuffer of the rebuild's
        particles): write the forces straight into out.force_* in its order
        -- collect_forces fused into the kernel (full lists only); the next
        collect_forces(out) is then a no-op."""
        pattern = as_pattern(pattern)
        mode = self._kernel_n3(newton3)
        tile_off, kmax, nbr, _ = self._list(pattern, self._list_n3(newton3))
        dev = self._pos4.device
        if stats_t is None:
            stats_t = N.new_stats(dev)
        elif zero_stats:
            stats_t.zero_()
        if part is not None and self._vls.get(self._key(pattern, newton3)) is None:
            raise ConfigurationError("group subsets need the segmented lists")
        vls = self._vls.get(self._key(pattern, newton3))
        if vls is not None and mode != 1:
            plan = vls["plan"]
            if energy:
                slots = int(N.load().lmd_vls_ev_slots(plan["ngroups"]))
                if ev_t is None or ev_t.numel() < 2 * slots:
                    if self._vls_ev is None or self._vls_ev.numel() < 2 * slots:
                        self._vls_ev = torch.empty(2 * slots, dtype=torch.float64, device=dev)
                    ev_t = self._vls_ev
            direct = out is not None and len(out) == self.n_owned
            fx, fy, fz = ((out.force_x, out.force_y, out.force_z) if direct
                          else (self._fx, self._fy, self._fz))
            disp = None if self._disp_slot < 0 else self._disp[self._disp_slot:]
            gidx, nidx = None, 0
            if part is not None:
                gidx = self._vls_parts(plan)[part]
                nidx = int(gidx.numel())
                if nidx == 0:      # an empty part (a null index means "all groups")
                    self._collected_into = out if direct else None
                    return stats_t
            flags = (N.FLAG_ENERGY if energy else 0) | (N.FLAG_DEFER_EV if defer_ev else 0)
            N.call("lmd_vls_force", mode, flags,
                   N.make_lj(self.params), self.n_owned, plan["rows"], N.ptr(self._rows),
                   N.ptr(plan["groups"]), plan["ngroups"], N.ptr(gidx), nidx, N.ptr(vls["nbr"]),
                   N.ptr(vls["segc"]), N.ptr(vls["slotmap"]), vls["cap_chunks"], N.ptr(disp),
                   self._vls_half_delta2(), N.ptr(self._perm) if direct else None, N.ptr(fx),
                   N.ptr(fy), N.ptr(fz), N.ptr(ev_t) if energy else None, N.ptr(stats_t),
                   N.stream())
            self._collected_into = out if direct else None
            return stats_t
        if self._pos4_stale:
            self._regen_pos4()
        if ev_t is None:
            slots = int(N.load().lmd_vl_ev_slots(self.n_owned, pattern.code))
            ev_t = torch.empty(2 * max(slots, 1), dtype=torch.float64, device=dev)
        stg = self._staging.get(self._key(pattern, newton3))
        if stg is not None and mode != 1:
            groups, _, gsize, _, bits = stg
            direct = out is not None and len(out) == self.n_owned
            fx, fy, fz = ((out.force_x, out.force_y, out.force_z) if direct
                          else (self._fx, self._fy, self._fz))
            N.call("lmd_force_vl_staged", mode, (N.FLAG_ENERGY if energy else 0) | self.knobs,
                   N.make_lj(self.params), self.n_owned, N.ptr(self._pos4), N.ptr(self._soa),
                   self._soa.shape[1], self.n_owned + self.n_halo, gsize, N.ptr(groups), bits,
                   N.ptr(tile_off), N.ptr(kmax),
                   N.ptr(nbr), N.ptr(self._perm) if direct else None, N.ptr(fx), N.ptr(fy),
                   N.ptr(fz), N.ptr(ev_t), N.ptr(stats_t), N.stream())
            self._collected_into = out if direct else None
            return stats_t
        if mode == 1:
            self._fx.zero_()
            self._fy.zero_()
            self._fz.zero_()
        direct = out is not None and mode != 1 and len(out) == self.n_owned
        fx, fy, fz = ((out.force_x, out.force_y, out.force_z) if direct
                      else (self._fx, self._fy, self._fz))
        N.call("lmd_force_vl", pattern.code, mode, (N.FLAG_ENERGY if energy else 0) | self.knobs,
               N.make_lj(self.params), self.n_owned, N.ptr(self._pos4),
               N.ptr(self._soa) if self.use_soa else None, self._soa.shape[1],
               N.ptr(tile_off), N.ptr(kmax), N.ptr(nbr),
               N.ptr(self._perm) if direct else None, N.ptr(fx), N.ptr(fy), N.ptr(fz),
               N.ptr(ev_t), N.ptr(stats_t), N.stream())
        self._collected_into = out if direct else None
        return stats_t

    def launch_force_overlapped(self, owned, exchange, pattern, newton3: bool,
                                energy: bool = False, stats_t=None, ev_t=None, out=None,
                                side_stream=None):
        """One force phase with an external ghost layer, the exchange hidden
        behind the interior groups: owned rows -> interior groups on a side
        stream, meanwhile ``exchange()`` (the ghost exchange, returning the
        (n_halo, 3) ghost rows) -> ghost rows -> boundary groups on the
        current stream -> join.  Same pairs and forces as refresh + launch."""
        pattern = as_pattern(pattern)
        self.ensure_lists(pattern, newton3)
        if self._vls.get(self._key(pattern, newton3)) is None or not self._external_halo:
            rows = exchange()
            self.refresh(owned, rows)
            return self.launch_force(pattern, newton3, energy, stats_t, ev_t, out)
        dev = self._rows.device
        if stats_t is None:
            stats_t = N.new_stats(dev)
        stats_t.zero_()
        main = torch.cuda.current_stream(dev)
        side = side_stream or torch.cuda.Stream(dev)
        self.refresh_owned(owned)
        forked = torch.cuda.Event()
        forked.record(main)
        side.wait_event(forked)
        with torch.cuda.stream(side):
            self.launch_force(pattern, newton3, energy, stats_t, ev_t, out, part="interior",
                              zero_stats=False, defer_ev=True)
        rows = exchange()
        self.refresh_ghosts(owned, rows)
        self.launch_force(pattern, newton3, energy, stats_t, ev_t, out, part="boundary",
                          zero_stats=False, defer_ev=True)
        main.wait_stream(side)
        if energy:
            self.reduce_ev(pattern, newton3, stats_t, ev_t)
        return stats_t

    def pair_count(self, st, newton3: bool) -> int:
        """pair_interactions in the reference's convention from a device
        stats record of launch_force (Newton3 on full lists: owned-owned
        pairs were seen from both sides)."""
        p = int(st.pair_interactions)
        if self._kernel_n3(newton3) == 2:
            h = int(st.pairs_owned_halo)
            p = (p - h) // 2 + h
        return p

    def vl_stats(self, newton3: bool, pattern, V: int):
        key = (self.structure_version, bool(newton3), pattern, V)
        hit = self._stats_cache.get(key)
        if hit is None:
            a, b = pattern.shape(V)
            t = N.new_stats(self._pos4.device)
            N.call("lmd_vl_stats", self.n_owned, a, b, V, N.ptr(self._count(newton3, pattern)), N.ptr(t),
                   N.stream())
            st = N.read_stats(t)
            hit = (int(st.kernel_invocations), int(st.lane_slots), int(st.useful_interactions))
            self._stats_cache[key] = hit
        return hit

    def compute_forces(self, traversal, newton3: bool, pattern, vector_width: int,
                       energy: bool = False) -> KernelStats:
        from .traversals import TraversalKind, as_traversal
        validate_vector_width(vector_width)
        if as_traversal(traversal) is not TraversalKind.VL:
            raise ConfigurationError(f"{traversal} traversal requires the verlet-list container")
        pattern = as_pattern(pattern)
        inv, slots, useful = self.vl_stats(newton3, pattern, vector_width)
        st = N.read_stats(self.launch_force(pattern, newton3, energy))
        if st.overlap:
            raise ParticleOverlapError("zero distance between interacting particles")
        return KernelStats(kernel_invocations=inv, lane_slots=slots, useful_interactions=useful,
                           pair_interactions=self.pair_count(st, newton3), epot=st.epot,
                           virial=st.virial)

    def compute_forces_once(self, traversal, newton3: bool, pattern, vector_width: int,
                            energy: bool = False):
        """``compute_forces`` for a container that is used once (the one-shot
        ``force_phase``): the list-free kernel ``lmd_vls_direct`` walks the
        candidates of the row-aligned groups, counts the list lengths for the
        statistics and evaluates the pairs inside the cutoff -- no lists are
        written.  Same KernelStats and forces (to summation order) as
        ``compute_forces``.  Returns None where it does not apply (other
        orders, half-list Newton3, groups too large to stage): the caller
        then takes ``compute_forces``."""
        from .traversals import TraversalKind, as_traversal
        validate_vector_width(vector_width)
        if as_traversal(traversal) is not TraversalKind.VL:
            raise ConfigurationError(f"{traversal} traversal requires the verlet-list container")
        pattern = as_pattern(pattern)
        mode = self._kernel_n3(newton3)
        if (not self.segmented or self._rows is None or mode == 1 or not self.n_owned
                or self._staged_for(pattern, False) == 0 or self._lists):
            return None
        plan = self._vls_plan_groups()
        if plan["rows"] == 0:
            return None
        dev = self._rows.device
        n, ng = self.n_owned, plan["ngroups"]
        rl = float(self.params.interaction_length)   # the walk keeps candidates within rl
        vol = float(np.prod(self.box.lengths))
        est = (n + self.n_halo) / vol * (4.0 / 3.0) * np.pi * rl ** 3
        cap = int(est * 1.25 + 24)
        stats_t = N.new_stats(dev)
        slots = int(N.load().lmd_vls_ev_slots(ng))
        ev_t = torch.empty(2 * max(slots, 1), dtype=torch.float64, device=dev) if energy else None
        count = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        half = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        info = plan["info"]
        while True:
            cap = (cap + 7) // 8 * 8
            scratch = torch.empty(ng * 128 * cap, dtype=torch.int16, device=dev)
            info[3:5].zero_()
            stats_t.zero_()
            N.call("lmd_vls_direct", self.grid, mode, N.FLAG_ENERGY if energy else 0,
                   N.make_lj(self.params), n, plan["rows"], N.ptr(self._rows),
                   N.ptr(plan["fs_own"]), N.ptr(self._o_count), N.ptr(plan["fs_img"]),
                   N.ptr(self._h_count), N.ptr(plan["groups"]), ng, cap, N.ptr(scratch), None,
                   N.ptr(self._fx), N.ptr(self._fy), N.ptr(self._fz),
                   N.ptr(ev_t) if energy else None, N.ptr(stats_t), N.ptr(count), N.ptr(half),
                   N.ptr(info), N.stream())
            seen = int(info[4].item())
            if seen <= cap:
                break
            if seen > 4096:
                return None
            cap = seen + 8
        del scratch
        self._collected_into = None
        self._counts[False] = count
        if self.n3_mode == "full_list":
            self._counts[True] = half
        inv, lane_slots, useful = self.vl_stats(newton3, pattern, vector_width)
        st = N.read_stats(stats_t)
        if st.overlap:
            raise ParticleOverlapError("zero distance between interacting particles")
        return KernelStats(kernel_invocations=inv, lane_slots=lane_slots,
                           useful_interactions=useful,
                           pair_interactions=self.pair_count(st, newton3), epot=st.epot,
                           virial=st.virial)

    def collect_forces(self, owned) -> None:
        if self._collected_into is not None and owned is self._collected_into:
            self._collected_into = None        # the kernel already wrote them
            return
        self._collected_into = None
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
