"""Device MD over a spatial brick decomposition (BASELINE
configs 4 and 5 at N GPUs): one process per GPU, each owning the particles of
its brick (``decomposition.BrickDecomposition``).

Per iteration, as the single-domain loop (``simulation.run_md``,
driver.py:171-224): pre-force half step; the rebuild decision (displacement
>= skin/2 or the period) is reduced over the ranks (MAX), because a rebuild
migrates particles, which is collective; at a rebuild positions are wrapped
into the global periodic box, every rank's particles move to the rank owning
their brick (state: position, velocity, force, old force, id), the ghost
layer (thickness rc + skin, exact periodic images across the global boundary)
is planned and the container rebuilt over [owned | ghosts]; between rebuilds
only the ghost positions move (one batched P2P group per axis stage).  Force
phase, collection and the post-force half step are local: ghost pairs are
one-sided (the owned side is i, traversals.py:157-160), so no force goes
back.  Pair counts are summed over the ranks.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _native as N
from .containers import needs_rebuild_buffer
from .domain import SimulationBox, apply_boundaries
from .driver import make_container
from .errors import ConfigurationError, ParticleOverlapError, SimulationDivergedError
from .integrator import POST_FORCE, PRE_FORCE, velocity_verlet_step
from .kernels import KernelStats, validate_vector_width
from .particles import HALO, ParticleBuffer
from .tuning import Configuration, ContainerKind, TimeMetric, Tuner, TuningPolicy

# migrated state: x y z | vx vy vz | fx fy fz | ofx ofy ofz | id
_STATE = ("pos_x", "pos_y", "pos_z", "vel_x", "vel_y", "vel_z", "force_x", "force_y", "force_z",
          "old_force_x", "old_force_y", "old_force_z")


@dataclass
class BrickRunSummary:
    steps: int
    wall_time_s: float
    force_time_s: float
    rebuilds: int
    particles_global: int
    particles_local: int
    ghosts_local: int
    pairs_per_step: list
    phase_selections: list = None

    @property
    def particle_steps_per_s(self) -> float:
        return self.particles_global * self.steps / self.wall_time_s if self.wall_time_s else 0.0


def _pack(buf: ParticleBuffer) -> torch.Tensor:
    cols = [getattr(buf, f) for f in _STATE] + [buf.id.to(torch.float64)]
    return torch.stack(cols, dim=1).contiguous()


def _unpack(rows: torch.Tensor, device) -> ParticleBuffer:
    out = ParticleBuffer.empty(rows.shape[0], device=device)
    for k, f in enumerate(_STATE):
        getattr(out, f).copy_(rows[:, k])
    out.id.copy_(rows[:, len(_STATE)].to(torch.int64))
    return out


def _ghost_buffer(ghost_pos: torch.Tensor, device) -> ParticleBuffer:
    g = ParticleBuffer.empty(ghost_pos.shape[0], device=device)
    g.pos_x.copy_(ghost_pos[:, 0])
    g.pos_y.copy_(ghost_pos[:, 1])
    g.pos_z.copy_(ghost_pos[:, 2])
    g.ownership.fill_(HALO)
    return g


def _positions(buf: ParticleBuffer) -> torch.Tensor:
    return torch.stack([buf.pos_x, buf.pos_y, buf.pos_z], dim=1).contiguous()


def _allreduce(t: torch.Tensor, dec, op=dist.ReduceOp.SUM) -> torch.Tensor:
    if dec.nranks > 1:
        if dec._host_staged(t):
            h = t.cpu()
            dist.all_reduce(h, op=op, group=dec.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=op, group=dec.group)
    return t


def run_md_bricks(owned: ParticleBuffer, dec, params, iterations: int, vector_width: int = 8,
                  *, config: Configuration | None = None, configurations=None,
                  policy: TuningPolicy | None = None, rebuild_period: int | None = None,
                  record: bool = True):
    """Run ``iterations`` MD steps of this rank's particles (global
    coordinates, inside its brick or anywhere: the first rebuild migrates
    them).  Returns (final local ParticleBuffer, BrickRunSummary).

    ``config`` fixes the configuration; otherwise ``configurations`` is the
    search space of a per-rank tuner (tuning.py:182-271) whose samples --
    the force phase's device time, CUDA events -- are MAX-reduced over the
    ranks before they are recorded, so every rank selects the same
    configuration.  One container per container kind; a
    container last rebuilt before the latest migration is rebuilt when next
    used, and that iteration's sample is displaced."""
    validate_vector_width(vector_width)
    if config is None:
        if not configurations:
            raise ConfigurationError("give a configuration or a search space")
        space = list(configurations)
        tuner = Tuner(space, policy or TuningPolicy(1, max(100, 2 * len(space)), "mean", "time"))
    else:
        space = [config]
        tuner = None
    for c in space:
        if c.container not in (ContainerKind.LINKED_CELLS, ContainerKind.VERLET_LISTS):
            raise ConfigurationError("brick MD runs the linked-cell or Verlet-list containers")
        if not c.is_valid():
            raise ConfigurationError(f"invalid configuration {c.label!r}")
    dev = owned.device
    gbox = SimulationBox(dec.lo, dec.hi, ("periodic",) * 3)
    kw = {} if rebuild_period is None else {"rebuild_period": rebuild_period}
    containers: dict = {}      # kind -> [container, epoch of its last rebuild]
    epoch = 0                  # bumped by every migration
    ghosts = None
    ref_pos = None             # owned positions at the last migration
    since_migration = 0
    rebuilds = 0
    pairs_per_step = []
    selections: list = []
    force_time = 0.0
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    stats_t = N.new_stats(dev)
    side = torch.cuda.Stream(device=dev) if dev.type == "cuda" else None
    metric = TimeMetric() if tuner is not None else None
    torch.cuda.synchronize(dev)
    if dec.nranks > 1:
        dist.barrier(group=dec.group)
    start = time.perf_counter()
    for it in range(iterations):
        velocity_verlet_step(owned, params, PRE_FORCE, check=False)
        cfg, _phase = tuner.next_configuration(it) if tuner is not None else (config, None)
        slot = containers.get(cfg.container)
        if slot is None:
            slot = containers[cfg.container] = [make_container(cfg.container, dec.local_box(),
                                                               params, **kw), -1]
        cont = slot[0]
        # the ghost layer was planned at the last migration: its validity
        # (displacement < skin/2, the period) is measured from there, not from
        # a container's own later rebuild
        period = rebuild_period or cont.rebuild_period
        need = ghosts is None or needs_rebuild_buffer(owned, ref_pos, params.skin,
                                                      since_migration, period)
        flag.fill_(1 if need else 0)
        need = bool(_allreduce(flag, dec, dist.ReduceOp.MAX).item())
        displaced = False
        if need:
            apply_boundaries(owned, gbox)
            bad = owned.extra.get("nonfinite")
            if bad is not None and int(bad.item()):
                raise SimulationDivergedError("non-finite particle state in the brick run")
            owned = _unpack(dec.migrate(_pack(owned)), dev)
            ref_pos = _positions(owned)
            ghosts = _ghost_buffer(dec.plan(ref_pos), dev)
            since_migration = 0
            epoch += 1
            rebuilds += 1
        # Steady state on segmented Verlet lists: the ghost exchange runs
        # while the interior groups (no ghost rows staged) are computing
        # (launch_force_overlapped); otherwise exchange, refresh, compute.
        overlapped = (not need and slot[1] == epoch
                      and cfg.container is ContainerKind.VERLET_LISTS
                      and cont._vls_for(cfg.pattern, cfg.newton3) is not None)
        if not need and not overlapped:
            rows = dec.exchange_positions(owned.pos_x, owned.pos_y, owned.pos_z)
            ghosts.pos_x.copy_(rows[:, 0])
            ghosts.pos_y.copy_(rows[:, 1])
            ghosts.pos_z.copy_(rows[:, 2])
        if slot[1] != epoch:
            cont.rebuild(owned, ghosts)
            slot[1] = epoch
            displaced = True
        if not overlapped:
            cont.refresh(owned, ghosts)
        cont.steps_since_rebuild += 1
        since_migration += 1
        if cfg.container is ContainerKind.VERLET_LISTS:
            displaced |= cont.ensure_lists(cfg.pattern, cfg.newton3)
        t0 = time.perf_counter()
        if metric is not None:
            metric.begin_region()
        if overlapped:
            o = owned
            stats_t = cont.launch_force_overlapped(
                o, lambda: dec.exchange_positions(o.pos_x, o.pos_y, o.pos_z), cfg.pattern,
                cfg.newton3, False, stats_t, side_stream=side)
            inv, lane_slots, useful = cont.vl_stats(cfg.newton3, cfg.pattern, vector_width)
            raw = N.read_stats(stats_t)
            if raw.overlap:
                raise ParticleOverlapError("zero distance between interacting particles")
            st = KernelStats(inv, lane_slots, useful, cont.pair_count(raw, cfg.newton3))
        else:
            st = cont.compute_forces(cfg.traversal, cfg.newton3, cfg.pattern, vector_width)
        if metric is not None:
            sample = torch.tensor([metric.end_region()], dtype=torch.float64, device=dev)
            sample = float(_allreduce(sample, dec, dist.ReduceOp.MAX).item())
            d = torch.tensor([1 if displaced else 0], dtype=torch.int32, device=dev)
            displaced = bool(_allreduce(d, dec, dist.ReduceOp.MAX).item())
            tuner.record_sample(sample, displaced=displaced)
        force_time += time.perf_counter() - t0
        cont.collect_forces(owned)
        velocity_verlet_step(owned, params, POST_FORCE, check=False)
        if record:
            p = torch.tensor([st.pair_interactions], dtype=torch.int64, device=dev)
            pairs_per_step.append(int(_allreduce(p, dec).item()))
    torch.cuda.synchronize(dev)
    if dec.nranks > 1:
        dist.barrier(group=dec.group)
    wall = time.perf_counter() - start
    n_local = len(owned)
    tot = torch.tensor([n_local], dtype=torch.int64, device=dev)
    n_global = int(_allreduce(tot, dec).item())
    nonfinite = owned.extra.get("nonfinite")
    if nonfinite is not None and int(nonfinite.item()):
        raise SimulationDivergedError("non-finite particle state in the brick run")
    if tuner is not None:
        selections = [c.label for c in tuner.phase_selection]
    summary = BrickRunSummary(iterations, wall, force_time, rebuilds, n_global, n_local,
                              len(ghosts) if ghosts is not None else 0, pairs_per_step,
                              selections)
    return owned, summary
