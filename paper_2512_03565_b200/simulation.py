"""Device-resident MD loop with the runtime tuner (driver.py:132-313).

Per iteration, as the reference's ``run_simulation`` (driver.py:171-224):
pre-force half step, tuner decision, container rebuild when
``needs_rebuild`` fires (displacement >= skin/2 or the period), images,
metric-bracketed force phase, force collection, tuner sample (displaced by a
rebuild -> retaken), post-force half step, boundaries, one record.  All state
stays in HBM; the force phase is bracketed with CUDA events on its stream
(``metric="time"``) or counted in lane slots (``"laneops"``).

Extensions: Verlet lists join the search space; ``retune_drift`` starts a new
tuning phase when the peak cell occupancy drifts by more than that fraction
since the last phase started ("re-tuning as density changes").
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .containers import LinkedCellsContainer, max_particles_per_cell
from .domain import apply_boundaries, as_box
from .driver import make_container
from .errors import ConfigurationError, ParticleOverlapError, ScenarioError, SimulationDivergedError
from .integrator import POST_FORCE, POST_THEN_PRE, PRE_FORCE, velocity_verlet_step
from .kernels import KernelStats, validate_vector_width
from .traversals import traversal_code
from .tuning import (PRODUCTION, Configuration, ContainerKind, Tuner, TuningPolicy,
                     make_metric_provider)

CSV_COLUMNS = (
    "iteration", "phase", "container", "traversal", "newton3", "pattern",
    "metric_value", "lane_slots", "useful_interactions", "blank_lanes",
    "pair_interactions", "particle_count",
)


@dataclass
class IterationRecord:
    """One CSV row (driver.py:36-56)."""

    iteration: int
    phase: str
    configuration: Configuration
    metric_value: float
    lane_slots: int
    useful_interactions: int
    blank_lanes: int
    pair_interactions: int
    particle_count: int

    def row(self) -> list:
        c = self.configuration
        return [str(self.iteration), self.phase, c.container.value, c.traversal.value,
                "true" if c.newton3 else "false", c.pattern.value, repr(self.metric_value),
                str(self.lane_slots), str(self.useful_interactions), str(self.blank_lanes),
                str(self.pair_interactions), str(self.particle_count)]


@dataclass
class RunSummary:
    per_config_metric: dict
    phase_selections: list
    failed_configs: list
    wall_time_s: float
    particle_count: int
    initial_max_per_cell: int
    final_max_per_cell: int
    final_max_speed: float
    force_time_s: float = 0.0    # device time of the force launches (CUDA events)
    steps: int = 0
    retunes: int = 0
    rebuilds: int = 0
    extra: dict = field(default_factory=dict)

    @property
    def total_metric(self) -> float:
        return sum(self.per_config_metric.values())

    @property
    def particle_steps_per_s(self) -> float:
        return self.particle_count * self.steps / self.wall_time_s if self.wall_time_s else 0.0


def _launch(cont, cfg: Configuration, V: int, energy: bool, owned=None):
    kind = cfg.container
    if kind is ContainerKind.LINKED_CELLS:
        code = traversal_code(cfg.traversal)
        return cont.launch_force(cfg.pattern, energy, traversal=code, newton3=cfg.newton3)
    if kind is ContainerKind.VERLET_LISTS:   # forces written in the caller's order
        return cont.launch_force(cfg.pattern, cfg.newton3, energy, out=owned)
    return cont.launch_force(energy, pattern=cfg.pattern)


def _geometry(cont, cfg: Configuration, V: int):
    """The geometric statistics of the structure the force phase ran on
    (cached per rebuild; read before the structure can change)."""
    kind = cfg.container
    if kind is ContainerKind.LINKED_CELLS:
        code = traversal_code(cfg.traversal)
        return cont._lc_stats(code, cfg.newton3, cfg.pattern, V)
    if kind is ContainerKind.VERLET_LISTS:
        return cont.vl_stats(cfg.newton3, cfg.pattern, V)
    return cont.vcl_stats(cfg.newton3, cfg.pattern, V)


def _stats_from(st, cont, cfg: Configuration, geo) -> KernelStats:
    kind = cfg.container
    if kind is ContainerKind.LINKED_CELLS:
        once = cont.uses_colored_n3(traversal_code(cfg.traversal), cfg.newton3)
        return LinkedCellsContainer.finish_stats(st, cfg.newton3 and not once, *geo)
    if kind is ContainerKind.VERLET_LISTS:
        if st.overlap:
            raise ParticleOverlapError("zero distance between interacting particles")
        return KernelStats(geo[0], geo[1], geo[2], cont.pair_count(st, cfg.newton3), st.epot,
                           st.virial)
    return LinkedCellsContainer.finish_stats(st, cfg.newton3, *geo)


def _finish(cont, cfg: Configuration, V: int, stats_t) -> KernelStats:
    return _stats_from(N.read_stats(stats_t), cont, cfg, _geometry(cont, cfg, V))


class _DeferredStats:
    """Force-phase statistics read one step late: the device record is copied
    to pinned memory right after the launch and parsed at the next step's
    host synchronisation (the rebuild decision), so a step needs one host
    read instead of two.  An overlap (ParticleOverlapError) is then raised at
    the start of the following step, before its force phase."""

    def __init__(self):
        import torch
        self.buf = [torch.empty(N.STATS_BYTES, dtype=torch.uint8).pin_memory()
                    for _ in range(2)]
        self.pending = None
        self.k = 0
        self.stream = torch.cuda.current_stream()   # fixed for the run

    def push(self, stats_t, cont, cfg, geo, record):
        import torch
        b = self.buf[self.k % 2]
        self.k += 1
        b.copy_(stats_t.view(torch.uint8), non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(self.stream)
        self.pending = (ev, b, cont, cfg, geo, record)

    def resolve(self):
        if self.pending is None:
            return
        ev, b, cont, cfg, geo, record = self.pending
        self.pending = None
        ev.synchronize()
        st = N.Stats.from_buffer_copy(b.numpy().tobytes())
        stats = _stats_from(st, cont, cfg, geo)
        if record is not None:
            record.pair_interactions = stats.pair_interactions


def run_md(owned, box, params, iterations: int, vector_width: int = 8, *,
           configurations=None, fixed_config: Configuration | None = None,
           policy: TuningPolicy | None = None, metric: str = "time",
           cluster_size: int | None = None, rebuild_period: int | None = None,
           retune_drift: float | None = None, energy: bool = False, record: bool = True,
           wrap: str = "always", fuse_halves: bool | None = None):
    """Run ``iterations`` MD steps on device-resident ``owned`` (our ParticleBuffer).

    Returns (records, summary).  With ``fixed_config`` the tuner is off.

    ``wrap="always"`` applies the boundaries after every step as the
    reference does (driver.py:214); in a large periodic system some particle
    then wraps every step, its displacement looks like a box length and
    ``needs_rebuild`` fires every step, so every tuning sample is displaced.
    ``fuse_halves`` (default on, effective with ``wrap="at_rebuild"``): a
    step's post-force half and the next step's pre-force half run as one pass
    over the particles (the same expressions: bit for bit the same
    trajectory).

    ``wrap="at_rebuild"`` keeps positions unwrapped between rebuilds and
    wraps them just before a rebuild (the usual MD practice): rebuilds follow
    the skin/period rule and the tuner can finish its phases.  Forces are the
    same up to rounding of the unwrapped coordinates."""
    if wrap not in ("always", "at_rebuild"):
        raise ConfigurationError(f"unknown wrap policy {wrap!r}")
    validate_vector_width(vector_width)
    box = as_box(box)
    if fixed_config is None:
        if not configurations:
            raise ConfigurationError("search space has no valid configuration")
        pol = policy or TuningPolicy(metric=metric)
        if policy is None:
            pol = TuningPolicy(pol.samples_per_config,
                               max(1000, pol.samples_per_config * len(configurations)),
                               pol.reduction, metric)
        tuner = Tuner(list(configurations), pol)
    else:
        if not fixed_config.is_valid():
            raise ConfigurationError(f"invalid configuration {fixed_config.label!r}")
        tuner = None
    lane_total = [0]
    deferred = tuner is None and metric in ("time", "iteration")
    if deferred:   # nobody waits for the samples: resolve the events after the run
        from .tuning import DeferredTimeMetric
        provider = DeferredTimeMetric()
    else:
        provider = make_metric_provider(metric, lambda: lane_total[0])
    containers: dict = {}
    late = _DeferredStats()
    records: list = []
    per_config: dict = {}
    margin = params.interaction_length
    initial_max = max_particles_per_cell(owned, box, margin)
    phase_max = initial_max
    retunes = 0
    rebuilds = 0
    force_events: list = []   # CUDA events around each force launch (device time)
    start = time.perf_counter()
    whole = metric == "iteration"
    try:
        # with positions wrapped at rebuilds only, nothing sits between a
        # step's post-force half and the next step's pre-force half: one
        # fused pass (the same arithmetic) serves both
        if fuse_halves is None:
            fuse_halves = True
        fuse_halves = bool(fuse_halves) and wrap == "at_rebuild"
        pre_done = False
        for it in range(iterations):
            if whole:
                provider.begin_region()
            if not pre_done:
                velocity_verlet_step(owned, params, PRE_FORCE, check=False)
            pre_done = False
            if tuner is not None:
                if retune_drift and it > 0 and tuner.selected is not None and it % 10 == 0:
                    cur = max_particles_per_cell(owned, box, margin)
                    if abs(cur - phase_max) > retune_drift * max(phase_max, 1):
                        tuner.request_retune()
                        phase_max = cur
                        retunes += 1
                cfg, phase = tuner.next_configuration(it)
            else:
                cfg, phase = fixed_config, PRODUCTION
            ckey = (cfg.container, cfg.cluster_size)
            cont = containers.get(ckey)
            if cont is None:
                kw = {} if rebuild_period is None else {"rebuild_period": rebuild_period}
                m = cfg.cluster_size or cluster_size or vector_width
                cont = make_container(cfg.container, box, params, cluster_size=m, **kw)
                containers[ckey] = cont
            rebuilt = False
            fresh = cont.reference_positions is None
            # containers that reduce the displacement inside their refresh
            # (segmented Verlet lists) decide and refresh in one pass
            fused = getattr(cont, "refresh_and_check", None)
            if fresh or (fused(owned) if fused is not None else cont.needs_rebuild(owned)):
                late.resolve()   # (the decision above synchronised)
                if wrap == "at_rebuild":
                    apply_boundaries(owned, box)
                cont.rebuild(owned)
                cont.refresh(owned)
                rebuilt = not fresh
                rebuilds += 1
            else:
                late.resolve()
                if fused is None:
                    cont.refresh(owned)
            cont.steps_since_rebuild += 1
            # lazily built structures (Verlet lists per interaction order) are
            # built here, outside the force-phase bracket: the reference's
            # bracket holds the force computation only (driver.py:203-207)
            built = cfg.container is ContainerKind.VERLET_LISTS and \
                cont.ensure_lists(cfg.pattern, cfg.newton3)
            if whole:
                # the iteration bracket sees every build: such samples are displaced
                rebuilt = rebuilt or fresh or built
            if not whole:
                provider.begin_region()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev0.record()
            stats_t = _launch(cont, cfg, vector_width, energy, owned)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev1.record()
            force_events.append((ev0, ev1))
            sample = provider.end_region() if metric not in ("laneops", "iteration") else None
            if deferred and not energy:
                geo = _geometry(cont, cfg, vector_width)
                stats = KernelStats(geo[0], geo[1], geo[2], -1)   # pairs filled in late
            else:
                stats = _finish(cont, cfg, vector_width, stats_t)
            lane_total[0] += stats.lane_slots
            if sample is None and not whole:
                sample = provider.end_region()
            cont.collect_forces(owned)
            if fuse_halves and it + 1 < iterations:
                velocity_verlet_step(owned, params, POST_THEN_PRE, check=False)
                pre_done = True
            else:
                velocity_verlet_step(owned, params, POST_FORCE, check=False)
            if wrap == "always":
                apply_boundaries(owned, box)
            if whole:
                sample = provider.end_region()
            if tuner is not None:
                tuner.record_sample(sample, displaced=rebuilt)
            rec = None
            if record:
                rec = IterationRecord(it, phase, cfg, sample, stats.lane_slots,
                                      stats.useful_interactions, stats.blank_lanes,
                                      stats.pair_interactions, len(owned))
                records.append(rec)
            if deferred and not energy:
                late.push(stats_t, cont, cfg, geo, rec)
            if not deferred:
                per_config[cfg.label] = per_config.get(cfg.label, 0.0) + sample
        late.resolve()
        if deferred:
            values = provider.resolve()
            for rec in records:
                rec.metric_value = values[int(rec.metric_value)]
            per_config[fixed_config.label] = float(sum(values))
        flag = owned.extra.get("nonfinite")
        if flag is not None and int(flag.item()):
            raise SimulationDivergedError("non-finite particle state")
    except SimulationDivergedError as exc:
        exc.records = records
        raise
    if wrap == "at_rebuild":
        apply_boundaries(owned, box)
    torch.cuda.synchronize()
    wall = time.perf_counter() - start
    force_time = sum(a.elapsed_time(b) for a, b in force_events) * 1e-3
    speed = torch.sqrt(owned.vel_x ** 2 + owned.vel_y ** 2 + owned.vel_z ** 2)
    failed, selections = [], []
    if tuner is not None:
        selections = [c.label for c in tuner.phase_selection]
    summary = RunSummary(
        per_config_metric=dict(sorted(per_config.items())), phase_selections=selections,
        failed_configs=failed, wall_time_s=wall, particle_count=len(owned),
        initial_max_per_cell=initial_max,
        final_max_per_cell=max_particles_per_cell(owned, box, margin),
        final_max_speed=float(speed.max().item()) if len(owned) else 0.0,
        force_time_s=force_time, steps=iterations, retunes=retunes, rebuilds=rebuilds)
    return records, summary


def emit_csv(records, path) -> None:
    """Records as CSV with the reference's column order (driver.py:262-270)."""
    if not records:
        raise ScenarioError("no records to write")
    lines = [",".join(CSV_COLUMNS)] + [",".join(r.row()) for r in records]
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("\n".join(lines) + "\n")


def read_records_csv(path) -> list:
    from .kernels import PatternKind
    from .traversals import TraversalKind
    with open(path, encoding="utf-8") as fh:
        lines = [ln.rstrip("\n") for ln in fh if ln.strip()]
    if tuple(lines[0].split(",")) != CSV_COLUMNS:
        raise ScenarioError(f"unexpected CSV header {lines[0]!r}")
    out = []
    for ln in lines[1:]:
        p = ln.split(",")
        cfg = Configuration(ContainerKind(p[2]), TraversalKind(p[3]), p[4] == "true",
                            PatternKind(p[5]))
        out.append(IterationRecord(int(p[0]), p[1], cfg, float(p[6]), int(p[7]), int(p[8]),
                                   int(p[9]), int(p[10]), int(p[11])))
    return out


def run_md_graph(owned, box, params, iterations: int, vector_width: int = 8, *,
                 config: Configuration, rebuild_period: int | None = None,
                 energy: bool = False):
    """``run_md`` for a fixed Verlet-list configuration with the steady-state
    step as a CUDA graph (the north star's "CUDA streams and graphs instead
    of a tracing compiler").

    After every rebuild two graphs are captured: (refresh -> force, written
    in the caller's order -> post-force half step) and (the next step's
    pre-force half step -> max-displacement kernel), each ending with an
    async copy of (stats, displacement) into pinned host memory.  Each later
    step is two replays and one host read, which decides the next rebuild
    (displacement >= skin/2 or the period); a rebuild step runs the same
    work eagerly and re-captures.  Positions
    are wrapped at rebuilds (``wrap="at_rebuild"``).  Same kernels in the
    same order as ``run_md``: identical trajectory.  Returns (records,
    summary)."""
    from .verlet_lists import VerletListContainer
    if config.container is not ContainerKind.VERLET_LISTS:
        raise ConfigurationError("run_md_graph runs the Verlet-list container")
    if not config.is_valid():
        raise ConfigurationError(f"invalid configuration {config.label!r}")
    validate_vector_width(vector_width)
    box = as_box(box)
    dev = owned.device
    kw = {} if rebuild_period is None else {"rebuild_period": rebuild_period}
    cont = VerletListContainer(box, params, device=dev, **kw)
    pattern, n3 = config.pattern, config.newton3
    stats_t = N.new_stats(dev)
    disp = torch.zeros(1, dtype=torch.float64, device=dev)
    host = torch.zeros(N.STATS_BYTES + 8, dtype=torch.uint8).pin_memory()
    dev_out = torch.zeros(N.STATS_BYTES + 8, dtype=torch.uint8, device=dev)
    slots = int(N.load().lmd_vl_ev_slots(len(owned), pattern.code))
    ev_t = torch.empty(2 * max(slots, 1), dtype=torch.float64, device=dev)
    half = (0.5 * params.skin) ** 2
    records: list = []
    pairs_total = 0
    rebuilds = 0

    def step():
        """One step from the refresh to the post-force half step."""
        cont.refresh(owned)
        cont.launch_force(pattern, n3, energy, stats_t, ev_t, out=owned)
        cont.collect_forces(owned)
        velocity_verlet_step(owned, params, POST_FORCE, check=False)
        dev_out[:N.STATS_BYTES].copy_(stats_t)

    def advance():
        """The next step's pre-force half step and displacement test."""
        velocity_verlet_step(owned, params, PRE_FORCE, check=False)
        N.call("lmd_max_displacement2", len(owned), N.ptr(owned.pos_x), N.ptr(owned.pos_y),
               N.ptr(owned.pos_z), N.ptr(cont.reference_positions), N.ptr(disp), N.stream())
        dev_out[N.STATS_BYTES:].copy_(disp.view(torch.uint8))

    def fetch():
        host.copy_(dev_out, non_blocking=True)

    def read():
        raw = host.numpy().tobytes()
        st = N.Stats.from_buffer_copy(raw[:N.STATS_BYTES])
        d2 = float(np.frombuffer(raw[N.STATS_BYTES:], dtype=np.float64)[0])
        return st, d2

    graphs = None
    side = torch.cuda.Stream(device=dev)
    start = time.perf_counter()
    velocity_verlet_step(owned, params, PRE_FORCE, check=False)
    need = True
    for it in range(iterations):
        last = it == iterations - 1
        if need:
            apply_boundaries(owned, box)
            cont.rebuild(owned)
            cont.ensure_lists(pattern, n3)
            step()
            if not last:
                advance()
            fetch()
            rebuilds += 1
            torch.cuda.current_stream().synchronize()
            # capture on a side stream with capture_begin / capture_end (the
            # torch.cuda.graph context also runs gc and empties the cache)
            graphs = (torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph())
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                for g_, fn in zip(graphs, (step, advance)):
                    g_.capture_begin()             # captured, not run
                    fn()
                    fetch()
                    g_.capture_end()
            torch.cuda.current_stream().wait_stream(side)
        else:
            graphs[0].replay()
            if not last:
                graphs[1].replay()
        torch.cuda.current_stream().synchronize()
        st, d2 = read()
        if st.overlap:
            raise ParticleOverlapError("zero distance between interacting particles")
        cont.steps_since_rebuild += 1
        geo = cont.vl_stats(n3, pattern, vector_width)
        pairs = cont.pair_count(st, n3)
        pairs_total += pairs
        records.append(IterationRecord(it, PRODUCTION, config, 0.0, geo[1], geo[2],
                                       geo[1] - geo[2], pairs, len(owned)))
        need = (cont.steps_since_rebuild >= cont.rebuild_period) or d2 >= half
    apply_boundaries(owned, box)
    torch.cuda.synchronize()
    wall = time.perf_counter() - start
    flag = owned.extra.get("nonfinite")
    if flag is not None and int(flag.item()):
        raise SimulationDivergedError("non-finite particle state")
    summary = RunSummary(per_config_metric={config.label: 0.0}, phase_selections=[],
                         failed_configs=[], wall_time_s=wall, particle_count=len(owned),
                         initial_max_per_cell=0, final_max_per_cell=0, final_max_speed=0.0,
                         force_time_s=0.0, steps=iterations, retunes=0,
                         extra={"rebuilds": rebuilds, "pairs_total": pairs_total})
    return records, summary


# ---------------------------------------------------------------- scenarios
# The reference's scenario-level entry points (driver.py:75-313) over the
# device MD loop: a ScenarioSpec (scenario.py:47-65; any object with its
# attributes) is materialised on the device and run with the spec's search
# space, tuning policy and metric.

def build_initial_state(spec, device="cuda"):
    """All lattice sources of ``spec`` in one owned buffer (driver.py:75-93):
    positions in x-fastest lattice order, ids sequential, source velocity plus
    uniform jitter drawn from ``default_rng(spec.seed)`` in the reference's
    call order."""
    from .particles import ParticleBuffer, lattice_positions
    rng = np.random.default_rng(spec.seed)
    pos, vel = [], []
    for src in spec.sources:
        p = lattice_positions(src.origin, src.counts, src.spacing)
        v = np.tile(np.asarray(src.velocity, dtype=np.float64).reshape(1, 3), (len(p), 1))
        pos.append(p)
        vel.append(v)
    pos = np.concatenate(pos) if pos else np.zeros((0, 3))
    vel = np.concatenate(vel) if vel else np.zeros((0, 3))
    offset = 0
    for src in spec.sources:
        n = int(np.prod(src.counts))
        if src.jitter > 0:
            for ax in range(3):
                vel[offset:offset + n, ax] += rng.uniform(-src.jitter, src.jitter, n)
        offset += n
    buf = ParticleBuffer.from_positions(pos, device=device)
    for ax, name in enumerate(("vel_x", "vel_y", "vel_z")):
        getattr(buf, name).copy_(torch.from_numpy(np.ascontiguousarray(vel[:, ax])))
    return buf


def resolve_search_space(spec) -> list:
    """enumerate_search_space over the spec's axes (driver.py:103-105)."""
    from .tuning import enumerate_search_space
    return enumerate_search_space(spec.containers, spec.traversals, spec.newton3_options,
                                  spec.patterns)


def run_simulation(spec, fixed_config: Configuration | None = None, **kw):
    """The reference's ``run_simulation`` (driver.py:132-224) on the device:
    returns (records, summary).  Without ``fixed_config`` the tuner searches
    ``resolve_search_space(spec)`` with the reference's default tuning
    interval ``max(1000, samples * |space|)``; the metric is ``spec.metric``
    ("laneops" is deterministic and reproduces the reference's records)."""
    owned = build_initial_state(spec)
    policy = None
    configs = None
    if fixed_config is None:
        configs = resolve_search_space(spec)
        if not configs:
            raise ConfigurationError("search space has no valid configuration")
        interval = spec.tuning_interval
        if interval is None:
            interval = max(1000, spec.samples_per_config * len(configs))
        policy = TuningPolicy(spec.samples_per_config, interval, spec.reduction, spec.metric)
    return run_md(owned, spec.box, spec.params, spec.iterations, spec.vector_width,
                  configurations=configs, fixed_config=fixed_config, policy=policy,
                  metric=spec.metric, cluster_size=spec.cluster_size,
                  rebuild_period=spec.rebuild_period, **kw)


def emit_summary(summary, path) -> None:
    """The reference's summary text (driver.py:296-313)."""
    lines = [
        f"particle_count: {summary.particle_count}",
        f"wall_time_s: {summary.wall_time_s:.3f}",
        f"total_force_phase_metric: {repr(summary.total_metric)}",
        f"initial_max_per_cell: {summary.initial_max_per_cell}",
        f"final_max_per_cell: {summary.final_max_per_cell}",
        f"final_max_speed: {repr(summary.final_max_speed)}",
        f"phase_selections: {' '.join(summary.phase_selections) or '-'}",
        f"failed_configs: {' '.join(summary.failed_configs) or '-'}",
        "per_config_metric:",
    ]
    for label, total in summary.per_config_metric.items():
        lines.append(f"  {label}: {repr(total)}")
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("\n".join(lines) + "\n")
