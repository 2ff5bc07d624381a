#!/usr/bin/env python
"""Benchmark: LJ FP64 pair-interactions/s on B200 (BASELINE.json metric).

Workload (N=1, the default ``--workload c4``): BASELINE config 4 --
16,777,216 particles on a 256^3 simple-cubic lattice at rho = 0.8 perturbed by
N(0, 0.05^2) per component (seed 42), periodic cube L = 275.77, LJ cutoff
2.5, FP64, Verlet lists with skin 0.3.  This is the configuration the
metric's 1/2/4/8-GPU series is quoted on and the largest BASELINE config
that fits one GPU.  A step is one force phase over the resident particles
(the reference's metric region, driver.py:203-207: refresh + kernel); the
neighbour structure is built before the timed region and its cost is
reported separately (``list_maintenance``: measured rebuild + list build,
amortised over the rebuild period).  The inputs (1.8 GB of particle state,
≈ 3 GB of lists) are far larger than the 126 MB L2, and the L2 is also
flushed (256 MiB write) before every timed step.

With --gpus N > 1: ``c4`` is strong scaling (the 16.8M-particle box split
into 2x1x1 / 2x2x1 / 2x2x2 bricks), ``c5`` weak scaling (8,388,608 particles
per GPU at rho 0.3, one brick per GPU), ``c2`` weak scaling (1M per GPU);
every step includes the NCCL point-to-point ghost exchange.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c4|c5|c2]
    python bench.py --impl reference ...   # the reference algorithm on host cores
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FLOPS_PER_PAIR = {False: 22, True: 25}   # SURVEY.md §8(d), counted on executor.py:93-111
DEFAULT_CONFIG = "vl,vl,false,v_by_one"
METRIC = "LJ FP64 pair-interactions/sec"
UNIT = "pair-interactions/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--workload", default="c4", choices=["c4", "c5", "c2"],
                    help="BASELINE config: c4 (16.8M lattice, strong scaling; default), "
                         "c5 (8.4M gas per GPU, weak), c2 (1M gas per GPU, weak)")
    ap.add_argument("--rho", type=float, default=0.8, help="c2 density")
    ap.add_argument("--n", "--particles", dest="n", type=int, default=None,
                    help="c2/c5: particles per GPU; c4: lattice side^3 (default 256^3)")
    ap.add_argument("--vector-width", type=int, default=8)
    ap.add_argument("--energy", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sweep", action="store_true", help="time every config, write gpurun_out/sweep.json")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
           0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], [], set()
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 3:
                    continue
                try:
                    sm.append(float(parts[0]))
                    mx.append(float(parts[1]))
                    mask = int(parts[2], 16)
                except ValueError:
                    continue
                for bit, name in REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        reasons.add(name)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------- workload
def make_workload(args, device, seed):
    """The per-GPU (c2, c5) or global (c4) workload, seeded."""
    from paper_2512_03565_b200 import workloads
    if args.workload == "c4":
        side = round(args.n ** (1.0 / 3.0)) if args.n else 256
        return workloads.config4(side, seed=seed, device=device)
    if args.workload == "c5":
        return workloads.config5(n=args.n or 8_388_608, seed=seed, device=device)
    return workloads.config2(args.rho, n=args.n or 1_000_000, seed=seed, device=device)


def scaling_of(args) -> str:
    return "strong" if args.workload == "c4" else "weak"


def params_for(cfg, w):
    from paper_2512_03565_b200 import LJParams
    # linked cells with cell size = cutoff (skin 0); Verlet/cluster lists skin 0.3
    skin = 0.0 if cfg.container.value == "lc" else w.skin
    return LJParams(cutoff=w.cutoff, skin=skin)


def fp64_peak_tflops(torch, N) -> float:
    """Measured FP64 DFMA peak on this GPU (lmd_dfma_burn, best of 5)."""
    sms = N.load().lmd_device_sm_count()
    blocks, threads, iters = sms * 8, 256, 400
    scratch = torch.empty(threads, dtype=torch.float64, device="cuda")
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    best = 1e30
    for rep in range(7):
        e0.record()
        N.call("lmd_dfma_burn", blocks, threads, iters, N.ptr(scratch), N.stream())
        e1.record()
        e1.synchronize()
        if rep >= 2:
            best = min(best, e0.elapsed_time(e1) * 1e-3)
    flops = blocks * threads * iters * 128 * 2.0
    return flops / best / 1e12


class Phase:
    """One force phase on a built container: refresh (positions -> backing,
    images or the exchanged ghost layer) + the force kernel."""

    def __init__(self, cfg, cont, buf, args, torch, N, dec=None, owned_rows=None):
        import paper_2512_03565_b200 as B
        self.torch = torch
        self.cfg, self.cont, self.buf, self.dec = cfg, cont, buf, dec
        self.owned_rows = owned_rows
        self.energy = args.energy
        self.kind = cfg.container.value
        dev = buf.device
        self.stats_t = N.new_stats(dev)
        if self.kind == "vl":
            slots = int(N.load().lmd_vl_ev_slots(cont.n_owned, cfg.pattern.code))
        elif self.kind == "lc":
            slots = max(int(N.load().lmd_lc_ev_slots(cont.grid)),
                        int(N.load().lmd_lc_n3_ev_slots(cont.grid)),
                        int(N.load().lmd_lc_tpi_ev_slots(cont.n_owned, cfg.pattern.code)))
        else:
            slots = int(N.load().lmd_vcl_ev_slots(cont.n_clusters))
        self.ev_t = torch.empty(2 * max(slots, 1), dtype=torch.float64, device=dev)
        self.trav = B.traversals.traversal_code(cfg.traversal)
        self.ghosts = None
        self.launch()   # builds lazily-built lists outside the timed region

    @property
    def overlapped(self) -> bool:
        """Brick runs on segmented Verlet lists hide the ghost exchange
        behind the interior groups (launch_force_overlapped)."""
        return (self.dec is not None and self.kind == "vl" and
                self.cont._vls_for(self.cfg.pattern, self.cfg.newton3) is not None)

    def refresh(self):
        if self.overlapped:
            return     # part of launch(): refresh, exchange and kernels interleave
        if self.dec is not None:
            b = self.buf
            rows = self.dec.exchange_positions(b.pos_x, b.pos_y, b.pos_z)
            if self.kind == "vl":
                self.cont.refresh(b, rows)
            else:
                self.ghosts.pos_x.copy_(rows[:, 0])
                self.ghosts.pos_y.copy_(rows[:, 1])
                self.ghosts.pos_z.copy_(rows[:, 2])
                self.cont.refresh(b, self.ghosts)
        elif self.kind == "lc":
            self.cont.refresh_positions(self.buf)
        elif self.kind == "vl":
            self.cont.refresh(self.buf)
        # vcl: refresh re-derives halo clusters (host-synchronising); not per step

    def launch(self):
        if self.overlapped:
            b = self.buf
            if not hasattr(self, "_side"):
                self._side = self.torch.cuda.Stream()
            return self.cont.launch_force_overlapped(
                b, lambda: self.dec.exchange_positions(b.pos_x, b.pos_y, b.pos_z),
                self.cfg.pattern, self.cfg.newton3, self.energy, self.stats_t, self.ev_t,
                side_stream=self._side)
        if self.kind == "vl":
            return self.cont.launch_force(self.cfg.pattern, self.cfg.newton3, self.energy,
                                          self.stats_t, self.ev_t)
        if self.kind == "lc":
            return self.cont.launch_force(self.cfg.pattern, self.energy, self.stats_t, self.ev_t,
                                          self.trav, self.cfg.newton3)
        return self.cont.launch_force(self.energy, self.stats_t, self.ev_t, pattern=self.cfg.pattern)

    @property
    def launches_per_step(self) -> int:
        # force kernel + refresh gathers (owned rows; images / ghost rows);
        # overlapped bricks: two force launches (interior, boundary), the
        # ghost pack kernels are counted apart
        if self.overlapped:
            return 2 + 2
        if self.kind == "vl":
            # segmented lists: one refresh launch (owned rows + derived images
            # + displacement) and the force kernel; a ghost layer adds its gather
            return 2 if self.dec is None else 3
        if self.kind == "lc":
            return 1 + 2
        return 1


def build_phase(cfg, w, args, torch, N, dec=None):
    import paper_2512_03565_b200 as B
    params = params_for(cfg, w)
    pos = w.positions if isinstance(w.positions, torch.Tensor) else torch.as_tensor(w.positions)
    pos = pos.to("cuda", torch.float64)
    if dec is None:
        box = B.SimulationBox.cube(w.box_length, periodic=True)
        buf = B.ParticleBuffer.from_positions(pos.cpu().numpy(), device="cuda")
        cont = B.make_container(cfg.container, box, params, cluster_size=args.vector_width)
        cont.rebuild(buf)
        cont.refresh(buf)
        phase = Phase(cfg, cont, buf, args, torch, N)
    else:
        box = dec.local_box()
        ids = torch.arange(pos.shape[0], dtype=torch.float64, device="cuda")
        rows = torch.cat([pos, ids[:, None]], dim=1)
        rows = dec.migrate(rows)
        owned_rows = rows.contiguous()
        ghost_rows = dec.plan(owned_rows)
        buf = B.ParticleBuffer.from_positions(owned_rows[:, :3].cpu().numpy(), device="cuda")
        owned_rows = torch.cat([torch.stack([buf.pos_x, buf.pos_y, buf.pos_z], 1),
                                owned_rows[:, 3:]], 1)
        ghosts = B.ParticleBuffer.from_positions(ghost_rows[:, :3].cpu().numpy(), device="cuda")
        cont = B.make_container(cfg.container, box, params, cluster_size=args.vector_width)
        cont.rebuild(buf, ghosts)
        cont.refresh(buf, ghosts)
        phase = Phase(cfg, cont, buf, args, torch, N, dec=dec, owned_rows=owned_rows)
        phase.ghosts = ghosts
    if cfg.container.value == "vl":
        geo = cont.vl_stats(cfg.newton3, cfg.pattern, args.vector_width)
    elif cfg.container.value == "lc":
        geo = cont._lc_stats(B.traversals.traversal_code(cfg.traversal), cfg.newton3,
                             cfg.pattern, args.vector_width)
    else:
        geo = cont.vcl_stats(cfg.newton3, cfg.pattern, args.vector_width)
    return phase, cont, buf, box, params, geo


def committed_traffic(label, workload):
    """DRAM bytes per launch of this configuration's force kernel on this
    workload, from the committed ncu capture (profiles/traffic.json), else
    None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh).get(workload, {}).get(label, {}).get("bytes")
    except (OSError, ValueError, AttributeError):
        return None


def algorithmic_bytes(cfg, cont, stats, n):
    """Bytes one force launch must move: positions (x, y, z: 24 B per particle
    and image; 32 B pos4 records where the kernel gathers those), forces
    (24 B per owned particle) and, for Verlet lists, one index per list entry
    at the width the kernel reads (segmented lists: 2 B per slot of the
    segments the launch runs; round-1 staged lists: 2 B per useful
    interaction; else 4 B)."""
    images = getattr(cont, "n_halo", 0) or 0
    vls = cont._vls_for(cfg.pattern, cfg.newton3) if hasattr(cont, "_vls_for") else None
    if vls is not None:
        ng = vls["plan"]["ngroups"]
        segc = vls["segc"][: 8 * ng].view(-1, 2).long()
        chunks = int(segc[:, 0].sum()) + (int(segc[:, 1].sum()) if cont._vls_outer() else 0)
        return int(24 * (n + images) + 24 * n + 2 * chunks * 8 * 32)
    staged = getattr(cont, "_staging", None)
    stg = next(iter(staged.values())) if staged else None
    pos_b = 24 if (stg is not None or getattr(cont, "use_soa", False)) else 32
    b = pos_b * (n + images) + 24 * n
    if cfg.container.value == "vl":
        b += (stg[4] // 8 if stg is not None else 4) * stats.useful_interactions
    return int(b)


def finish(cfg, st, geo, cont):
    """KernelStats in the reference's pair convention for the kernel that ran
    (the container knows whether Newton3 pairs were seen from both sides)."""
    from paper_2512_03565_b200 import KernelStats
    from paper_2512_03565_b200.containers import LinkedCellsContainer
    from paper_2512_03565_b200.traversals import traversal_code
    if cfg.container.value == "lc":
        once = cont.uses_colored_n3(traversal_code(cfg.traversal), cfg.newton3)
        return LinkedCellsContainer.finish_stats(st, cfg.newton3 and not once, *geo)
    if cfg.container.value == "vcl":
        return LinkedCellsContainer.finish_stats(st, cfg.newton3, *geo)
    return KernelStats(geo[0], geo[1], geo[2], cont.pair_count(st, cfg.newton3))


def time_steps(phase, steps, flush, torch):
    """Per-step CUDA events around (refresh + force) and around the force
    kernel alone; the L2 is flushed (untimed) before every step."""
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    for k in range(steps):
        flush.fill_(k & 0xFF)
        ev[k][0].record()
        phase.refresh()
        ev[k][1].record()
        phase.launch()
        ev[k][2].record()
    torch.cuda.synchronize()
    step = [a.elapsed_time(c) * 1e-3 for a, b, c in ev]
    kern = [b.elapsed_time(c) * 1e-3 for a, b, c in ev]
    return step, kern


def time_rebuild(phase, torch, reps: int = 2):
    """Neighbour-structure maintenance of a Verlet-list phase, measured: the
    container rebuild (binning, images) + list build, wall clock between two
    synchronisations (host work and reads included), best of ``reps``; and
    the list build alone in CUDA events.  None for containers rebuilt inside
    every step (LC re-bins its images in refresh)."""
    if phase.kind != "vl":
        return None
    cont = phase.cont
    wall, gpu = [], []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if phase.dec is None:
            cont.rebuild(phase.buf)
        else:
            cont.rebuild(phase.buf, phase.ghosts)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        cont.ensure_lists(phase.cfg.pattern, phase.cfg.newton3)
        e1.record()
        torch.cuda.synchronize()
        wall.append(time.perf_counter() - t0)
        gpu.append(e0.elapsed_time(e1) * 1e-3)
    phase.refresh()
    return min(wall), min(gpu)


def cpu_baseline_lc(w, cfg, params, threads):
    from oracle import oracle as O
    span = w.box_length
    pos = w.positions.cpu().numpy() if hasattr(w.positions, "cpu") else w.positions
    trav = cfg.traversal.value
    n3 = cfg.newton3
    if cfg.container.value != "lc":
        # the reference has no Verlet lists: its own algorithm for
        # the same pairs is linked cells with cell size = cutoff
        from paper_2512_03565_b200 import LJParams
        trav, n3 = "lc_c01", False
        params = LJParams(cutoff=params.cutoff, skin=0.0)
    if threads > 1 and n3:
        trav, n3 = "lc_c01", False       # the parallel baseline sweeps Newton3-off units
    t0 = time.perf_counter()
    h = O.PreparedLC(pos, np.zeros(3), np.full(3, span), [True] * 3, params, trav, n3,
                     cfg.pattern.value, 8, omp=threads > 1)
    prep = time.perf_counter() - t0
    return h, prep, trav, n3


def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_2512_03565_b200 as B
    from paper_2512_03565_b200 import _native as N

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # LMD_DEVICE / LMD_DIST_BACKEND=gloo: run the multi-rank path on one GPU
    # (host-staged communication) to exercise it where only one GPU exists
    local = int(os.environ.get("LMD_DEVICE", local))
    backend = os.environ.get("LMD_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cfg = B.Configuration.parse(args.config)
    dec = None
    if world > 1:
        # weak scaling: every rank's brick is the N=1 box (same density), the
        # global periodic box stacks the bricks; one NCCL ghost exchange per step
        from paper_2512_03565_b200.decomposition import BrickDecomposition, brick_grid
        grid = brick_grid(world)
        if scaling_of(args) == "strong":
            # strong scaling: every rank generates the same global system
            # (seeded) and keeps the particles of its brick
            w = make_workload(args, "cuda", 42)
            params0 = params_for(cfg, w)
            dec = BrickDecomposition(np.zeros(3), np.full(3, w.box_length),
                                     params0.interaction_length, rank, world, grid=grid)
            pos = torch.as_tensor(w.positions).to("cuda", torch.float64)
            w.positions = pos[dec.owner_of(pos) == rank].contiguous()
        else:
            # weak scaling: every rank's brick is the N=1 box (same density), the
            # global periodic box stacks the bricks
            w = make_workload(args, "cuda", 42 + rank)
            Lb = w.box_length
            c = (rank % grid[0], (rank // grid[0]) % grid[1], rank // (grid[0] * grid[1]))
            w.positions = (torch.as_tensor(w.positions).to("cuda", torch.float64)
                           + torch.tensor([c[0] * Lb, c[1] * Lb, c[2] * Lb],
                                          dtype=torch.float64, device="cuda"))
            params0 = params_for(cfg, w)
            dec = BrickDecomposition(np.zeros(3), np.array(grid, dtype=np.float64) * Lb,
                                     params0.interaction_length, rank, world, grid=grid)
    else:
        w = make_workload(args, "cuda", 42)
    dec_error = None
    try:
        phase, cont, buf, box, params, geo = build_phase(cfg, w, args, torch, N, dec)
    except Exception as exc:  # the decomposed path could not be built: say so, run replicas
        if dec is None:
            raise
        dec_error = f"{type(exc).__name__}: {exc}"[:300]
        print(f"[bench] brick decomposition failed on rank {rank}: {dec_error}", file=sys.stderr)
        dec = None
        w = make_workload(args, "cuda", 42 + rank)
        phase, cont, buf, box, params, geo = build_phase(cfg, w, args, torch, N, None)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    peak = fp64_peak_tflops(torch, N)

    for _ in range(max(args.warmup, 3)):
        flush.fill_(1)
        phase.refresh()
        phase.launch()
    torch.cuda.synchronize()
    st = N.read_stats(phase.stats_t)
    stats = finish(cfg, st, geo, cont)
    pairs = stats.pair_interactions
    n_local = int(buf.pos_x.shape[0])

    sampler = ClockSampler(local)
    sampler.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    per_step, per_kernel = time_steps(phase, args.steps, flush, torch)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    t_step = sum(per_step)
    t_kern = sum(per_kernel)
    st2 = N.read_stats(phase.stats_t)
    assert st2.pair_interactions == st.pair_interactions and not st2.overlap
    t_max = t_step
    total_pairs = pairs
    if world > 1:
        t = torch.tensor([t_step], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
        p = torch.tensor([pairs], dtype=torch.int64, device="cuda")
        dist.all_reduce(p)
        total_pairs = int(p.item())

    value = total_pairs * args.steps / t_max
    avg_launch = t_kern / args.steps
    # segmented lists: the timed steps run the inner segment alone (the state
    # is static, so no particle has moved delta / 2 -- as in the BASELINE MD
    # runs, where dt = 0.001 and a rebuild every 10 steps keep displacements
    # below it); the launch with both segments is timed beside it
    outer_ms = None
    if phase.kind == "vl" and cont._vls_for(cfg.pattern, cfg.newton3) is not None and dec is None:
        slot, cont._disp_slot = cont._disp_slot, -1     # no displacement record: both segments
        ts = []
        for k in range(5):
            flush.fill_(k)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            phase.launch()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        cont._disp_slot = slot
        st3 = N.read_stats(phase.stats_t)
        assert st3.pair_interactions == st.pair_interactions
        outer_ms = statistics.median(ts)
        phase.launch()
    maint = None
    rb = time_rebuild(phase, torch)
    if rb is not None:
        period = cont.rebuild_period
        step_s = t_max / args.steps
        maint = {"rebuild_and_lists_ms": rb[0] * 1e3, "list_build_gpu_ms": rb[1] * 1e3,
                 "rebuild_period": period,
                 "amortized_ms_per_step": (step_s + rb[0] / period) * 1e3,
                 "amortized_pairs_per_s": total_pairs / (step_s + rb[0] / period),
                 "note": "rank 0; outside the timed region: container rebuild (binning, "
                         "images) + list build, wall clock between synchronisations, "
                         "amortised over the rebuild period" +
                         ("; ghost migration/planning not included" if dec else "")}
    flops = pairs * FLOPS_PER_PAIR[cfg.newton3]
    achieved = flops / avg_launch / 1e12

    # ------------------------------------------------ e2e through the public API
    e2e = None
    if args.e2e_steps > 0 and world == 1:
        host = {k: np.ascontiguousarray(v) for k, v in
                zip(("pos_x", "pos_y", "pos_z"), w.positions.cpu().numpy().T)}
        n = len(host["pos_x"])

        class HostBuffer:
            pass

        hb = HostBuffer()
        for k, v in host.items():
            setattr(hb, k, torch.from_numpy(v).pin_memory())
        for k in ("vel_x", "vel_y", "vel_z", "old_force_x", "old_force_y", "old_force_z"):
            setattr(hb, k, None)
        for k in ("force_x", "force_y", "force_z"):
            setattr(hb, k, torch.zeros(n, dtype=torch.float64).pin_memory())
        hb.id = None
        hb.ownership = torch.zeros(n, dtype=torch.int8).pin_memory()
        B.force_phase(hb, box, params, cfg, args.vector_width)       # warm
        torch.cuda.synchronize()
        times = []
        for _ in range(args.e2e_steps):
            flush.fill_(3)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s_e2e = B.force_phase(hb, box, params, cfg, args.vector_width)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
            assert s_e2e.pair_interactions == pairs
        e2e = {"value": pairs * args.e2e_steps / sum(times), "unit": UNIT,
               "h2d_bytes_per_step": int(n * (3 * 8 + 1)),
               "d2h_bytes_per_step": int(n * 3 * 8),
               "steps": args.e2e_steps,
               "note": "force_phase() on pinned host SoA buffers: H2D positions, device "
                       "binning / images / group plan, the one-shot force path (candidate "
                       "walk + exact evaluation, no lists written: the container lives for "
                       "this call only), D2H forces"}
    elif args.e2e_steps > 0 and dec is not None:
        # every rank: its brick's particles in pinned host buffers ->
        # force_phase_bricks (H2D, ghost planning + exchange, binning, lists,
        # kernel, D2H); time = max over ranks, pairs = sum over ranks
        n = n_local

        class HostBuffer:
            pass

        hb = HostBuffer()
        for k in ("pos_x", "pos_y", "pos_z"):
            setattr(hb, k, getattr(buf, k).cpu().pin_memory())
        for k in ("vel_x", "vel_y", "vel_z", "old_force_x", "old_force_y", "old_force_z"):
            setattr(hb, k, None)
        for k in ("force_x", "force_y", "force_z"):
            setattr(hb, k, torch.zeros(n, dtype=torch.float64).pin_memory())
        hb.id = None
        hb.ownership = torch.zeros(n, dtype=torch.int8).pin_memory()
        B.force_phase_bricks(hb, dec, params, cfg, args.vector_width)       # warm
        torch.cuda.synchronize()
        t_sum, p_e2e = 0.0, 0
        for _ in range(args.e2e_steps):
            flush.fill_(3)
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            s_e2e = B.force_phase_bricks(hb, dec, params, cfg, args.vector_width)
            torch.cuda.synchronize()
            t_sum += time.perf_counter() - t0
            p_e2e = s_e2e.pair_interactions
        tt = torch.tensor([t_sum], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        pp = torch.tensor([p_e2e], dtype=torch.int64, device="cuda")
        dist.all_reduce(pp)
        assert int(pp.item()) == total_pairs, (int(pp.item()), total_pairs)
        hh = torch.tensor([n * (3 * 8 + 1), n * 3 * 8], dtype=torch.int64, device="cuda")
        dist.all_reduce(hh)
        e2e = {"value": int(pp.item()) * args.e2e_steps / float(tt.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(hh[0].item()), "d2h_bytes_per_step": int(hh[1].item()),
               "steps": args.e2e_steps,
               "note": "force_phase_bricks() on every rank's pinned host SoA buffers: H2D "
                       "positions, ghost planning + exchange, device binning / neighbour "
                       "build, force kernel, D2H forces; max over ranks"}
    elif args.e2e_steps > 0:
        e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
               "note": "replicas: e2e is measured at N=1 (force_phase is single-domain)"}

    # ------------------------------------------------------------ CPU baseline
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            h, prep, trav, n3 = cpu_baseline_lc(w, cfg, params, 1)
            t0 = time.perf_counter()
            _, ost = h.execute(1)
            dt = time.perf_counter() - t0
            h.close()
            cpu = {"value": ost.pair_interactions / dt, "unit": UNIT, "cores": 1, "kind": "port",
                   "sample": f"one full force phase of the same {w.n}-particle workload, "
                             f"{trav} newton3={n3}, oracle/lj_oracle.c (bitwise restatement of "
                             f"the reference's numba sweep), 1 thread; prepare {prep:.1f}s "
                             f"untimed, sweep {dt:.2f}s",
                   "cpu_pairs_match_gpu": ost.pair_interactions == pairs}
        except Exception as exc:  # pragma: no cover - reported, not fatal
            cpu = {"value": None, "error": repr(exc)}

    if args.sweep and rank == 0 and world == 1:
        sweep(args, w, torch, N, flush)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_max / args.steps * 1e3,
            "higher_is_better": True, "scaling": scaling_of(args), "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "particles_rank0": n_local,
                       "box_length_per_gpu": w.box_length, "cutoff": w.cutoff,
                       "skin": params.skin, "configuration": cfg.label,
                       "vector_width": args.vector_width,
                       "pairs_per_step": total_pairs, "pairs_per_step_rank0": pairs,
                       "useful_interactions_rank0": stats.useful_interactions,
                       "candidate_efficiency": pairs / max(stats.useful_interactions, 1),
                       "step": "refresh (positions -> cell order, images/ghosts) + force "
                               "kernel" + (f" + {backend} ghost exchange" if world > 1 else ""),
                       "kernel_ms_rank0": avg_launch * 1e3,
                       "list_segments": (None if outer_ms is None else
                                         f"inner (rc + {cont.inner_skin}) alone in the timed steps: "
                                         "no particle has moved half of it since the build, "
                                         "decided on the device per launch; "
                                         "kernel_ms_both_segments_rank0 = the same launch "
                                         "running the outer segment (up to rc + skin) too"),
                       "kernel_ms_both_segments_rank0": outer_ms,
                       "l2": "inputs larger than L2 (1.8 GB state at c4) and L2 flushed "
                             "(256 MiB write) before every timed step",
                       "parallelism": (f"bricks {dec.grid}, {backend} P2P ghost exchange"
                                       if dec else ("replicas (decomposition failed: "
                                                    f"{dec_error})" if dec_error
                                                    else ("replicas" if world > 1
                                                          else "single"))),
                       "inputs": w.note},
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak,
                         "flops_per_pair": FLOPS_PER_PAIR[cfg.newton3],
                         "kernel": "force kernel alone (CUDA events on its stream)",
                         "peak_source": "measured in this run: lmd_dfma_burn (DFMA, 2 flop)",
                         "traffic": committed_traffic(cfg.label, w.name),
                         "algorithmic_bytes": algorithmic_bytes(cfg, cont, stats, n_local),
                         "hbm_gbs_achieved": algorithmic_bytes(cfg, cont, stats, n_local)
                         / avg_launch / 1e9},
            "list_maintenance": maint,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": args.steps * phase.launches_per_step,
            "clocks": clocks,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def sweep(args, w, torch, N, flush):
    import paper_2512_03565_b200 as B
    rows = []
    labels = [c.label for c in B.enumerate_search_space(
        [B.ContainerKind.LINKED_CELLS, B.ContainerKind.VERLET_LISTS,
         B.ContainerKind.VERLET_CLUSTER_LISTS],
        [B.TraversalKind.LC_C01, B.TraversalKind.LC_C08, B.TraversalKind.LC_C18,
         B.TraversalKind.VL, B.TraversalKind.VCL],
        [False, True], list(B.PATTERN_ORDER))]
    for label in labels:
        cfg = B.Configuration.parse(label)
        phase, cont, *_ = build_phase(cfg, w, args, torch, N)
        for _ in range(3):
            phase.launch()
        _, t = time_steps(phase, 5, flush, torch)
        st = N.read_stats(phase.stats_t)
        pairs = finish(cfg, st, (0, 0, 0), cont).pair_interactions
        row = {"config": label, "ms": min(t) * 1e3, "pairs": pairs,
               "pairs_per_s": pairs / min(t)}
        if hasattr(cont, "gpu_lane_stats") and not (cfg.container.value == "lc" and
                                                     cont.uses_colored_n3(phase.trav,
                                                                          cfg.newton3)):
            try:
                steps, active = (cont.gpu_lane_stats(cfg.pattern, phase.trav, cfg.newton3)
                                 if cfg.container.value == "lc"
                                 else cont.gpu_lane_stats(cfg.pattern, cfg.newton3))
                row.update({"gpu_lane_steps": steps, "gpu_active_lanes": active,
                            "gpu_lane_utilisation": active / max(steps, 1),
                            # N3 runs evaluate ordered pairs; the reported count is Newton3's
                            "gpu_pair_lanes_fraction": (None if cfg.newton3
                                                        else pairs / max(steps, 1))})
            except Exception as exc:  # noqa: BLE001 -- reported, not fatal
                row["gpu_lane_stats_error"] = str(exc)[:200]
        rows.append(row)
        print(f"sweep {label:36s} {min(t) * 1e3:8.3f} ms  {pairs / min(t):.3e} pairs/s",
              file=sys.stderr)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "sweep.json"), "w") as fh:
        json.dump(rows, fh, indent=1)


def run_reference(args):
    """The reference algorithm (oracle port of lanemd's execute_packed, all host
    threads) on this arm's workload/config/metric; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch

    import paper_2512_03565_b200 as B
    from oracle import oracle as O
    cfg = B.Configuration.parse(args.config)
    device = "cuda" if torch.cuda.is_available() else "cpu"
    w = make_workload(args, device, 42)
    params = params_for(cfg, w)
    threads = O.max_threads()
    h, prep, trav, n3 = cpu_baseline_lc(w, cfg, params, threads)
    for _ in range(min(max(args.warmup, 1), 2)):   # a CPU sweep needs no long warm-up
        h.execute(threads)
    times = []
    pairs = None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _, st = h.execute(threads)
        times.append(time.perf_counter() - t0)
        pairs = st.pair_interactions
    h.close()
    value = pairs * args.steps / sum(times)
    sample = (f"{args.steps} force phases (execute only) of {w.name}, {trav} newton3={n3}, "
              f"oracle/lj_oracle.c with OpenMP over i-cell unit groups (bitwise the "
              f"sequential reference sweep); prepare {prep:.1f}s untimed")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sum(times) / args.steps * 1e3, "higher_is_better": True,
            "scaling": scaling_of(args), "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": w.name, "configuration": cfg.label,
                       "executed": f"lc,{trav},{str(n3).lower()}", "pairs_per_step": pairs},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
