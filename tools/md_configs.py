"""Run the BASELINE MD configurations on one GPU and report particle-steps/s.

    python tools/md_configs.py --config 1            # 8,000 lattice, LC c08 N3, 1 + 10 steps
    python tools/md_configs.py --config 3 --steps 300 # droplet, VCL M in {4,8,32}, tuner / 100
    python tools/md_configs.py --config 5 --steps 400 # 8.4M gas, tuner / 200 over LC x VL
    python tools/md_configs.py --config 2             # 1M at rho 0.2/0.5/0.8: every order x
                                                      # {LC c01/c08/c18, VL} x Newton3, 100 steps
    python tools/md_configs.py --config 4             # 16.8M perturbed lattice, VL, 200 steps

Every step runs the whole velocity-Verlet step on the device (integrator,
boundaries, neighbour maintenance, images, force phase) through
``paper_2512_03565_b200.run_md``.  One JSON line per run.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--metric", default="iteration",
                    help="tuner metric: iteration (whole MD step), time (force phase), laneops")
    ap.add_argument("--rho", default="0.2,0.5,0.8")
    ap.add_argument("--rebuild-period", type=int, default=None,
                    help="configs 3-5: steps between forced rebuilds (default: the container's "
                         "10); a large value leaves the skin / 2 displacement rule alone "
                         "in charge")
    ap.add_argument("--vcl-stream", action="store_true",
                    help="config 3: the packed stream kernel (cluster-aligned M x 32/M "
                         "mapping) for every order instead of the order's lane template")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    if args.vcl_stream:
        from paper_2512_03565_b200.clusters import VerletClusterContainer
        VerletClusterContainer.ORDER_KERNELS = False
    if args.config == 2:
        return sweep_config2(args)
    t_gen = time.perf_counter()
    if args.config == 1:
        w = workloads.config1()
        params = B.LJParams(cutoff=2.5, skin=0.0, dt=0.001)
        fixed = B.Configuration.parse("lc,lc_c08,true,one_by_v")
        configs, interval, steps = None, None, args.steps or 10
    elif args.config == 3:
        w = workloads.config3(n=args.n or 2_000_000, device="cuda")
        params = B.LJParams(cutoff=3.0, skin=0.3, dt=0.001)
        fixed = None
        configs = B.enumerate_search_space([B.ContainerKind.VERLET_CLUSTER_LISTS],
                                           [B.TraversalKind.VCL], [False],
                                           [B.PatternKind.V_BY_ONE, B.PatternKind.HALF_BY_TWO],
                                           cluster_sizes=[4, 8, 32])
        interval, steps = 100, args.steps or 1000
    elif args.config == 4:
        w = workloads.config4(device="cuda")
        params = B.LJParams(cutoff=2.5, skin=0.3, dt=0.001)
        fixed = B.Configuration.parse("vl,vl,false,v_by_one")
        configs, interval, steps = None, None, args.steps or 200
    elif args.config == 5:
        w = workloads.config5(n=args.n or 8_388_608, device="cuda")
        params = B.LJParams(cutoff=2.5, skin=0.3, dt=0.001)
        fixed = None
        configs = B.enumerate_search_space([B.ContainerKind.LINKED_CELLS,
                                            B.ContainerKind.VERLET_LISTS],
                                           [B.TraversalKind.LC_C01, B.TraversalKind.VL],
                                           [False], [B.PatternKind.V_BY_ONE,
                                                     B.PatternKind.HALF_BY_TWO,
                                                     B.PatternKind.TWO_BY_HALF])
        interval, steps = 200, args.steps or 2000
    else:
        raise SystemExit("configs 1-5 only")
    t_gen = time.perf_counter() - t_gen
    box = B.SimulationBox.cube(w.box_length, periodic=True)
    pos = w.positions if isinstance(w.positions, torch.Tensor) else torch.as_tensor(w.positions)
    buf = B.ParticleBuffer.from_positions(pos.cpu().numpy(), device="cuda")
    v = torch.as_tensor(w.velocities).to("cuda", torch.float64)
    buf.vel_x.copy_(v[:, 0]); buf.vel_y.copy_(v[:, 1]); buf.vel_z.copy_(v[:, 2])
    seed_cfg = fixed or configs[0]
    B.force_phase(buf, box, params, seed_cfg, 8)            # forces for the first kick
    torch.cuda.synchronize()
    policy = None
    if configs:
        policy = B.TuningPolicy(1, interval, "mean", args.metric)
    records, summary = B.run_md(buf, box, params, steps, 8, configurations=configs,
                                fixed_config=fixed, policy=policy, metric=args.metric,
                                retune_drift=0.2 if configs else None,
                                rebuild_period=args.rebuild_period,
                                wrap="always" if args.config == 1 else "at_rebuild")
    torch.cuda.synchronize()
    pairs = sum(r.pair_interactions for r in records)
    out = {
        "config": args.config, "workload": w.name, "particles": len(buf), "steps": steps,
        "particle_steps_per_s": summary.particle_steps_per_s,
        "wall_s": summary.wall_time_s, "force_time_s": summary.force_time_s,
        "pair_interactions_per_s_force": pairs / max(summary.force_time_s, 1e-12),
        "pair_interactions_per_step_last": records[-1].pair_interactions,
        "phase_selections": summary.phase_selections, "retunes": summary.retunes,
        "initial_max_per_cell": summary.initial_max_per_cell,
        "final_max_per_cell": summary.final_max_per_cell,
        "generation_s": t_gen, "note": w.note,
        "tuning_iterations": sum(r.phase == "tuning" for r in records),
        "configs_seen": sorted({r.configuration.label for r in records}),
        "vcl_stream_kernel": bool(args.vcl_stream),
        "metric": args.metric, "rebuild_period": args.rebuild_period or "container default (10)",
        "rebuilds": summary.rebuilds,
    }
    per = {}
    for r in records:
        per.setdefault((r.phase, r.configuration.label), []).append(r.metric_value)
    out["mean_metric_ms"] = {f"{ph}:{lab}": round(sum(v) / len(v) * 1e-6, 4)
                             for (ph, lab), v in sorted(per.items())}
    if args.config == 1:
        out["pairs_per_step"] = [r.pair_interactions for r in records]
    print(json.dumps(out))


def sweep_config2(args):
    """BASELINE config 2: every interaction order x {linked cells (cell = rc),
    Verlet lists (skin 0.3, rebuilt every 10 steps)} x Newton3, 100 MD steps
    each, at each density; one JSON line per run."""
    steps = args.steps or 100
    for rho in [float(r) for r in args.rho.split(",")]:
        w = workloads.config2(rho, n=args.n or 1_000_000, device="cuda")
        box = B.SimulationBox.cube(w.box_length, periodic=True)
        pos0 = w.positions.cpu().numpy()
        v0 = torch.as_tensor(w.velocities).to("cuda", torch.float64)
        cfgs = B.enumerate_search_space(
            [B.ContainerKind.LINKED_CELLS, B.ContainerKind.VERLET_LISTS],
            [B.TraversalKind.LC_C01, B.TraversalKind.LC_C08, B.TraversalKind.LC_C18,
             B.TraversalKind.VL], [False, True], list(B.PATTERN_ORDER))
        for cfg in cfgs:
            skin = 0.0 if cfg.container is B.ContainerKind.LINKED_CELLS else 0.3
            params = B.LJParams(cutoff=2.5, skin=skin, dt=0.001)
            buf = B.ParticleBuffer.from_positions(pos0, device="cuda")
            buf.vel_x.copy_(v0[:, 0]); buf.vel_y.copy_(v0[:, 1]); buf.vel_z.copy_(v0[:, 2])
            B.force_phase(buf, box, params, cfg, 8)
            torch.cuda.synchronize()
            records, summary = B.run_md(buf, box, params, steps, 8, fixed_config=cfg,
                                        rebuild_period=10 if skin else None,
                                        wrap="at_rebuild")
            torch.cuda.synchronize()
            pairs = sum(r.pair_interactions for r in records)
            print(json.dumps({
                "config": 2, "rho": rho, "configuration": cfg.label, "particles": len(buf),
                "steps": steps, "particle_steps_per_s": summary.particle_steps_per_s,
                "wall_s": summary.wall_time_s, "force_time_s": summary.force_time_s,
                "pair_interactions_per_s_force": pairs / max(summary.force_time_s, 1e-12),
                "pair_interactions_per_s_wall": pairs / max(summary.wall_time_s, 1e-12),
                "pairs_per_step_last": records[-1].pair_interactions}), flush=True)


if __name__ == "__main__":
    main()
