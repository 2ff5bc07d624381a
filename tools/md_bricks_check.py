"""Brick-decomposed MD (run_md_bricks) against the single-domain MD loop on
the same system: per-step global pair counts must be equal and the final
positions (minimum image, matched by id) equal to rounding.

    torchrun --nproc-per-node 2 tools/md_bricks_check.py [--config vl,vl,false,v_by_one]

With LMD_DIST_BACKEND=gloo LMD_DEVICE=0 all ranks share one GPU (host-staged
exchange).  Rank 0 prints one JSON line."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import workloads  # noqa: E402
from paper_2512_03565_b200.decomposition import BrickDecomposition, brick_grid  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="vl,vl,false,v_by_one")
    ap.add_argument("--particles", type=int, default=200_000)
    ap.add_argument("--rho", type=float, default=0.8)
    ap.add_argument("--steps", type=int, default=25)
    ap.add_argument("--single", type=int, default=1, help="also run the single-domain check")
    ap.add_argument("--tune", type=int, default=0,
                    help="tune over VL / LC x two orders instead of --config (no single check)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LMD_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    backend = os.environ.get("LMD_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cfg = B.Configuration.parse(args.config)
    skin = 0.0 if cfg.container is B.ContainerKind.LINKED_CELLS else 0.3
    params = B.LJParams(cutoff=2.5, skin=skin, dt=0.001)
    w = workloads.config2(args.rho, n=args.particles, device="cuda")
    L = w.box_length
    box = B.SimulationBox.cube(L, periodic=True)
    pos = w.positions.cpu().numpy()
    vel = np.asarray(w.velocities.cpu() if hasattr(w.velocities, "cpu") else w.velocities)
    full = B.ParticleBuffer.from_positions(pos, device="cuda")
    v = torch.as_tensor(vel).to("cuda", torch.float64)
    full.vel_x.copy_(v[:, 0]); full.vel_y.copy_(v[:, 1]); full.vel_z.copy_(v[:, 2])
    B.force_phase(full, box, params, cfg, 8)          # forces for the first half step
    dec = BrickDecomposition(np.zeros(3), np.full(3, L), params.interaction_length, rank, world,
                             grid=brick_grid(world))
    mine = dec.owner_of(full.positions()) == rank
    idx = torch.nonzero(mine).flatten()
    local_buf = B.ParticleBuffer.empty(int(idx.numel()), device="cuda")
    for f in ("pos_x", "pos_y", "pos_z", "vel_x", "vel_y", "vel_z", "force_x", "force_y",
              "force_z", "old_force_x", "old_force_y", "old_force_z"):
        getattr(local_buf, f).copy_(getattr(full, f)[idx])
    local_buf.id.copy_(full.id[idx])
    if args.tune:
        space = [B.Configuration.parse(x) for x in ("vl,vl,false,v_by_one", "vl,vl,false,half_by_two",
                                                    "lc,lc_c01,false,v_by_one",
                                                    "lc,lc_c18,true,half_by_two")]
        owned, summ = B.run_md_bricks(local_buf, dec, B.LJParams(cutoff=2.5, skin=0.3, dt=0.001),
                                      args.steps, 8, configurations=space,
                                      policy=B.TuningPolicy(2, 40, "mean", "time"))
        args.single = 0
    else:
        owned, summ = B.run_md_bricks(local_buf, dec, params, args.steps, 8, config=cfg,
                                      rebuild_period=10 if skin else None)
    mine_rows = torch.cat([owned.id.to(torch.float64)[:, None], owned.positions()], 1).cpu()
    gathered = [None] * world
    sels = [None] * world
    if world > 1:
        dist.all_gather_object(gathered, mine_rows)
        dist.all_gather_object(sels, summ.phase_selections)
    else:
        gathered = [mine_rows]
        sels = [summ.phase_selections]
    if rank == 0:
        out = {"config": args.config, "ranks": world, "grid": list(dec.grid),
               "particles": summ.particles_global, "steps": args.steps,
               "rebuilds": summ.rebuilds, "particle_steps_per_s": summ.particle_steps_per_s,
               "pairs_per_step": summ.pairs_per_step[:5] + ["..."] + summ.pairs_per_step[-2:],
               "phase_selections": summ.phase_selections,
               "selections_agree": all(x == sels[0] for x in sels)}
        if args.single:
            t0 = time.perf_counter()
            recs, _ = B.run_md(full, box, params, args.steps, 8, fixed_config=cfg,
                               rebuild_period=10 if skin else None, wrap="at_rebuild")
            single_pairs = [r.pair_interactions for r in recs]
            rows = torch.cat(gathered)
            order = torch.argsort(rows[:, 0])
            rows = rows[order]
            ref = full.positions().cpu()[rows[:, 0].long()]
            d = rows[:, 1:] - ref
            d -= L * torch.round(d / L)
            out.update({"single_pairs_equal": single_pairs == summ.pairs_per_step,
                        "max_position_diff": float(d.abs().max()),
                        "ids_complete": bool(torch.equal(rows[:, 0].long(),
                                                         torch.arange(len(rows)))),
                        "single_domain_s": time.perf_counter() - t0})
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
