"""Bank-aware Verlet-list entry order (csrc/vl.cu vl_bank_kernel) on the bench
workload: for each gather variant -- pos4 records in ascending order, SoA
gathers in ascending order, SoA gathers bank-scheduled with R proposal
rounds -- the force-kernel time (L2 flushed, CUDA events), the list build
time (incl. the schedule pass), the pair count, and the schedule quality
measured on the list itself: mean over fill steps of the summed per-half
largest bank-pair multiplicity (2 = conflict-free, the cost unit of the
64-bit gather, tools/bank_probe.cu) and the share of idle slots.  Also checks
that every lane keeps exactly its own entries (sorted per-lane multisets
equal).  One JSON line per variant."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import _native as N  # noqa: E402
from paper_2512_03565_b200 import workloads  # noqa: E402

rho = float(os.environ.get("RHO", "0.8"))
w = workloads.config2(rho, n=int(os.environ.get("N", "1000000")), device="cuda")
box = B.SimulationBox.cube(w.box_length, periodic=True)
buf = B.ParticleBuffer.from_positions(w.positions.cpu().numpy(), device="cuda")
cont = B.VerletListContainer(box, B.LJParams(cutoff=2.5, skin=0.3))
cont.rebuild(buf)
cont.refresh(buf)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
patterns = os.environ.get("PATTERNS", "v_by_one").split(",")
rounds = [int(r) for r in os.environ.get("ROUNDS", "0,2").split(",")]


def timed(fn, reps=6):
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts) * 1e3


def lanes_view(pat, newton3=False):
    """(ntiles, steps_cap, 32) view of the list plus per-tile step counts."""
    key = next(k for k in cont._lists if k[0] == pat.code)
    tile_off, kmax, nbr, total = cont._lists[key]
    stg = cont._staging.get(key)
    bits = stg[4] if stg else 32
    ntiles = int(N.load().lmd_vl_num_tiles(cont.n_owned, pat.code))
    b = pat.shape(32)[1]
    cap = total // (ntiles * 32)
    if bits == 16:
        u = nbr.view(torch.int16).long() & 0xFFFF
        u = torch.where(u == 0xFFFF, torch.full_like(u, -1), u)
        v = u[: ntiles * cap * 32].view(ntiles, cap // 8, 32, 8).permute(0, 1, 3, 2)
    else:
        v = nbr[: ntiles * cap * 32].view(ntiles, cap // 4, 32, 4).permute(0, 1, 3, 2)
    return v.reshape(ntiles, cap, 32), (kmax[:ntiles] // b).long(), cont.n_owned + cont.n_halo


def quality(v, steps, sentinel):
    tot_load = 0
    tot_steps = 0
    idle = 0
    slots = 0
    for a in range(0, v.shape[0], 2048):
        blk = v[a:a + 2048].long()
        st = steps[a:a + 2048]
        valid = torch.arange(blk.shape[1], device=blk.device)[None, :] < st[:, None]
        real = (blk >= 0) & (blk != sentinel)
        bank = torch.where(real, blk & 15, torch.full_like(blk, 16))
        oh = torch.nn.functional.one_hot(bank, 17)[..., :16]          # (t, s, 32, 16)
        m = oh[:, :, :16].sum(2).amax(-1) + oh[:, :, 16:].sum(2).amax(-1)
        tot_load += int((m * valid).sum())
        tot_steps += int(valid.sum())
        idle += int(((~real) & valid[:, :, None]).sum())
        slots += int(valid.sum()) * 32
    return tot_load / tot_steps, idle / slots


def lane_sorted(v, steps, sentinel):
    x = v.clone().long()
    x[(x < 0) | (x == sentinel)] = 1 << 40
    return torch.sort(x, dim=1).values


groups_env = [int(g) for g in os.environ.get("STAGE_GROUPS", "128,256,512").split(",")]
variants = ([("pos4", False, -1, 0), ("soa", True, -1, 0)]
            + [(f"soa_bank{r}", True, r, 0) for r in rounds]
            + [(f"staged{g}", True, -1, g) for g in groups_env]
            + [(f"staged{g}_bank{r}", True, r, g) for g in groups_env for r in rounds])
for pname in patterns:
    pat = B.PatternKind(pname)
    ref_sorted = None
    ref_f = None
    for gname, soa, r, grp in variants:
        cont.use_soa = soa
        cont.bank_rounds = r
        cont.staged_group = grp
        cont.rebuild(buf)
        cont.refresh(buf)
        torch.cuda.synchronize()
        tb = timed(lambda: (cont._lists.clear(), cont._list(pat, False)), reps=3)
        st = cont.launch_force(pat, False)
        us = timed(lambda: cont.launch_force(pat, False, stats_t=st))
        s = N.read_stats(st)
        v, steps, sentinel = lanes_view(pat)
        load, idle = quality(v, steps, sentinel)
        if grp:
            same = None
            stg = next(iter(cont._staging.values()))
            extra = {"smem_rows": stg[1], "groups_over_capacity": stg[3], "index_bits": stg[4]}
        else:
            srt = lane_sorted(v, steps, sentinel)
            if ref_sorted is None:
                ref_sorted = srt
            same = bool(torch.equal(srt, ref_sorted))
            extra = {}
        f = torch.stack([cont._fx, cont._fy, cont._fz])
        if ref_f is None:
            ref_f = f.clone()
        extra["max_force_diff"] = float((f - ref_f).abs().max())
        if grp and os.environ.get("DBG"):
            for dbg in (1, 2):
                cont.knobs = dbg << 8
                extra[f"dbg{dbg}_us"] = round(timed(lambda: cont.launch_force(pat, False, stats_t=st)), 1)
            cont.knobs = 0
        print(json.dumps({"pattern": pname, "gather": gname, "force_us": round(us, 1),
                          **extra,
                          "build_us": round(tb, 1), "pairs": s.pair_interactions,
                          "half_max_load_per_gather": round(load, 3), "idle_share": round(idle, 4),
                          "lane_entries_equal": same, "rho": rho}), flush=True)
