"""Segmented staged lists (csrc/vls.cu) vs the round-1 staged path on one
workload: force kernel time (CUDA events, L2 flushed), pairs, max force
difference, list build time.  python tools/vls_compare.py [c2|c4]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import _native as N, workloads  # noqa: E402


def timed(cont, buf, reps=10):
    st = N.new_stats("cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        cont.refresh(buf)
        cont.launch_force("v_by_one", False, stats_t=st)
    ts = []
    for k in range(reps):
        flush.fill_(k)
        cont.refresh(buf)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        cont.launch_force("v_by_one", False, stats_t=st)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    s = N.read_stats(st)
    cont.collect_forces(buf)
    return min(ts), sorted(ts)[len(ts) // 2], s.pair_interactions, buf.forces().clone()


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "c2"
    torch.cuda.set_device(0)
    w = workloads.config4(256) if which == "c4" else workloads.config2(0.8, n=1_000_000, device="cuda")
    pos = w.positions.cpu().numpy() if hasattr(w.positions, "cpu") else w.positions
    box = B.SimulationBox.cube(w.box_length, periodic=True)
    params = B.LJParams(cutoff=2.5, skin=0.3)
    out = {"workload": w.name}
    forces = {}
    for label, seg, inner, pers in (("round1_staged", False, 0.1, False),
                                    ("vls_inner0.1", True, 0.1, False),
                                    ("vls_outer_only", True, 0.3, False),
                                    ("vls_inner0.05", True, 0.05, False)):
        buf = B.ParticleBuffer.from_positions(pos, device="cuda")
        cont = B.make_container("vl", box, params)
        cont.segmented = seg
        cont.inner_skin = inner
        cont.rebuild(buf)
        cont.refresh(buf)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cont.ensure_lists("v_by_one", False)
        torch.cuda.synchronize()
        tb = time.perf_counter() - t0
        # second build timing (warm)
        cont.rebuild(buf)
        cont.refresh(buf)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cont.ensure_lists("v_by_one", False)
        torch.cuda.synchronize()
        tb2 = time.perf_counter() - t0
        tmin, tmed, pairs, f = timed(cont, buf)
        forces[label] = f
        vls = cont._vls_for("v_by_one", False)
        row = {"force_ms_min": tmin, "force_ms_med": tmed, "pairs": pairs,
               "pairs_per_s": pairs / (tmin * 1e-3), "list_build_s": tb2, "first_build_s": tb,
               "segmented_used": vls is not None}
        if vls is not None:
            ng = vls["plan"]["ngroups"]
            segc = vls["segc"][: 8 * ng].view(-1, 2).long()
            row.update({"groups": ng, "rows": vls["plan"]["rows"],
                        "chunks_inner": int(segc[:, 0].sum()), "chunks_outer": int(segc[:, 1].sum()),
                        "cap_chunks": vls["cap_chunks"]})
        out[label] = row
        print(label, json.dumps(row), flush=True)
        del cont, buf
        torch.cuda.empty_cache()
    ref = forces["round1_staged"]
    scale = torch.clamp(ref.abs().max(dim=1).values, min=1.0)
    for k, f in forces.items():
        out[k]["max_rel_diff_vs_round1"] = float(((f - ref).abs().max(dim=1).values / scale).max())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
