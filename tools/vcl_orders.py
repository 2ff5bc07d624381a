"""VCL interaction orders as warp mappings (lmd_force_vcl_order) vs the
packed stream kernel, on BASELINE config 3 (2M droplet, rc 3.0, skin 0.3):
force-kernel time per order and cluster size (CUDA events, best of 5),
pair counts, max force difference.  python tools/vcl_orders.py [n]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import _native as N, workloads  # noqa: E402

ORDERS = ("one_by_v", "v_by_one", "two_by_half", "half_by_two")


def timed(cont, pattern, reps=5):
    st = N.new_stats("cuda")
    for _ in range(2):
        cont.launch_force(False, st, pattern=pattern)
    best = 1e9
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        cont.launch_force(False, st, pattern=pattern)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    s = N.read_stats(st)
    f = torch.stack([cont._fx, cont._fy, cont._fz], 1).clone()
    return best, int(s.pair_interactions), f


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
    torch.cuda.set_device(0)
    w = workloads.config3(n=n, device="cuda")
    pos = w.positions.cpu().numpy()
    box = B.SimulationBox.cube(w.box_length, periodic=True)
    params = B.LJParams(cutoff=w.cutoff, skin=0.3)
    out = {"workload": w.name, "rows": []}
    for m in (4, 8, 32):
        buf = B.ParticleBuffer.from_positions(pos, device="cuda")
        cont = B.make_container("vcl", box, params, cluster_size=m)
        cont.rebuild(buf)
        cont.refresh(buf)
        cont.order_kernels = False
        t_ref, p_ref, f_ref = timed(cont, None)
        out["rows"].append({"M": m, "kernel": "stream", "ms": t_ref, "pairs": p_ref,
                            "pairs_per_s": p_ref / (t_ref * 1e-3)})
        print(f"M={m:2d} stream      {t_ref:8.3f} ms {p_ref / t_ref / 1e-3:.3e} pairs/s",
              flush=True)
        cont.order_kernels = "strict"     # the lane-template kernel for every order
        for o in ORDERS:
            t, p, f = timed(cont, o)
            scale = torch.clamp(f_ref.abs().max(dim=1).values, min=1.0)
            err = float(((f - f_ref).abs().max(dim=1).values / scale).max())
            out["rows"].append({"M": m, "kernel": o, "ms": t, "pairs": p, "pairs_equal": p == p_ref,
                                "pairs_per_s": p / (t * 1e-3), "max_rel_diff_vs_stream": err})
            print(f"M={m:2d} {o:11s} {t:8.3f} ms {p / t / 1e-3:.3e} pairs/s  eq={p == p_ref} "
                  f"err={err:.1e}", flush=True)
        del cont, buf
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
