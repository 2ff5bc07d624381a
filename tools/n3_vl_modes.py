"""Verlet-list Newton3 modes on one workload (default BASELINE C4): force
kernel time, list-build time and counted pairs for Newton3 off, Newton3 by
the reference's pair bookkeeping on full lists (the default) and real half
lists with FP64 atomics on the j side (n3_mode="half_list").  L2 flushed
between launches.      python tools/n3_vl_modes.py [c4|c2]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import _native as N, workloads  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c4"
torch.cuda.set_device(0)
w = workloads.config4(256) if which == "c4" else workloads.config2(0.8, n=1_000_000, device="cuda")
pos = w.positions.cpu().numpy() if hasattr(w.positions, "cpu") else w.positions
box = B.SimulationBox.cube(w.box_length, periodic=True)
params = B.LJParams(cutoff=2.5, skin=0.3)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rows = []
ref = None
for label, n3, mode in (("newton3 off", False, "full_list"),
                        ("newton3 on, full lists + pair bookkeeping", True, "full_list"),
                        ("newton3 on, half lists + FP64 atomics", True, "half_list")):
    buf = B.ParticleBuffer.from_positions(pos, device="cuda")
    cont = B.make_container("vl", box, params)
    cont.n3_mode = mode
    cont.rebuild(buf)
    cont.refresh(buf)
    e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
    e0.record()
    cont.ensure_lists("v_by_one", n3)
    e1.record()
    torch.cuda.synchronize()
    build_ms = e0.elapsed_time(e1)
    st = N.new_stats("cuda")
    ts = []
    for k in range(6):
        flush.fill_(k)
        a, b = (torch.cuda.Event(enable_timing=True) for _ in range(2))
        a.record()
        cont.launch_force("v_by_one", n3, stats_t=st)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    pairs = cont.pair_count(N.read_stats(st), n3)
    cont.collect_forces(buf)
    f = buf.forces().clone()
    if ref is None:
        ref = f
    row = {"mode": label, "force_ms": min(ts[1:]), "lists_ms": build_ms, "counted_pairs": pairs,
           "segmented_kernel": cont._vls_for("v_by_one", n3) is not None,
           "max_force_diff_vs_n3_off": float((f - ref).abs().max() / ref.abs().max())}
    rows.append(row)
    print(json.dumps(row), flush=True)
    del cont, buf
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
with open(f"gpurun_out/n3_vl_modes_{which}.json", "w") as fh:
    json.dump({"workload": w.name, "rows": rows}, fh, indent=1)
