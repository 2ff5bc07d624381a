"""Segmented Verlet-list build + force launches on a C4-like lattice (side^3
particles, default 160), with the bank-ordered and the plain entry order --
the target of ncu captures of vls_build_kernel / vls_force_kernel.
    python tools/vls_build_profile.py [side] [bank: 0 | -1 | both]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import _native as N, workloads  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 160
which = sys.argv[2] if len(sys.argv) > 2 else "both"
banks = (0, -1) if which == "both" else (int(which),)
torch.cuda.set_device(0)
w = workloads.config4(side)
pos = w.positions.cpu().numpy() if hasattr(w.positions, "cpu") else w.positions
box = B.SimulationBox.cube(w.box_length, periodic=True)
params = B.LJParams(cutoff=2.5, skin=0.3)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ref = None
for bank in banks:
    buf = B.ParticleBuffer.from_positions(pos, device="cuda")
    cont = B.make_container("vl", box, params)
    cont.bank_rounds = bank
    st = N.new_stats("cuda")
    for rep in range(3):
        cont.rebuild(buf)
        cont.refresh(buf)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record()
        cont.ensure_lists("v_by_one", False)
        e[1].record()
        flush.fill_(rep)
        e[2].record()
        cont.launch_force("v_by_one", False, stats_t=st)
        e[3].record()
        torch.cuda.synchronize()
        inner = e[2].elapsed_time(e[3])
        slot, cont._disp_slot = cont._disp_slot, -1     # both segments
        flush.fill_(rep)
        e[2].record()
        cont.launch_force("v_by_one", False, stats_t=st)
        e[3].record()
        torch.cuda.synchronize()
        cont._disp_slot = slot
        print(f"side {side} bank {bank}: lists {e[0].elapsed_time(e[1]):.3f} ms, force inner "
              f"{inner:.3f} ms, both segments {e[2].elapsed_time(e[3]):.3f} ms, "
              f"pairs {N.read_stats(st).pair_interactions}", flush=True)
    cont.collect_forces(buf)
    f = buf.forces().clone()
    if ref is None:
        ref = f
    else:
        scale = float(ref.abs().max())
        print("max force difference between the orders / max |F|:",
              float((f - ref).abs().max()) / scale)
    vls = cont._vls_for("v_by_one", False)
    print("cap_chunks", vls["cap_chunks"], "next cap_ent", cont._vls_cap, "rows", vls["plan"]["rows"],
          "info", vls["plan"]["info"].tolist())
    del cont, buf
    torch.cuda.empty_cache()

# the list-free one-shot kernel (force_phase's path) on the same state
buf = B.ParticleBuffer.from_positions(pos, device="cuda")
for rep in range(3):
    cont = B.make_container("vl", box, params)
    cont.rebuild(buf)
    cont.refresh(buf)
    torch.cuda.synchronize()
    e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
    e0.record()
    st1 = cont.compute_forces_once("vl", False, "v_by_one", 8)
    e1.record()
    torch.cuda.synchronize()
    print(f"side {side} one-shot (plan + list-free kernel + statistics): "
          f"{e0.elapsed_time(e1):.3f} ms, pairs {st1.pair_interactions}", flush=True)
cont.collect_forces(buf)
if ref is not None:
    print("max force difference one-shot vs lists / max |F|:",
          float((buf.forces() - ref).abs().max()) / float(ref.abs().max()))
