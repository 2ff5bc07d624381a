"""One segmented Verlet-list build + a few force launches on a C4-like lattice
(side^3 particles, default 160) -- the target of ncu captures of
vls_build_kernel / vls_force_kernel.  python tools/vls_build_profile.py [side]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import _native as N, workloads  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 160
torch.cuda.set_device(0)
w = workloads.config4(side)
pos = w.positions.cpu().numpy() if hasattr(w.positions, "cpu") else w.positions
box = B.SimulationBox.cube(w.box_length, periodic=True)
params = B.LJParams(cutoff=2.5, skin=0.3)
buf = B.ParticleBuffer.from_positions(pos, device="cuda")
cont = B.make_container("vl", box, params)
st = N.new_stats("cuda")
for rep in range(3):
    cont.rebuild(buf)
    cont.refresh(buf)
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    cont.ensure_lists("v_by_one", False)
    e1.record()
    cont.launch_force("v_by_one", False, stats_t=st)
    e2.record()
    torch.cuda.synchronize()
    print(f"side {side}: lists {e0.elapsed_time(e1):.3f} ms, force {e1.elapsed_time(e2):.3f} ms, "
          f"pairs {N.read_stats(st).pair_interactions}", flush=True)
vls = cont._vls_for("v_by_one", False)
print("cap_chunks", vls["cap_chunks"], "next cap_ent", cont._vls_cap, "rows", vls["plan"]["rows"],
      "build smem", int(N.load().lmd_vls_build_smem(vls["plan"]["rows"], (vls["cap_chunks"] - 2) * 8)),
      "info", vls["plan"]["info"].tolist())
