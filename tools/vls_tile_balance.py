import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2512_03565_b200 as B
from paper_2512_03565_b200 import workloads
w = workloads.config4(256)
box = B.SimulationBox.cube(w.box_length, periodic=True)
params = B.LJParams(cutoff=2.5, skin=0.3)
buf = B.ParticleBuffer.from_positions(w.positions.cpu().numpy(), device="cuda")
cont = B.make_container("vl", box, params)
cont.rebuild(buf); cont.refresh(buf); cont.ensure_lists("v_by_one", False)
vls = cont._vls_for("v_by_one", False)
ng = vls["plan"]["ngroups"]
segc = vls["segc"][: 8 * ng].view(ng, 4, 2).double()
cin = segc[:, :, 0]
cnt = vls["plan"]["groups"][: ng * 64].view(ng, 64)[:, 1]
print("groups", ng, "particles per group: mean", float(cnt.double().mean()), "share with 128:", float((cnt == 128).double().mean()), "96:", float((cnt == 96).double().mean()), "<=64:", float((cnt <= 64).double().mean()))
mx = cin.max(dim=1).values
print("inner chunks per tile: mean", float(cin.mean()), "mean of per-group max", float(mx.mean()), "=> warp-slots idle at block ends:", 1 - float(cin.sum() / (4 * mx.sum())))
for t in range(4): print(" tile", t, "mean chunks", float(cin[:, t].mean()))
both = segc.sum(dim=2); mb = both.max(dim=1).values
print("both segments: idle", 1 - float(both.sum() / (4 * mb.sum())))
