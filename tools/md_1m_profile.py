import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2512_03565_b200 as B
from paper_2512_03565_b200 import workloads
w = workloads.config2(0.8, n=1_000_000, device="cuda")
box = B.SimulationBox.cube(w.box_length, periodic=True)
params = B.LJParams(cutoff=2.5, skin=0.3, dt=0.001)
cfg = B.Configuration.parse("vl,vl,false,v_by_one")
buf = B.ParticleBuffer.from_positions(w.positions.cpu().numpy(), device="cuda")
v = torch.as_tensor(w.velocities).to("cuda", torch.float64)
buf.vel_x.copy_(v[:, 0]); buf.vel_y.copy_(v[:, 1]); buf.vel_z.copy_(v[:, 2])
B.force_phase(buf, box, params, cfg, 8)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rec, summ = B.run_md(buf, box, params, 100, 8, fixed_config=cfg, rebuild_period=10, wrap="at_rebuild")
    torch.cuda.synchronize(); print("wall per step ms", (time.perf_counter() - t0) * 10, "force ms/step", summ.force_time_s * 10, summ.rebuilds)
