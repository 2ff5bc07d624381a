"""CUDA kernel table (torch.profiler) of 20 VL MD steps on BASELINE config 2 (1M, rho 0.8)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2512_03565_b200 as B
from paper_2512_03565_b200 import workloads
w = workloads.config2(0.8, n=1_000_000, device="cuda")
params = B.LJParams(cutoff=2.5, skin=0.3, dt=0.001)
box = B.SimulationBox.cube(w.box_length, periodic=True)
cfg = B.Configuration.parse("vl,vl,false,v_by_one")
buf = B.ParticleBuffer.from_positions(w.positions.cpu().numpy(), device="cuda")
v = torch.as_tensor(w.velocities).to("cuda", torch.float64)
buf.vel_x.copy_(v[:, 0]); buf.vel_y.copy_(v[:, 1]); buf.vel_z.copy_(v[:, 2])
B.force_phase(buf, box, params, cfg, 8)
B.run_md(buf, box, params, 20, 8, fixed_config=cfg, rebuild_period=10, wrap="at_rebuild")
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    B.run_md(buf, box, params, 20, 8, fixed_config=cfg, rebuild_period=10, wrap="at_rebuild")
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=22))
