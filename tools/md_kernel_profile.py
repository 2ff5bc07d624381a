"""CUDA kernel table (torch.profiler) of 20 MD steps of BASELINE config 1."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2512_03565_b200 as B
from paper_2512_03565_b200 import workloads
w = workloads.config1()
params = B.LJParams(cutoff=2.5, skin=0.0, dt=0.001)
box = B.SimulationBox.cube(w.box_length, periodic=True)
cfg = B.Configuration.parse("lc,lc_c08,true,one_by_v")
buf = B.ParticleBuffer.from_positions(w.positions, device="cuda")
B.force_phase(buf, box, params, cfg, 8)
B.run_md(buf, box, params, 20, 8, fixed_config=cfg)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    B.run_md(buf, box, params, 20, 8, fixed_config=cfg)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
