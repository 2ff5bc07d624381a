"""CUDA kernel table (torch.profiler) and per-step wall time of VCL MD steps
on BASELINE config 3 (2M droplet, rc 3.0, skin 0.3, M = 8)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import workloads  # noqa: E402

w = workloads.config3(n=int(os.environ.get("N", "2000000")), device="cuda")
params = B.LJParams(cutoff=3.0, skin=0.3, dt=0.001)
box = B.SimulationBox.cube(w.box_length, periodic=True)
cfg = B.Configuration.parse("vcl,vcl,false,half_by_two,m8")
buf = B.ParticleBuffer.from_positions(w.positions.cpu().numpy(), device="cuda")
v = torch.as_tensor(w.velocities).to("cuda", torch.float64)
buf.vel_x.copy_(v[:, 0]); buf.vel_y.copy_(v[:, 1]); buf.vel_z.copy_(v[:, 2])
B.force_phase(buf, box, params, cfg, 8)
B.run_md(buf, box, params, 10, 8, fixed_config=cfg, wrap="at_rebuild")
torch.cuda.synchronize()
t0 = time.perf_counter()
B.run_md(buf, box, params, 40, 8, fixed_config=cfg, wrap="at_rebuild")
torch.cuda.synchronize()
print(f"{(time.perf_counter() - t0) * 1e3 / 40:.3f} ms/step")
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    B.run_md(buf, box, params, 10, 8, fixed_config=cfg, wrap="at_rebuild")
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=16))
