"""Host-side profile (cProfile) of run_md on BASELINE config 1 (8,000
particles, LC c08 Newton3, rebuild every step): where the ~ms per step go."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import workloads  # noqa: E402

w = workloads.config1()
params = B.LJParams(cutoff=2.5, skin=0.0, dt=0.001)
box = B.SimulationBox.cube(w.box_length, periodic=True)
cfg = B.Configuration.parse(os.environ.get("CONFIG", "lc,lc_c08,true,one_by_v"))
buf = B.ParticleBuffer.from_positions(w.positions, device="cuda")
v = torch.as_tensor(w.velocities).to("cuda", torch.float64)
buf.vel_x.copy_(v[:, 0]); buf.vel_y.copy_(v[:, 1]); buf.vel_z.copy_(v[:, 2])
B.force_phase(buf, box, params, cfg, 8)
B.run_md(buf, box, params, 20, 8, fixed_config=cfg)
torch.cuda.synchronize()
steps = int(os.environ.get("STEPS", "200"))
t0 = time.perf_counter()
prof = cProfile.Profile()
prof.enable()
records, summary = B.run_md(buf, box, params, steps, 8, fixed_config=cfg)
torch.cuda.synchronize()
prof.disable()
dt = time.perf_counter() - t0
print(f"{steps} steps: {dt * 1e3 / steps:.3f} ms/step (under cProfile), "
      f"{summary.particle_steps_per_s:.3e} particle-steps/s")
pstats.Stats(prof).sort_stats("cumulative").print_stats(35)
