"""Host profile (cProfile) of the VL MD loop on BASELINE config 2 (1M, rho 0.8,
skin 0.3, rebuilt every 10 steps): per-step cost outside the kernels."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import workloads  # noqa: E402

w = workloads.config2(0.8, n=1_000_000, device="cuda")
params = B.LJParams(cutoff=2.5, skin=0.3, dt=0.001)
box = B.SimulationBox.cube(w.box_length, periodic=True)
cfg = B.Configuration.parse(os.environ.get("CONFIG", "vl,vl,false,v_by_one"))
buf = B.ParticleBuffer.from_positions(w.positions.cpu().numpy(), device="cuda")
v = torch.as_tensor(w.velocities).to("cuda", torch.float64)
buf.vel_x.copy_(v[:, 0]); buf.vel_y.copy_(v[:, 1]); buf.vel_z.copy_(v[:, 2])
B.force_phase(buf, box, params, cfg, 8)
B.run_md(buf, box, params, 20, 8, fixed_config=cfg, rebuild_period=10, wrap="at_rebuild")
torch.cuda.synchronize()
steps = int(os.environ.get("STEPS", "100"))
t0 = time.perf_counter()
r, s = B.run_md(buf, box, params, steps, 8, fixed_config=cfg, rebuild_period=10,
                wrap="at_rebuild")
torch.cuda.synchronize()
print(f"plain: {(time.perf_counter() - t0) * 1e3 / steps:.3f} ms/step")
prof = cProfile.Profile()
prof.enable()
B.run_md(buf, box, params, steps, 8, fixed_config=cfg, rebuild_period=10, wrap="at_rebuild")
torch.cuda.synchronize()
prof.disable()
pstats.Stats(prof).sort_stats("tottime").print_stats(25)
