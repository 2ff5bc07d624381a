"""run_md vs run_md_graph (CUDA-graph steady state) on BASELINE config 2
(1M, rho 0.8) and config 4 (16.8M) with Verlet lists: ms per step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import workloads  # noqa: E402

cfg = B.Configuration.parse("vl,vl,false,v_by_one")
params = B.LJParams(cutoff=2.5, skin=0.3, dt=0.001)
for name, w in (("c2 rho0.8 100k", workloads.config2(0.8, n=100_000, device="cuda")),
                ("c2 rho0.8 1M", workloads.config2(0.8, n=1_000_000, device="cuda")),
                ("c4 16.8M", workloads.config4(device="cuda"))):
    box = B.SimulationBox.cube(w.box_length, periodic=True)
    steps = 50 if "16.8M" in name else 100
    res = {}
    for mode in ("eager", "graph"):
        buf = B.ParticleBuffer.from_positions(w.positions.cpu().numpy(), device="cuda")
        v = torch.as_tensor(w.velocities).to("cuda", torch.float64)
        buf.vel_x.copy_(v[:, 0]); buf.vel_y.copy_(v[:, 1]); buf.vel_z.copy_(v[:, 2])
        B.force_phase(buf, box, params, cfg, 8)
        run = (lambda n: B.run_md_graph(buf, box, params, n, 8, config=cfg, rebuild_period=10)) \
            if mode == "graph" else \
            (lambda n: B.run_md(buf, box, params, n, 8, fixed_config=cfg, rebuild_period=10,
                                wrap="at_rebuild"))
        run(10)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        recs, _ = run(steps)
        torch.cuda.synchronize()
        res[mode] = (time.perf_counter() - t0) * 1e3 / steps
    print(f"{name}: eager {res['eager']:.3f} ms/step, graph {res['graph']:.3f} ms/step, "
          f"{len(buf) / res['graph'] * 1e3:.3e} particle-steps/s (graph)", flush=True)
# capture / replay cost of the two graphs at the last size
t0 = time.perf_counter()
g = torch.cuda.CUDAGraph()
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    g.capture_begin()
    B._native.call("lmd_verlet_step", len(buf), 1, 0.001, 1.0, *[B._native.ptr(getattr(buf, f)) for f in
                   ("pos_x", "pos_y", "pos_z", "vel_x", "vel_y", "vel_z", "force_x", "force_y",
                    "force_z", "old_force_x", "old_force_y", "old_force_z")],
                   B._native.ptr(buf.extra["nonfinite"]), B._native.stream())
    g.capture_end()
torch.cuda.current_stream().wait_stream(side)
torch.cuda.synchronize()
print(f"one-kernel capture+instantiate: {(time.perf_counter() - t0) * 1e3:.3f} ms")
