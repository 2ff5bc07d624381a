"""Time one VL container rebuild (1M, rho 0.8) and list its CPU-side ops and
kernels (torch.profiler): what the e2e path's 'rebuild' stage is made of."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import workloads  # noqa: E402

w = workloads.config2(0.8, n=1_000_000, device="cuda")
box = B.SimulationBox.cube(w.box_length, periodic=True)
buf = B.ParticleBuffer.from_positions(w.positions.cpu().numpy(), device="cuda")
kind = os.environ.get("KIND", "vl")
for _ in range(3):
    cont = B.make_container(kind, box, B.LJParams(cutoff=2.5, skin=0.3 if kind == "vl" else 0.0))
    cont.rebuild(buf)
    cont.refresh(buf)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    cont = B.make_container(kind, box, B.LJParams(cutoff=2.5, skin=0.3 if kind == "vl" else 0.0))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cont.rebuild(buf)
    cont.refresh(buf)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print(f"{kind} rebuild+refresh: min {min(ts) * 1e3:.3f} ms")
cont = B.make_container(kind, box, B.LJParams(cutoff=2.5, skin=0.3 if kind == "vl" else 0.0))
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    cont.rebuild(buf)
    cont.refresh(buf)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=22))
