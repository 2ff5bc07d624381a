"""Profile one VCL rebuild + refresh (1M, rho 0.8, rc 2.5, skin 0.3) for a
cluster size: wall time and the kernel / host-op table."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import workloads  # noqa: E402

M = int(os.environ.get("M", "4"))
w = workloads.config2(0.8, n=1_000_000, device="cuda")
box = B.SimulationBox.cube(w.box_length, periodic=True)
buf = B.ParticleBuffer.from_positions(w.positions.cpu().numpy(), device="cuda")
params = B.LJParams(cutoff=2.5, skin=0.3)
for _ in range(2):
    c = B.VerletClusterContainer(box, params, M)
    c.rebuild(buf)
    c.refresh(buf)
torch.cuda.synchronize()
for _ in range(3):
    c = B.VerletClusterContainer(box, params, M)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    c.rebuild(buf)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    c.refresh(buf)
    torch.cuda.synchronize()
    print(f"M={M} rebuild {(t1 - t0) * 1e3:.2f} ms  refresh {(time.perf_counter() - t1) * 1e3:.2f} ms")
c = B.VerletClusterContainer(box, params, M)
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    c.rebuild(buf)
    c.refresh(buf)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))
