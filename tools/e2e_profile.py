"""Kernel/CPU timeline of one-shot force_phase calls on pinned host buffers
(the e2e path), via torch.profiler.  Prints per-stage wall times and the
kernel table."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile, record_function  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import workloads  # noqa: E402

w = workloads.config2(0.8, n=1_000_000, device="cuda")
host = w.positions.cpu().numpy()
box = B.SimulationBox.cube(w.box_length, periodic=True)
label = os.environ.get("CONFIG", "vl,vl,false,v_by_one")
cfg = B.Configuration.parse(label)
params = B.LJParams(cutoff=2.5, skin=0.0 if cfg.container.value == "lc" else 0.3)


class HB:
    pass


hb = HB()
for k, v in zip(("pos_x", "pos_y", "pos_z"), host.T):
    setattr(hb, k, torch.from_numpy(np.ascontiguousarray(v)).pin_memory())
for k in ("force_x", "force_y", "force_z"):
    setattr(hb, k, torch.zeros(len(host), dtype=torch.float64).pin_memory())
hb.ownership = torch.zeros(len(host), dtype=torch.int8).pin_memory()
for _ in range(3):
    B.force_phase(hb, box, params, cfg, 8)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    B.force_phase(hb, box, params, cfg, 8)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print(f"{label}: one-shot force_phase wall min {min(ts) * 1e3:.2f} ms, median {sorted(ts)[2] * 1e3:.2f} ms")
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    with record_function("force_phase"):
        B.force_phase(hb, box, params, cfg, 8)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30))
prof.export_chrome_trace(os.path.join(os.environ.get("OUT", "gpurun_out"), "e2e_trace.json"))
