"""Time the Verlet-cluster-list force kernel per cluster size M on the bench
workload (1M uniform, rc 2.5, skin 0.3).  L2 flushed between launches."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import _native as N  # noqa: E402
from paper_2512_03565_b200 import workloads  # noqa: E402

w = workloads.config2(0.8, n=int(os.environ.get("N", "1000000")), device="cuda")
box = B.SimulationBox.cube(w.box_length, periodic=True)
buf = B.ParticleBuffer.from_positions(w.positions.cpu().numpy(), device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
params = B.LJParams(cutoff=2.5, skin=float(os.environ.get("SKIN", "0.3")))
for m in [int(x) for x in os.environ.get("MS", "4,8,16,32").split(",")]:
    cont = B.VerletClusterContainer(box, params, m)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cont.rebuild(buf)
    cont.refresh(buf)
    torch.cuda.synchronize()
    tb = time.perf_counter() - t0
    st = cont.launch_force(False)
    ts = []
    for _ in range(5):
        flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        cont.launch_force(False, st)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    s = N.read_stats(st)
    inv, slots, useful = cont.vcl_stats(False, B.PatternKind.V_BY_ONE, 8)
    print(f"M={m:2d}  force {min(ts) * 1e3:8.1f} us  rebuild+refresh {tb * 1e3:7.1f} ms  "
          f"pairs={s.pair_interactions}  useful(tests)={useful}  "
          f"eff={s.pair_interactions / max(useful, 1):.3f}", flush=True)
