"""Time the linked-cell full-shell force kernel, inline LJ vs hit-compacting
queue (csrc/force_lc.cu), per pattern on the bench workload (rc = 2.5, cell =
rc).  L2 flushed between launches; pair counts printed for a cross-check."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import _native as N  # noqa: E402
from paper_2512_03565_b200 import workloads  # noqa: E402

w = workloads.config2(0.8, n=int(os.environ.get("N", "1000000")), device="cuda")
box = B.SimulationBox.cube(w.box_length, periodic=True)
buf = B.ParticleBuffer.from_positions(w.positions.cpu().numpy(), device="cuda")
cont = B.LinkedCellsContainer(box, B.LJParams(cutoff=2.5, skin=0.0))
cont.rebuild(buf)
cont.refresh(buf)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for pname in os.environ.get("PATTERNS", "one_by_v,v_by_one,two_by_half,half_by_two").split(","):
    pat = B.PatternKind(pname)
    for queue in (False,):
        st = cont.launch_force(pat)
        ts = []
        for _ in range(5):
            flush.fill_(1)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            cont.launch_force(pat, stats_t=st)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        s = N.read_stats(st)
        print(f"{pname:12s} queue={int(queue)}  {min(ts) * 1e3:8.1f} us  pairs={s.pair_interactions}",
              flush=True)
