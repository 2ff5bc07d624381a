"""LC Newton3 (lc_c08 / lc_c18, Newton3 on) executed as colored dual-write
passes vs as the 27-cell full shell with Newton3 bookkeeping: force-phase
time per pattern on BASELINE config 1 (8,000 particles) and on the 1M
bench workload.  L2 flushed between launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import workloads  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for w in (workloads.config1(), workloads.config2(0.8, n=1_000_000, device="cuda")):
    pos = w.positions.cpu().numpy() if hasattr(w.positions, "cpu") else w.positions
    box = B.SimulationBox.cube(w.box_length, periodic=True)
    buf = B.ParticleBuffer.from_positions(pos, device="cuda")
    for trav in ("lc_c08", "lc_c18"):
        code = B.traversals.traversal_code(B.TraversalKind(trav))
        for pat in ("one_by_v", "half_by_two"):
            row = []
            for mode in ("colored", "full_shell"):
                cont = B.LinkedCellsContainer(box, B.LJParams(cutoff=2.5, skin=0.0))
                cont.n3_mode = mode
                cont.rebuild(buf)
                cont.refresh(buf)
                st = cont.launch_force(pat, traversal=code, newton3=True)
                ts = []
                for _ in range(5):
                    flush.fill_(1)
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    cont.launch_force(pat, stats_t=st, traversal=code, newton3=True)
                    e1.record()
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1))
                row.append(f"{mode} {min(ts) * 1e3:9.1f} us")
            print(f"{w.name:28s} {trav} {pat:12s} " + "   ".join(row), flush=True)
