"""Time lmd_force_vl kernel variants (unroll x persistent grid) per pattern on
the bench workload.  Prints one line per variant; L2 flushed between launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import workloads  # noqa: E402

w = workloads.config2(0.8, n=int(os.environ.get("N", "1000000")), device="cuda")
box = B.SimulationBox.cube(w.box_length, periodic=True)
buf = B.ParticleBuffer.from_positions(w.positions.cpu().numpy(), device="cuda")
cont = B.VerletListContainer(box, B.LJParams(cutoff=2.5, skin=0.3))
cont.rebuild(buf)
cont.refresh(buf)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
patterns = os.environ.get("PATTERNS", "v_by_one,half_by_two").split(",")
for pname in patterns:
    pat = B.PatternKind(pname)
    for n3 in (False,):
        for ucode, u, soa in ((0, 4, 0), (2, 2, 0), (2, 2, 1)):
            for pers in (0, 1):
                cont.knobs = (ucode << 4) | (pers << 6)
                cont.use_soa = bool(soa)
                cont.refresh(buf)
                st = cont.launch_force(pat, n3)
                ts = []
                for _ in range(6):
                    flush.fill_(1)
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    cont.launch_force(pat, n3, stats_t=st)
                    e1.record()
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1))
                from paper_2512_03565_b200 import _native as N
                s = N.read_stats(st)
                print(f"{pname:12s} n3={int(n3)} U={u} soa={soa} persistent={pers}  {min(ts)*1e3:8.1f} us  "
                      f"pairs={s.pair_interactions}", flush=True)
