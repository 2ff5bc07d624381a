"""Time the Verlet-list force kernels per pattern on the bench workload:
per-particle lists (csrc/vl.cu; gather modes pos4 / SoA, line-aligned
entry order) and i-cluster
lists (csrc/vl_ci.cu, CI = 2 and 4).  One line per variant; L2 flushed
between launches; also the build time of each list layout."""
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
cont = B.VerletListContainer(box, B.LJParams(cutoff=2.5, skin=0.3))
cont.rebuild(buf)
cont.refresh(buf)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
patterns = os.environ.get("PATTERNS", "v_by_one,half_by_two").split(",")
cis = [int(c) for c in os.environ.get("CIS", "1,2,4").split(",")]
aligns = [int(a) for a in os.environ.get("ALIGNS", "0,16").split(",")]


def timed(fn, reps=6):
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts) * 1e3


for pname in patterns:
    pat = B.PatternKind(pname)
    for ci, al in [(c, a) for c in cis for a in aligns]:
        cont.i_cluster = ci
        cont.align_window = al
        variants = (("pos4", 0, False), ("soa", 0, True))
        if ci > 1 or os.environ.get("FAST"):
            variants = (("pos4", 0, False),)
        for gname, knob, soa in variants:
            if ci > 1 and gname != "pos4":
                continue
            cont.knobs = knob
            cont.use_soa = soa
            cont.refresh(buf)
            cont._lists.clear()
            torch.cuda.synchronize()
            tb = timed(lambda: (cont._lists.clear(), cont._list(pat, False)), reps=3)
            st = cont.launch_force(pat, False)
            us = timed(lambda: cont.launch_force(pat, False, stats_t=st))
            s = N.read_stats(st)
            ent = cont.list_entries(pat, False)
            print(f"{pname:12s} CI={ci} align={al:2d} gather={gname:4s}  force {us:8.1f} us  "
                  f"build {tb:8.1f} us  entries={ent}  pairs={s.pair_interactions}", flush=True)
