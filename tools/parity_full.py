"""Parity at the BASELINE's full sizes: GPU force phases (VL v_by_one and LC
c01 v_by_one, thread per particle; energy and virial on) against the oracle's
bitwise restatement of the reference force phase (LC c01, with energy and
virial) on the same seeded state.  One JSON line per workload:
pair counts, max per-particle force error relative to max(|F_ref|, 1),
energy / virial relative errors, |sum F| / sum |F| (momentum)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2512_03565_b200 import workloads  # noqa: E402


def run(w):
    pos = w.positions.cpu().numpy() if hasattr(w.positions, "cpu") else np.asarray(w.positions)
    L = w.box_length
    box = B.SimulationBox.cube(L, periodic=True)
    lo, hi = np.zeros(3), np.full(3, L)
    t0 = time.perf_counter()
    of, ost = O.force_phase_lc(pos, lo, hi, [True] * 3, B.LJParams(cutoff=2.5, skin=0.0),
                               "lc_c01", False, "one_by_v", 8)
    t_or = time.perf_counter() - t0
    out = {"workload": w.name, "particles": len(pos), "oracle_pairs": ost.pair_interactions,
           "oracle_s": round(t_or, 2)}
    fmax = np.maximum(np.abs(of).max(axis=1), 1.0)
    for label, skin in (("vl,vl,false,v_by_one", 0.3), ("lc,lc_c01,false,v_by_one", 0.0)):
        cfg = B.Configuration.parse(label)
        buf = B.ParticleBuffer.from_positions(pos, device="cuda")
        st = B.force_phase(buf, box, B.LJParams(cutoff=2.5, skin=skin), cfg, 8, energy=True)
        f = buf.forces().cpu().numpy()
        err = float((np.abs(f - of).max(axis=1) / fmax).max())
        out[label] = {
            "pairs_equal": st.pair_interactions == ost.pair_interactions,
            "max_force_rel_err": err,
            "epot_rel_err": abs(st.epot - ost.epot) / abs(ost.epot),
            "virial_rel_err": abs(st.virial - ost.virial) / abs(ost.virial),
            "momentum": float(np.abs(f.sum(axis=0)).max() / np.abs(f).sum()),
        }
        del buf
        torch.cuda.empty_cache()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    torch.cuda.set_device(0)
    for rho in (0.2, 0.5, 0.8):
        run(workloads.config2(rho, n=1_000_000, device="cuda"))
    if os.environ.get("C4", "1") == "1":
        run(workloads.config4(device="cuda"))
