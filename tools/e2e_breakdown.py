"""Time the stages of a one-shot force_phase on pinned host buffers (the
bench's e2e path), each stage between two synchronisations.
    python tools/e2e_breakdown.py [c4|c2]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import workloads  # noqa: E402
from paper_2512_03565_b200.containers import device_soa  # noqa: E402
from paper_2512_03565_b200.driver import _compute_once, _one_shot, _write_forces_back  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c4"
w = workloads.config4(256) if which == "c4" else workloads.config2(0.8, n=1_000_000, device="cuda")
host = w.positions.cpu().numpy() if hasattr(w.positions, "cpu") else np.asarray(w.positions)
box = B.SimulationBox.cube(w.box_length, periodic=True)
for label in os.environ.get("CONFIGS", "vl,vl,false,v_by_one").split("+"):
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
    for rep in range(3):
        T = {}
        torch.cuda.synchronize()
        t = time.perf_counter()
        d = device_soa(hb)
        torch.cuda.synchronize(); T["h2d"] = time.perf_counter() - t; t = time.perf_counter()
        cont = B.make_container(cfg.container, box, params, cluster_size=8)
        lean = _one_shot(cont)
        cont.rebuild(d)
        if not lean:
            cont.refresh(d)
        torch.cuda.synchronize(); T["rebuild"] = time.perf_counter() - t; t = time.perf_counter()
        st = _compute_once(cont, cfg, 8, False)
        torch.cuda.synchronize(); T["force path + stats"] = time.perf_counter() - t; t = time.perf_counter()
        cont.collect_forces(d)
        torch.cuda.synchronize(); T["collect"] = time.perf_counter() - t; t = time.perf_counter()
        _write_forces_back(hb, d)
        torch.cuda.synchronize(); T["d2h"] = time.perf_counter() - t
        n = len(host)
        print(label, w.name, " ".join(f"{k}={v*1e3:.2f}ms" for k, v in T.items()),
              f"total={sum(T.values())*1e3:.2f}ms pairs={st.pair_interactions}",
              f"h2d {n*25/T['h2d']/1e9:.1f} GB/s d2h {n*24/T['d2h']/1e9:.1f} GB/s", flush=True)
        del cont, d
