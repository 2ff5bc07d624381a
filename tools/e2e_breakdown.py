"""Time the stages of a one-shot force_phase on host buffers (e2e path)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import workloads  # noqa: E402
from paper_2512_03565_b200.containers import device_soa  # noqa: E402

w = workloads.config2(0.8, n=1_000_000, device="cuda")
host = w.positions.cpu().numpy()
box = B.SimulationBox.cube(w.box_length, periodic=True)
for label in os.environ.get("CONFIGS", "vl,vl,false,v_by_one+lc,lc_c01,false,half_by_two").split("+"):
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
        cont.rebuild(d)
        torch.cuda.synchronize(); T["rebuild"] = time.perf_counter() - t; t = time.perf_counter()
        cont.refresh(d)
        torch.cuda.synchronize(); T["refresh"] = time.perf_counter() - t; t = time.perf_counter()
        if cfg.container.value == "vl":
            cont._list(cfg.pattern, cfg.newton3)
            torch.cuda.synchronize(); T["lists"] = time.perf_counter() - t; t = time.perf_counter()
        st = cont.compute_forces(cfg.traversal, cfg.newton3, cfg.pattern, 8)
        torch.cuda.synchronize(); T["force+stats"] = time.perf_counter() - t; t = time.perf_counter()
        cont.collect_forces(d)
        for k in ("force_x", "force_y", "force_z"):
            getattr(hb, k).copy_(getattr(d, k))
        torch.cuda.synchronize(); T["d2h"] = time.perf_counter() - t
        print(label, " ".join(f"{k}={v*1e3:.2f}ms" for k, v in T.items()),
              f"total={sum(T.values())*1e3:.2f}ms", flush=True)
