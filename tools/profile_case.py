"""Small driver for ncu: build one container on the bench workload and launch
its force kernel a few times (the launches ncu captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2512_03565_b200 as B  # noqa: E402
from paper_2512_03565_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="vl,vl,false,v_by_one", help="comma-separated labels joined by +")
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--rho", type=float, default=0.8)
ap.add_argument("--launches", type=int, default=3)
args = ap.parse_args()
w = workloads.config2(args.rho, n=args.n, device="cuda")
for label in args.config.split("+"):
    cfg = B.Configuration.parse(label)
    skin = 0.0 if cfg.container.value == "lc" else 0.3
    params = B.LJParams(cutoff=2.5, skin=skin)
    box = B.SimulationBox.cube(w.box_length, periodic=True)
    buf = B.ParticleBuffer.from_positions(w.positions.cpu().numpy(), device="cuda")
    cont = B.make_container(cfg.container, box, params, cluster_size=8)
    # container knobs from the environment, e.g. VL_KNOBS=segmented=0,staged_group=128
    for kv in filter(None, os.environ.get("VL_KNOBS", "").split(",")):
        name, val = kv.split("=")
        setattr(cont, name, type(getattr(cont, name))(int(val) if val.isdigit() else val))
    cont.rebuild(buf)
    cont.refresh(buf)
    for _ in range(args.launches):
        st = cont.compute_forces(cfg.traversal, cfg.newton3, cfg.pattern, 8)
    torch.cuda.synchronize()
    print(label, st)
