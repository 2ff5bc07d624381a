"""bench.py itself on a small workload: the JSON line carries the contract's
keys, and the pair count it reports is the reference's (Newton3 bookkeeping
included) -- checked against the oracle on the same seeded state."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N = 60_000
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
        "e2e", "cpu_baseline", "gpu_launches", "clocks")


def _bench(cfg, extra=()):
    cmd = [sys.executable, "bench.py", "--config", cfg, "--steps", "3", "--warmup", "3",
           "--workload", "c2", "--particles", str(N), *extra]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])


@pytest.fixture(scope="module")
def state():
    sys.path.insert(0, ROOT)
    from paper_2512_03565_b200 import workloads
    w = workloads.config2(0.8, n=N, device="cuda")
    return w.positions.cpu().numpy(), w.box_length


@pytest.mark.parametrize("cfg", ["vl,vl,false,v_by_one", "lc,lc_c08,true,v_by_one",
                                 "vl,vl,true,half_by_two", "lc,lc_c01,false,half_by_two"])
def test_bench_line_and_pair_convention(cfg, state):
    pos, L = state
    d = _bench(cfg, ("--e2e-steps", "1") if cfg.startswith("vl,vl,false") else
               ("--e2e-steps", "0", "--no-cpu-baseline"))
    for k in KEYS:
        assert k in d, k
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"]
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["steps"] == 3
    cont, trav, n3, pat = cfg.split(",")
    from paper_2512_03565_b200 import LJParams
    params = LJParams(cutoff=2.5, skin=0.0)
    if trav == "vl":
        _, ost = O.force_phase_vl(pos, np.zeros(3), np.full(3, L), [True] * 3,
                                  LJParams(cutoff=2.5, skin=0.3), n3 == "true", pat, 8)
    else:
        _, ost = O.force_phase_lc(pos, np.zeros(3), np.full(3, L), [True] * 3, params, trav,
                                  n3 == "true", pat, 8)
    assert d["config"]["pairs_per_step"] == ost.pair_interactions
    if d["e2e"] and d["e2e"].get("value"):
        assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
