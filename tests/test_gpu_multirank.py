"""The multi-rank bench path (brick decomposition, ghost exchange, weak
scaling) run with the real kernels: two ranks share the one GPU, the ghost
exchange goes host-staged through gloo (NCCL on a multi-GPU node moves the
same tensors directly).  The global pair count must be twice the single
box's up to the brick interface (each brick sees its neighbour instead of
its own periodic image)."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_ranks_on_one_gpu_gloo():
    env = dict(os.environ, LMD_DIST_BACKEND="gloo", LMD_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29561", "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "3", "--workload", "c2", "--particles", "200000"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2 and d["config"]["parallelism"].startswith("bricks (2, 1, 1)")
    single = subprocess.run([sys.executable, "bench.py", "--steps", "2", "--warmup", "3",
                             "--workload", "c2", "--n=200000", "--e2e-steps", "0",
                             "--no-cpu-baseline"], cwd=ROOT,
                            capture_output=True, text=True, timeout=600)
    assert single.returncode == 0, single.stderr[-2000:]
    s = json.loads([ln for ln in single.stdout.splitlines() if ln.startswith("{")][-1])
    one = s["config"]["pairs_per_step"]
    assert abs(d["config"]["pairs_per_step"] - 2 * one) < 1e-3 * one


def test_strong_scaling_c4_bricks_match_single_domain():
    """The headline workload (BASELINE config 4, here a 48^3 lattice) split
    into 2x1x1 bricks: the global pair count equals the single-domain count
    exactly (ghost pairs are one-sided, counted once on the owning rank)."""
    env = dict(os.environ, LMD_DIST_BACKEND="gloo", LMD_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29564", "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "3", "--workload", "c4", "--particles", str(48 ** 3)]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["scaling"] == "strong" and d["config"]["parallelism"].startswith("bricks (2, 1, 1)")
    single = subprocess.run([sys.executable, "bench.py", "--steps", "2", "--warmup", "3",
                             "--workload", "c4", f"--n={48 ** 3}", "--e2e-steps", "0",
                             "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True,
                            timeout=600)
    assert single.returncode == 0, single.stderr[-2000:]
    s = json.loads([ln for ln in single.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["config"]["pairs_per_step"] == s["config"]["pairs_per_step"]
    # e2e at N > 1: force_phase_bricks on every rank's host buffers (the
    # bench asserts its global pair count equals the device-resident run's)
    assert d["e2e"]["value"] and d["e2e"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 48 ** 3 * 25


def test_brick_md_two_ranks_matches_single_domain():
    """run_md_bricks on 2 ranks (one GPU, gloo): migration at every rebuild,
    ghost exchange every step; per-step global pair counts equal to the
    single-domain loop's and final positions equal to rounding."""
    env = dict(os.environ, LMD_DIST_BACKEND="gloo", LMD_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29562", "tools/md_bricks_check.py",
           "--particles", "60000", "--steps", "22"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["rebuilds"] >= 3 and d["ids_complete"]
    assert d["single_pairs_equal"]
    assert d["max_position_diff"] < 1e-10


def test_brick_md_tuner_ranks_agree():
    """Per-rank tuners with MAX-reduced samples select the same
    configurations on every rank."""
    env = dict(os.environ, LMD_DIST_BACKEND="gloo", LMD_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29563", "tools/md_bricks_check.py",
           "--particles", "60000", "--steps", "50", "--tune", "1"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["selections_agree"] and len(d["phase_selections"]) >= 1
