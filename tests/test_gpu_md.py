"""Device MD loop: the reference's driver semantics (config 1 trajectory) and
the tuner (full-search sampling, laneops / replay selection)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import golden

import paper_2512_03565_b200 as B
from paper_2512_03565_b200 import (PATTERN_ORDER, Configuration, ContainerKind, LJParams,
                                   ParticleBuffer, SimulationBox, TraversalKind, TuningPolicy,
                                   enumerate_search_space)
from paper_2512_03565_b200.simulation import emit_csv, read_records_csv, run_md

pytestmark = pytest.mark.gpu


def test_run_md_config1_matches_reference_trajectory(tmp_path):
    g = golden("config1.npz")
    box = SimulationBox.cube(22.0, periodic=True)
    params = LJParams(cutoff=2.5, skin=0.0, dt=0.001)
    buf = ParticleBuffer.from_positions(g["pos0"], device="cuda")
    v = torch.as_tensor(g["vel0"], device="cuda")
    buf.vel_x.copy_(v[:, 0]); buf.vel_y.copy_(v[:, 1]); buf.vel_z.copy_(v[:, 2])
    cfg = Configuration.parse("lc,lc_c08,true,one_by_v")
    B.force_phase(buf, box, params, cfg, 8)          # seed forces for the first kick
    records, summary = run_md(buf, box, params, 10, 8, fixed_config=cfg, metric="laneops")
    assert [r.pair_interactions for r in records] == g["pairs_per_step"].tolist()
    assert np.abs(buf.positions().cpu().numpy() - g["pos10"]).max() < 1e-12
    path = tmp_path / "run.csv"
    emit_csv(records, path)
    assert read_records_csv(path) == records


def test_tuner_samples_every_config_and_selects_by_replay(tmp_path):
    rng = np.random.default_rng(11)
    grid = np.stack(np.meshgrid(*[np.arange(5)] * 3, indexing="ij"), -1).reshape(-1, 3)
    pos = 4.0 + grid * 1.2 + rng.uniform(-0.02, 0.02, grid.shape)
    box = SimulationBox(np.zeros(3), np.full(3, 14.0), ("reflective",) * 3)
    params = LJParams(cutoff=2.5, skin=0.5, dt=0.001)
    configs = enumerate_search_space([ContainerKind.LINKED_CELLS],
                                     [TraversalKind.LC_C01, TraversalKind.LC_C08], [False, True],
                                     list(PATTERN_ORDER))
    assert len(configs) == 12
    target = configs[7]
    schedule = []
    for _ in range(3):
        schedule.extend(k // 2 for k in range(24))
        schedule.extend([None] * 6)
    lines = [str(5.0) if i is None else str(1.0 if configs[i] == target else 10.0 + i)
             for i in schedule]
    replay = tmp_path / "replay.txt"
    replay.write_text("\n".join(lines) + "\n")
    buf = ParticleBuffer.from_positions(pos, device="cuda")
    records, summary = run_md(buf, box, params, 90, 8, configurations=configs,
                              policy=TuningPolicy(2, 30, "mean", f"replay:{replay}"),
                              metric=f"replay:{replay}", rebuild_period=100000)
    assert summary.phase_selections == [target.label] * 3
    for start in (0, 30, 60):
        window = records[start:start + 24]
        assert all(r.phase == "tuning" for r in window)
        seen = {}
        for r in window:
            seen[r.configuration.label] = seen.get(r.configuration.label, 0) + 1
        assert seen == {c.label: 2 for c in configs}


@pytest.mark.parametrize("metric", ["time", "iteration"])
def test_time_metric_tuner_runs_all_containers(metric):
    rng = np.random.default_rng(5)
    n = 4000
    span = (n / 0.7) ** (1 / 3)
    k = int(np.ceil(n ** (1 / 3)))
    grid = np.stack(np.meshgrid(*[np.arange(k)] * 3, indexing="ij"), -1).reshape(-1, 3)[:n]
    pos = (grid + 0.5) * (span / k) + rng.uniform(-0.1, 0.1, (n, 3))
    box = SimulationBox.cube(span, periodic=True)
    params = LJParams(cutoff=2.5, skin=0.3, dt=0.001)
    configs = enumerate_search_space(list(ContainerKind), list(TraversalKind), [False],
                                     [B.PatternKind.V_BY_ONE, B.PatternKind.HALF_BY_TWO])
    buf = ParticleBuffer.from_positions(pos, device="cuda")
    records, summary = run_md(buf, box, params, len(configs) + 5, 8, configurations=configs,
                              policy=TuningPolicy(1, len(configs) + 5, "mean", metric),
                              metric=metric)
    assert len(summary.phase_selections) == 1
    pairs = {r.pair_interactions for r in records[:2]}
    assert min(r.metric_value for r in records) > 0
    if metric == "iteration":   # the whole step contains the force phase
        force = {r.configuration.label: r.metric_value for r in records}
        assert all(v > 0 for v in force.values())


def test_energy_metric_reads_board_energy():
    """NVML energy over a ~0.3 s DFMA burn is positive; run_md accepts the
    metric (samples are coarse, >= 0)."""
    m = B.make_metric_provider("energy", lambda: 0)
    out = torch.empty(148 * 8 * 256, dtype=torch.float64, device="cuda")
    m.begin_region()
    import time as _t
    t0 = _t.perf_counter()
    while _t.perf_counter() - t0 < 0.3:
        B._native.call("lmd_dfma_burn", 148 * 8, 256, 20000, B._native.ptr(out), None)
        torch.cuda.synchronize()
    assert m.end_region() > 0
    rng = np.random.default_rng(2)
    grid = np.stack(np.meshgrid(*[np.arange(10)] * 3, indexing="ij"), -1).reshape(-1, 3)
    pos = (grid + 0.5) * 1.1 + rng.uniform(-0.05, 0.05, grid.shape)
    buf = ParticleBuffer.from_positions(pos, device="cuda")
    cfg = B.Configuration.parse("vl,vl,false,v_by_one")
    records, _ = run_md(buf, SimulationBox.cube(11.0, periodic=True), LJParams(cutoff=2.5,
                        skin=0.3, dt=0.001), 4, 8, fixed_config=cfg, metric="energy")
    assert all(r.metric_value >= 0 for r in records)


def test_graph_md_matches_eager_md():
    """run_md_graph (steady-state step replayed as a CUDA graph) gives the
    same trajectory, bitwise, and the same per-step pair counts as run_md."""
    rng = np.random.default_rng(9)
    k = 18
    grid = np.stack(np.meshgrid(*[np.arange(k)] * 3, indexing="ij"), -1).reshape(-1, 3)
    span = k * 1.12
    pos = (grid + 0.5) * 1.12 + rng.uniform(-0.1, 0.1, grid.shape)
    vel = rng.normal(0.0, 1.0, grid.shape)
    box = SimulationBox.cube(span, periodic=True)
    params = LJParams(cutoff=2.5, skin=0.3, dt=0.002)
    cfg = B.Configuration.parse("vl,vl,false,v_by_one")
    out = []
    for graph in (False, True):
        buf = ParticleBuffer.from_positions(pos, device="cuda")
        v = torch.as_tensor(vel, device="cuda")
        buf.vel_x.copy_(v[:, 0]); buf.vel_y.copy_(v[:, 1]); buf.vel_z.copy_(v[:, 2])
        B.force_phase(buf, box, params, cfg, 8)
        if graph:
            recs, summ = B.run_md_graph(buf, box, params, 25, 8, config=cfg, rebuild_period=10)
            assert summ.extra["rebuilds"] >= 3
        else:
            recs, _ = run_md(buf, box, params, 25, 8, fixed_config=cfg, rebuild_period=10,
                             wrap="at_rebuild")
        out.append((buf.positions().cpu().numpy(), [r.pair_interactions for r in recs]))
    assert out[0][1] == out[1][1]
    assert np.array_equal(out[0][0], out[1][0])


def test_vl_refresh_and_check_decides_like_needs_rebuild():
    """The MD loop's fused rebuild decision (displacement reduced inside the
    Verlet-list refresh) equals needs_rebuild's (containers.py:23-38) on
    displacements just below, at and above skin / 2, and leaves the container
    refreshed when no rebuild is due."""
    rng = np.random.default_rng(3)
    side, a = 16, 1.1
    n, L = side ** 3, side * a
    grid = np.stack(np.meshgrid(*[np.arange(side)] * 3, indexing="ij"), -1).reshape(-1, 3)
    pos = (grid + 0.5) * a + rng.uniform(-0.1, 0.1, (n, 3))
    box = SimulationBox.cube(L, periodic=True)
    params = LJParams(cutoff=2.5, skin=0.3, dt=0.001)
    cfg = Configuration.parse("vl,vl,false,v_by_one")
    for move, expect in ((0.149999, False), (0.15, True), (0.2, True), (0.0, False)):
        buf = ParticleBuffer.from_positions(pos, device="cuda")
        cont = B.make_container("vl", box, params, rebuild_period=1000)
        cont.rebuild(buf)
        cont.refresh(buf)
        cont.ensure_lists(cfg.pattern, False)
        buf.pos_x[n // 2] += move * 0.6
        buf.pos_y[n // 2] -= move * 0.8
        want = cont.needs_rebuild(buf)
        got = cont.refresh_and_check(buf)
        assert got == want
        if move in (0.2, 0.0):
            assert got == expect
        if not got:   # refreshed: the forces are those of the moved positions
            st = cont.compute_forces("vl", False, cfg.pattern, 8)
            cont.collect_forces(buf)
            ref = ParticleBuffer.from_positions(buf.positions().cpu().numpy(), device="cuda")
            st2 = B.force_phase(ref, box, params, cfg, 8)
            assert st.pair_interactions == st2.pair_interactions
            scale = float(ref.forces().abs().max())
            assert float((buf.forces() - ref.forces()).abs().max()) <= 1e-12 * scale
    # the period rule
    buf = ParticleBuffer.from_positions(pos, device="cuda")
    cont = B.make_container("vl", box, params, rebuild_period=2)
    cont.rebuild(buf)
    cont.steps_since_rebuild = 2
    assert cont.refresh_and_check(buf) is True



def test_fused_integrator_halves_are_bitwise_the_two_launches():
    """run_md with the post-force half and the next pre-force half fused into
    one pass (the default with wrap="at_rebuild") gives bit for bit the
    trajectory of the two separate launches."""
    rng = np.random.default_rng(21)
    side, a = 14, 1.12
    n, L = side ** 3, side * a
    grid = np.stack(np.meshgrid(*[np.arange(side)] * 3, indexing="ij"), -1).reshape(-1, 3)
    pos = (grid + 0.5) * a + rng.uniform(-0.08, 0.08, (n, 3))
    vel = rng.normal(0.0, 1.0, (n, 3))
    box = SimulationBox.cube(L, periodic=True)
    params = LJParams(cutoff=2.5, skin=0.3, dt=0.002)
    cfg = Configuration.parse("vl,vl,false,v_by_one")
    out = []
    for fuse in (False, True):
        buf = ParticleBuffer.from_positions(pos, device="cuda")
        v = torch.as_tensor(vel, device="cuda")
        buf.vel_x.copy_(v[:, 0]); buf.vel_y.copy_(v[:, 1]); buf.vel_z.copy_(v[:, 2])
        B.force_phase(buf, box, params, cfg, 8)
        records, _ = run_md(buf, box, params, 23, 8, fixed_config=cfg, rebuild_period=7,
                            wrap="at_rebuild", fuse_halves=fuse)
        out.append(([r.pair_interactions for r in records], buf.positions().cpu().numpy(),
                    buf.velocities().cpu().numpy(), buf.forces().cpu().numpy()))
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1])
    assert np.array_equal(out[0][2], out[1][2])
    assert np.array_equal(out[0][3], out[1][3])
