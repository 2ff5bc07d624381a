"""The reference's remaining public entry points around the force path,
against fixtures produced by the unmodified reference (tests/golden/api.npz,
make_golden.py:api): the standalone cluster API (containers.py:216-299) and
the scenario driver (driver.py:75-313: build_initial_state,
resolve_search_space, run_simulation, emit_summary)."""

from __future__ import annotations

import types

import numpy as np
import pytest
import torch

from conftest import golden

import paper_2512_03565_b200 as B
from paper_2512_03565_b200 import (ContainerKind, LJParams, PatternKind, SimulationBox,
                                   TraversalKind)


def spec():
    """tests/golden/make_golden.py:api_spec restated with this package's types
    (a ScenarioSpec-shaped object: scenario.py:47-65)."""
    src = types.SimpleNamespace(origin=np.full(3, 0.6), counts=(8, 8, 8), spacing=1.2,
                                velocity=np.array([0.1, -0.05, 0.0]), jitter=0.8)
    return types.SimpleNamespace(
        box=SimulationBox.cube(9.6, periodic=True), params=LJParams(cutoff=2.5, skin=0.3,
                                                                    dt=0.002),
        sources=[src], iterations=60, seed=7, vector_width=8, cluster_size=4,
        rebuild_period=5, samples_per_config=2, tuning_interval=30, reduction="mean",
        metric="laneops",
        containers=[ContainerKind.LINKED_CELLS, ContainerKind.VERLET_CLUSTER_LISTS],
        traversals=[TraversalKind.LC_C01, TraversalKind.LC_C08, TraversalKind.VCL],
        newton3_options=[False, True], patterns=[PatternKind.ONE_BY_V, PatternKind.V_BY_ONE])


def test_resolve_search_space():
    g = golden("api.npz")
    assert [c.label for c in B.resolve_search_space(spec())] == [str(x) for x in g["space"]]


def test_emit_summary_format(tmp_path):
    s = B.RunSummary(per_config_metric={"lc,lc_c01,false,one_by_v": 3.0}, phase_selections=[],
                     failed_configs=[], wall_time_s=1.23456, particle_count=7,
                     initial_max_per_cell=2, final_max_per_cell=3, final_max_speed=0.5)
    path = tmp_path / "summary.txt"
    B.emit_summary(s, path)
    assert path.read_text() == (
        "particle_count: 7\nwall_time_s: 1.235\ntotal_force_phase_metric: 3.0\n"
        "initial_max_per_cell: 2\nfinal_max_per_cell: 3\nfinal_max_speed: 0.5\n"
        "phase_selections: -\nfailed_configs: -\nper_config_metric:\n"
        "  lc,lc_c01,false,one_by_v: 3.0\n")


@pytest.mark.gpu
@pytest.mark.parametrize("m", [4, 8])
def test_build_clusters_and_neighbor_lists(m):
    g = golden("api.npz")
    buf = B.ParticleBuffer.from_positions(g["cl_pos"], device="cuda")
    cl = B.build_clusters(buf, m)
    assert len(cl) == len(g[f"cl{m}_nreal"])
    assert [c.n_real for c in cl] == g[f"cl{m}_nreal"].tolist()
    assert np.array_equal(np.stack([c.buffer.id.cpu().numpy() for c in cl]), g[f"cl{m}_ids"])
    assert np.array_equal(np.stack([c.aabb_min for c in cl]), g[f"cl{m}_amin"])
    assert np.array_equal(np.stack([c.aabb_max for c in cl]), g[f"cl{m}_amax"])
    assert np.array_equal(np.stack([c.buffer.positions().cpu().numpy() for c in cl]),
                          g[f"cl{m}_pos"])
    for n3 in (False, True):
        lists = B.build_cluster_neighbor_lists(cl, 2.7, n3)
        flat = np.array([(k, z) for k, zs in enumerate(lists) for z in zs],
                        dtype=np.int64).reshape(-1, 2)
        assert np.array_equal(flat, g[f"cl{m}_pairs_n3{int(n3)}"]), n3


@pytest.mark.gpu
def test_build_initial_state_and_run_simulation_reproduce_reference(tmp_path):
    g = golden("api.npz")
    sp = spec()
    b0 = B.build_initial_state(sp)
    assert np.array_equal(b0.positions().cpu().numpy(), g["init_pos"])
    vel = torch.stack([b0.vel_x, b0.vel_y, b0.vel_z], 1).cpu().numpy()
    assert np.array_equal(vel, g["init_vel"])
    records, summary = B.run_simulation(sp)
    assert [r.configuration.label for r in records] == [str(x) for x in g["rec_label"]]
    assert [r.phase for r in records] == [str(x) for x in g["rec_phase"]]
    got = np.array([[r.metric_value, r.lane_slots, r.useful_interactions, r.blank_lanes,
                     r.pair_interactions] for r in records])
    assert np.array_equal(got, g["rec_num"])
    assert summary.phase_selections == [str(x) for x in g["sum_selections"]]
    assert list(summary.per_config_metric) == [str(x) for x in g["sum_metric_labels"]]
    assert np.array_equal(np.array(list(summary.per_config_metric.values())),
                          g["sum_metric_values"])
    assert [summary.initial_max_per_cell, summary.final_max_per_cell] == g["sum_cells"].tolist()
    assert abs(summary.final_max_speed - float(g["sum_speed"][0])) <= 1e-10
    B.emit_csv(records, tmp_path / "run.csv")
    back = B.read_records_csv(tmp_path / "run.csv")
    assert [r.pair_interactions for r in back] == [r.pair_interactions for r in records]
