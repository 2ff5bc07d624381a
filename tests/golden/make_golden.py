"""Generate the golden fixtures that pin the oracle (and through it the GPU path).

Runs the UNMODIFIED reference package (lanemd, imported read-only from
/root/reference/pkg/src) on seeded inputs and stores inputs + outputs as
compressed .npz files next to this script.  Only this container has the
reference; the fixtures travel with the repository.

    python tests/golden/make_golden.py
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import lanemd  # noqa: F401
    return lanemd


def jittered_lattice(rng, counts, spacing, jitter):
    grid = np.mgrid[0:counts[0], 0:counts[1], 0:counts[2]]
    pos = grid.reshape(3, -1).T * spacing + spacing / 2
    return pos + rng.uniform(-jitter, jitter, pos.shape)


def make_buffer(L, pos):
    n = len(pos)
    b = L.ParticleBuffer.empty(n)
    if n:
        b.pos_x[:], b.pos_y[:], b.pos_z[:] = np.asarray(pos, dtype=np.float64).T
    b.id[:] = np.arange(n)
    return b


def random_instance(rng, periodic):
    """Like the reference's acceptance criterion 1 instance generator."""
    n = int(rng.integers(16, 301))
    density = rng.uniform(0.2, 0.7)
    span = (n / density) ** (1 / 3)
    per_axis = math.ceil(n ** (1 / 3))
    spacing = span / per_axis
    pos = jittered_lattice(rng, (per_axis,) * 3, spacing, 0.25 * spacing)[:n]
    cutoff = float(min(rng.uniform(1.5, 3.5), span / 1.5))
    if periodic:
        cutoff = float(min(cutoff, span / 2.2))
    return pos, span * 1.001, cutoff, 0.2 * cutoff


def instances(L):
    from lanemd.driver import force_phase
    from lanemd.kernels import PATTERN_ORDER
    from lanemd.tuning import ContainerKind, enumerate_search_space
    from lanemd.traversals import TraversalKind
    configs = enumerate_search_space(
        [ContainerKind.LINKED_CELLS, ContainerKind.VERLET_CLUSTER_LISTS],
        [TraversalKind.LC_C01, TraversalKind.LC_C08, TraversalKind.LC_C18, TraversalKind.VCL],
        [False, True], list(PATTERN_ORDER))
    assert len(configs) == 28
    rng = np.random.default_rng(20240817)
    out = {}
    labels = [c.label for c in configs]
    out["labels"] = np.array(labels)
    for k in range(8):
        periodic = k % 2 == 1
        pos, span, cutoff, skin = random_instance(rng, periodic)
        kind = L.BoundaryKind.PERIODIC if periodic else L.BoundaryKind.REFLECTIVE
        box = L.SimulationBox(np.zeros(3), np.full(3, span), (kind,) * 3)
        params = L.LJParams(cutoff=cutoff, skin=skin)
        out[f"i{k}_pos"] = pos
        out[f"i{k}_box"] = np.array([span, float(periodic), cutoff, skin])
        stats = np.zeros((len(configs), 3, 4), dtype=np.int64)
        for ci, cfg in enumerate(configs):
            for vi, V in enumerate((4, 8, 16)):
                buf = make_buffer(L, pos)
                st = force_phase(buf, box, params, cfg, V)
                stats[ci, vi] = (st.kernel_invocations, st.lane_slots, st.useful_interactions,
                                 st.pair_interactions)
                # forces do not depend on the pattern; store one per
                # (container, traversal, newton3) and cluster size
                pkey = cfg.label.rsplit(",", 1)[0]
                if cfg.container is ContainerKind.VERLET_CLUSTER_LISTS:
                    pkey += f",M{V}"
                key = f"i{k}_F_{pkey}"
                if key not in out:
                    out[key] = buf.forces()
                else:
                    assert np.array_equal(out[key], buf.forces())
        out[f"i{k}_stats"] = stats
    np.savez_compressed(os.path.join(HERE, "instances.npz"), **out)


def config1(L):
    """BASELINE config 1: 20^3 SC lattice, spacing 1.1, L = 22, rc = 2.5, skin 0."""
    from lanemd import (POST_FORCE, PRE_FORCE, apply_boundaries, velocity_verlet_step)
    from lanemd.driver import force_phase
    from lanemd.kernels import PatternKind
    from lanemd.traversals import TraversalKind
    from lanemd.tuning import Configuration, ContainerKind
    parts = L.generate_cube_lattice((0.0, 0.0, 0.0), (20, 20, 20), 1.1)
    buf = L.soa_from_particles(parts)
    rng = np.random.default_rng(42)
    v = rng.normal(0.0, 1.0, (8000, 3))
    v -= v.mean(axis=0)
    buf.vel_x[:], buf.vel_y[:], buf.vel_z[:] = v.T
    box = L.SimulationBox(np.zeros(3), np.full(3, 22.0), (L.BoundaryKind.PERIODIC,) * 3)
    params = L.LJParams(cutoff=2.5, skin=0.0, dt=0.001)
    out = {"pos0": buf.positions(), "vel0": v.copy()}
    cont = L.LinkedCellsContainer(box, params)
    cells = cont.linear_index(cont.cell_coords(buf, clip_ring=False))
    cont.rebuild(buf)
    out["cell0"] = cells.astype(np.int32)
    out["perm0"] = cont._perm.astype(np.int32)
    halo = L.build_halo(buf, box, params.interaction_length)
    out["halo_pos"] = halo.positions()
    out["halo_id"] = halo.id.copy()
    out["halo_cell"] = cont.linear_index(cont.cell_coords(halo, clip_ring=True)).astype(np.int32)
    for label, cfg in (("c08n3", Configuration(ContainerKind.LINKED_CELLS, TraversalKind.LC_C08,
                                               True, PatternKind.ONE_BY_V)),
                       ("c01", Configuration(ContainerKind.LINKED_CELLS, TraversalKind.LC_C01,
                                             False, PatternKind.V_BY_ONE))):
        b = buf.copy()
        st = force_phase(b, box, params, cfg, 8)
        out[f"F0_{label}"] = b.forces()
        out[f"stats0_{label}"] = np.array([st.kernel_invocations, st.lane_slots,
                                           st.useful_interactions, st.pair_interactions])
    # 1 force evaluation + 10 velocity-Verlet steps with LC c08 Newton3
    cfg = Configuration(ContainerKind.LINKED_CELLS, TraversalKind.LC_C08, True,
                        PatternKind.ONE_BY_V)
    force_phase(buf, box, params, cfg, 8)
    pairs = []
    for _ in range(10):
        velocity_verlet_step(buf, params, PRE_FORCE)
        st = force_phase(buf, box, params, cfg, 8)
        pairs.append(st.pair_interactions)
        velocity_verlet_step(buf, params, POST_FORCE)
        apply_boundaries(buf, box)
    out["pos10"] = buf.positions()
    out["vel10"] = np.stack([buf.vel_x, buf.vel_y, buf.vel_z], axis=1)
    out["F10"] = buf.forces()
    out["pairs_per_step"] = np.array(pairs)
    np.savez_compressed(os.path.join(HERE, "config1.npz"), **out)


def functor(L):
    """compute_pair_vectorized on small buffers with halo/dummy entries."""
    from lanemd import compute_pair_vectorized
    from lanemd.kernels import PATTERN_ORDER
    rng = np.random.default_rng(7)
    params = L.LJParams(cutoff=2.5, skin=0.5)
    out = {}
    k = 0
    for ni, nj in ((37, 37), (21, 13), (1, 8), (33, 5), (0, 7)):
        pi = rng.uniform(0, 6.0, (ni, 3))
        pj = rng.uniform(0, 6.0, (nj, 3))
        own_i = np.zeros(ni, dtype=np.int8)
        own_j = np.zeros(nj, dtype=np.int8)
        if ni > 4:
            own_i[3] = 1
            own_i[-1] = 2
        if nj > 4:
            own_j[2] = 2
            own_j[4] = 1
        for same in (False, True):
            if same and ni != nj:
                continue
            for n3 in (False, True):
                for pat in PATTERN_ORDER:
                    for V in (4, 8, 16):
                        bi = make_buffer(L, pi)
                        bi.ownership[:] = own_i
                        if same:
                            bj = bi
                        else:
                            bj = make_buffer(L, pj)
                            bj.ownership[:] = own_j
                        st = compute_pair_vectorized(bi, bj, params, n3, same, pat, V)
                        out[f"c{k}_meta"] = np.array([ni, nj, int(same), int(n3),
                                                      PATTERN_ORDER.index(pat), V])
                        out[f"c{k}_pi"] = pi
                        out[f"c{k}_pj"] = pj
                        out[f"c{k}_oi"] = own_i
                        out[f"c{k}_oj"] = own_j
                        out[f"c{k}_fi"] = bi.forces()
                        out[f"c{k}_fj"] = bj.forces()
                        out[f"c{k}_stats"] = np.array([st.kernel_invocations, st.lane_slots,
                                                       st.useful_interactions,
                                                       st.pair_interactions])
                        k += 1
    out["count"] = np.array(k)
    np.savez_compressed(os.path.join(HERE, "functor.npz"), **out)


def clusters(L):
    """VerletClusterContainer structure for a small periodic instance."""
    rng = np.random.default_rng(11)
    pos = rng.uniform(0, 9.0, (150, 3))
    params = L.LJParams(cutoff=2.2, skin=0.4)
    box = L.SimulationBox(np.zeros(3), np.full(3, 9.0), (L.BoundaryKind.PERIODIC,) * 3)
    out = {"pos": pos}
    for M in (4, 8):
        buf = make_buffer(L, pos)
        cont = L.VerletClusterContainer(box, params, M)
        cont.rebuild(buf)
        halo = L.build_halo(buf, box, params.interaction_length)
        cont.refresh(buf, halo)
        out[f"M{M}_perm"] = cont._perm
        out[f"M{M}_slots"] = cont._slots
        out[f"M{M}_counts"] = cont._real_counts
        out[f"M{M}_amin"] = cont._aabb_min
        out[f"M{M}_amax"] = cont._aabb_max
        b = cont._backing
        out[f"M{M}_padded"] = np.stack([b.pos_x, b.pos_y, b.pos_z], axis=1)
        for n3 in (False, True):
            lists = cont.neighbor_lists[n3]
            flat = [(k, z) for k, zs in enumerate(lists) for z in zs]
            out[f"M{M}_pairs_n3{int(n3)}"] = np.array(flat, dtype=np.int64).reshape(-1, 2)
        links = [(k, h) for k, hs in enumerate(cont.halo_links) for h in hs]
        out[f"M{M}_halo_links"] = np.array(links, dtype=np.int64).reshape(-1, 2)
    np.savez_compressed(os.path.join(HERE, "clusters.npz"), **out)


def api_spec(L):
    """The scenario run by api(): a jittered lattice block, periodic box, a
    small mixed search space tuned with the deterministic laneops metric."""
    from lanemd.kernels import PatternKind
    from lanemd.scenario import CubeSource, ScenarioSpec
    from lanemd.traversals import TraversalKind
    from lanemd.tuning import ContainerKind
    box = L.SimulationBox(np.zeros(3), np.full(3, 9.6), (L.BoundaryKind.PERIODIC,) * 3)
    params = L.LJParams(cutoff=2.5, skin=0.3, dt=0.002)
    src = CubeSource(origin=np.full(3, 0.6), counts=(8, 8, 8), spacing=1.2,
                     velocity=np.array([0.1, -0.05, 0.0]), jitter=0.8)
    return ScenarioSpec(box=box, params=params, sources=[src], iterations=60, seed=7,
                        vector_width=8, cluster_size=4, rebuild_period=5,
                        samples_per_config=2, tuning_interval=30, reduction="mean",
                        metric="laneops",
                        containers=[ContainerKind.LINKED_CELLS,
                                    ContainerKind.VERLET_CLUSTER_LISTS],
                        traversals=[TraversalKind.LC_C01, TraversalKind.LC_C08,
                                    TraversalKind.VCL],
                        newton3_options=[False, True],
                        patterns=[PatternKind.ONE_BY_V, PatternKind.V_BY_ONE])


def api(L):
    """Standalone cluster API (containers.py:216-299) and the scenario
    driver (driver.py:75-313: build_initial_state, resolve_search_space,
    run_simulation) on small seeded inputs."""
    from lanemd.containers import build_cluster_neighbor_lists, build_clusters
    from lanemd.driver import build_initial_state, resolve_search_space, run_simulation
    out = {}
    rng = np.random.default_rng(21)
    pos = rng.uniform(0, 12.0, (300, 3))
    out["cl_pos"] = pos
    for M in (4, 8):
        buf = make_buffer(L, pos)
        cl = build_clusters(buf, M)
        out[f"cl{M}_ids"] = np.stack([c.buffer.id for c in cl])
        out[f"cl{M}_nreal"] = np.array([c.n_real for c in cl])
        out[f"cl{M}_amin"] = np.stack([c.aabb_min for c in cl])
        out[f"cl{M}_amax"] = np.stack([c.aabb_max for c in cl])
        out[f"cl{M}_pos"] = np.stack([c.buffer.positions() for c in cl])
        for n3 in (False, True):
            lists = build_cluster_neighbor_lists(cl, 2.7, n3)
            flat = [(k, z) for k, zs in enumerate(lists) for z in zs]
            out[f"cl{M}_pairs_n3{int(n3)}"] = np.array(flat, dtype=np.int64).reshape(-1, 2)
    spec = api_spec(L)
    b0 = build_initial_state(spec)
    out["init_pos"] = b0.positions()
    out["init_vel"] = np.stack([b0.vel_x, b0.vel_y, b0.vel_z], axis=1)
    out["space"] = np.array([c.label for c in resolve_search_space(spec)])
    records, summary = run_simulation(spec)
    out["rec_label"] = np.array([r.configuration.label for r in records])
    out["rec_phase"] = np.array([r.phase for r in records])
    out["rec_num"] = np.array([[r.metric_value, r.lane_slots, r.useful_interactions,
                                r.blank_lanes, r.pair_interactions] for r in records])
    out["sum_selections"] = np.array(summary.phase_selections)
    out["sum_metric_labels"] = np.array(list(summary.per_config_metric.keys()))
    out["sum_metric_values"] = np.array(list(summary.per_config_metric.values()))
    out["sum_cells"] = np.array([summary.initial_max_per_cell, summary.final_max_per_cell])
    out["sum_speed"] = np.array([summary.final_max_speed])
    np.savez_compressed(os.path.join(HERE, "api.npz"), **out)


def main():
    L = _ref()
    if len(sys.argv) > 1 and sys.argv[1] == "api":
        api(L)
        return
    instances(L)
    config1(L)
    functor(L)
    clusters(L)
    api(L)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
