"""The CPU oracle is pinned against the reference's own outputs.

Golden fixtures (tests/golden/*.npz) were produced by the unmodified
reference package; the oracle must reproduce them BIT FOR BIT (forces) and
exactly (statistics, cell assignment, permutations, halo images, cluster
structure).  When the reference itself is importable (this container only)
extra randomized instances are compared live.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np
import pytest

from conftest import (P, REFERENCE_SRC, brute_energy_virial, brute_forces, forces_close,
                      golden, jittered_lattice)
from oracle import oracle as O

PATTERNS = ("one_by_v", "v_by_one", "two_by_half", "half_by_two")


def _cfg(label):
    cont, trav, n3, pat = label.split(",")
    return cont, trav, n3 == "true", pat


def _run(pos, span, periodic, params, label, V):
    cont, trav, n3, pat = _cfg(label)
    lo, hi = np.zeros(3), np.full(3, span)
    if cont == "lc":
        return O.force_phase_lc(pos, lo, hi, [periodic] * 3, params, trav, n3, pat, V)
    return O.force_phase_vcl(pos, lo, hi, [periodic] * 3, params, V, n3, pat, V)


def test_oracle_matches_reference_instances_bitwise():
    g = golden("instances.npz")
    labels = [str(x) for x in g["labels"]]
    assert len(labels) == 28
    for k in range(8):
        pos = g[f"i{k}_pos"]
        span, periodic, cutoff, skin = g[f"i{k}_box"]
        params = P(cutoff=cutoff, skin=skin)
        stats = g[f"i{k}_stats"]
        for ci, label in enumerate(labels):
            for vi, V in enumerate((4, 8, 16)):
                f, st = _run(pos, span, bool(periodic), params, label, V)
                assert st.as_tuple() == tuple(stats[ci, vi]), (k, label, V)
                pkey = label.rsplit(",", 1)[0] + (f",M{V}" if label.startswith("vcl") else "")
                assert np.array_equal(f, g[f"i{k}_F_{pkey}"]), (k, label, V)


def test_oracle_config1_cells_halo_forces_and_trajectory():
    g = golden("config1.npz")
    pos = g["pos0"]
    params = P(cutoff=2.5, skin=0.0)
    lo, hi = np.zeros(3), np.full(3, 22.0)
    cell, perm, dims = O.lc_bin(pos, lo, hi, 2.5)
    assert dims.tolist() == [8, 8, 8]
    assert np.array_equal(cell, g["cell0"])
    assert np.array_equal(perm, g["perm0"])
    hpos, hid = O.build_halo(pos, lo, hi, [True] * 3, 2.5)
    assert np.array_equal(hpos, g["halo_pos"]) and np.array_equal(hid, g["halo_id"])
    hcell, _, _ = O.lc_bin(hpos, lo, hi, 2.5, ring=True)
    assert np.array_equal(hcell, g["halo_cell"])
    f, st = O.force_phase_lc(pos, lo, hi, [True] * 3, params, "lc_c08", True, "one_by_v", 8)
    assert np.array_equal(f, g["F0_c08n3"])
    assert st.as_tuple() == tuple(g["stats0_c08n3"])
    assert st.pair_interactions == 250764
    f, st = O.force_phase_lc(pos, lo, hi, [True] * 3, params, "lc_c01", False, "v_by_one", 8)
    assert np.array_equal(f, g["F0_c01"])
    assert st.as_tuple() == tuple(g["stats0_c01"])
    assert st.pair_interactions == 448000
    # 1 force evaluation + 10 velocity-Verlet steps (BASELINE config 1)
    s = {k: np.ascontiguousarray(v) for k, v in zip(("x", "y", "z"), pos.T)}
    s.update({k: np.ascontiguousarray(v) for k, v in zip(("vx", "vy", "vz"), g["vel0"].T)})
    f, _ = O.force_phase_lc(pos, lo, hi, [True] * 3, params, "lc_c08", True, "one_by_v", 8)
    s.update({k: np.ascontiguousarray(v) for k, v in zip(("fx", "fy", "fz"), f.T)})
    s.update({k: np.zeros(len(pos)) for k in ("ox", "oy", "oz")})
    pairs = []
    for _ in range(10):
        O.verlet(s, 0, 0.001, 1.0)
        p = np.stack([s["x"], s["y"], s["z"]], axis=1)
        f, st = O.force_phase_lc(p, lo, hi, [True] * 3, params, "lc_c08", True, "one_by_v", 8)
        pairs.append(st.pair_interactions)
        s["fx"][:], s["fy"][:], s["fz"][:] = f.T
        O.verlet(s, 1, 0.001, 1.0)
        assert not O.apply_boundaries(s, lo, hi, [True] * 3)
    assert pairs == g["pairs_per_step"].tolist()
    assert np.array_equal(np.stack([s["x"], s["y"], s["z"]], axis=1), g["pos10"])
    assert np.array_equal(np.stack([s["vx"], s["vy"], s["vz"]], axis=1), g["vel10"])
    assert np.array_equal(np.stack([s["fx"], s["fy"], s["fz"]], axis=1), g["F10"])


def test_oracle_functor_bitwise():
    g = golden("functor.npz")
    params = P(cutoff=2.5, skin=0.5)
    for k in range(int(g["count"])):
        ni, nj, same, n3, pi_, V = g[f"c{k}_meta"].tolist()
        fi, fj, st = O.pair_sweep(g[f"c{k}_pi"], g[f"c{k}_pj"], params, bool(n3), bool(same),
                                  PATTERNS[pi_], V, own_i=g[f"c{k}_oi"], own_j=g[f"c{k}_oj"])
        assert np.array_equal(fi, g[f"c{k}_fi"]), k
        if not same:
            assert np.array_equal(fj, g[f"c{k}_fj"]), k
        assert st.as_tuple() == tuple(g[f"c{k}_stats"]), k


def test_oracle_cluster_structure():
    g = golden("clusters.npz")
    pos = g["pos"]
    for M in (4, 8):
        s = O.vcl_structure(pos, np.zeros(3), np.full(3, 9.0), 2.6, M)
        assert np.array_equal(s["order"], g[f"M{M}_perm"])
        assert np.array_equal(s["slots"], g[f"M{M}_slots"])
        assert np.array_equal(s["counts"], g[f"M{M}_counts"])
        assert np.array_equal(s["aabb_min"], g[f"M{M}_amin"])
        assert np.array_equal(s["aabb_max"], g[f"M{M}_amax"])
        assert np.array_equal(s["padded"], g[f"M{M}_padded"])


@pytest.mark.parametrize("periodic", [False, True])
def test_oracle_energy_virial_vs_all_pairs(rng, periodic):
    pos = jittered_lattice(rng, (6, 6, 6), 1.15, 0.12)
    span = 6 * 1.15
    params = P(cutoff=2.2, skin=0.3)
    L = np.full(3, span) if periodic else None
    ref_f = brute_forces(pos, params, L)
    e_ref, w_ref = brute_energy_virial(pos, params, L)
    lo, hi = np.zeros(3), np.full(3, span)
    for trav, n3 in (("lc_c01", False), ("lc_c08", True), ("lc_c18", False)):
        f, st = O.force_phase_lc(pos, lo, hi, [periodic] * 3, params, trav, n3, "one_by_v", 8)
        assert forces_close(f, ref_f)
        assert abs(st.epot - e_ref) <= 1e-12 * abs(e_ref)
        assert abs(st.virial - w_ref) <= 1e-12 * max(abs(w_ref), 1.0)
    for n3 in (False, True):
        f, st = O.force_phase_vl(pos, lo, hi, [periodic] * 3, params, n3, "one_by_v", 8)
        assert forces_close(f, ref_f)
        assert abs(st.epot - e_ref) <= 1e-12 * abs(e_ref)


@pytest.mark.parametrize("periodic", [False, True])
def test_oracle_verlet_list_pairs_exact(rng, periodic):
    span = 9.0
    pos = rng.uniform(0, span, (300, 3))
    length = 2.6
    lo, hi = np.zeros(3), np.full(3, span)
    pi, pj, ph = O.vl_pairs(pos, lo, hi, [periodic] * 3, length, False)
    got = set(zip(pi.tolist(), pj.tolist()))
    assert len(got) == len(pi)
    d = pos[:, None, :] - pos[None, :, :]
    if periodic:
        d -= span * np.round(d / span)
    r2 = (d ** 2).sum(axis=2)
    np.fill_diagonal(r2, np.inf)
    want = set(zip(*np.nonzero(r2 < length * length)))
    assert got == {(int(a), int(b)) for a, b in want}
    # half lists: every unordered owned pair once, halo pairs from both sides
    hi_, hj, hh = O.vl_pairs(pos, lo, hi, [periodic] * 3, length, True)
    owned_pairs = {frozenset((a, b)) for a, b, h in zip(hi_.tolist(), hj.tolist(), hh.tolist())
                   if not h}
    n_owned_half = int((hh == 0).sum())
    assert len(owned_pairs) == n_owned_half
    assert n_owned_half * 2 + int((hh == 1).sum()) == len(pi)


def test_oracle_verlet_lists_match_linked_cells(rng):
    pos = jittered_lattice(rng, (7, 7, 7), 1.1, 0.2)
    span = 7 * 1.1
    params = P(cutoff=2.5, skin=0.3)
    lo, hi = np.zeros(3), np.full(3, span)
    f_lc, s_lc = O.force_phase_lc(pos, lo, hi, [True] * 3, params, "lc_c01", False, "one_by_v", 8)
    for n3 in (False, True):
        f, st = O.force_phase_vl(pos, lo, hi, [True] * 3, params, n3, "one_by_v", 8)
        assert forces_close(f, f_lc)
    f, st = O.force_phase_vl(pos, lo, hi, [True] * 3, params, False, "one_by_v", 8)
    assert st.pair_interactions == s_lc.pair_interactions


def test_oracle_overlap_is_reported():
    pos = np.array([[1.0, 1.0, 1.0], [1.0, 1.0, 1.0], [3.0, 3.0, 3.0]])
    with pytest.raises(O.OracleError) as exc:
        O.force_phase_lc(pos, np.zeros(3), np.full(3, 9.0), [False] * 3, P(cutoff=2.2, skin=0.4),
                         "lc_c08", True, "one_by_v", 8)
    assert exc.value.code == O.OVERLAP


@pytest.mark.skipif(not os.path.isdir(REFERENCE_SRC), reason="reference not mounted")
def test_oracle_live_against_reference_random():
    sys.path.insert(0, REFERENCE_SRC)
    import lanemd
    from lanemd.driver import force_phase
    from lanemd.kernels import PATTERN_ORDER
    from lanemd.traversals import TraversalKind
    from lanemd.tuning import ContainerKind, enumerate_search_space
    configs = enumerate_search_space(
        [ContainerKind.LINKED_CELLS, ContainerKind.VERLET_CLUSTER_LISTS],
        [TraversalKind.LC_C01, TraversalKind.LC_C08, TraversalKind.LC_C18, TraversalKind.VCL],
        [False, True], list(PATTERN_ORDER))
    rng = np.random.default_rng(99)
    for trial in range(4):
        n = int(rng.integers(16, 300))
        dens = rng.uniform(0.2, 0.7)
        span = (n / dens) ** (1 / 3)
        pa = math.ceil(n ** (1 / 3))
        sp = span / pa
        pos = jittered_lattice(rng, (pa,) * 3, sp, 0.25 * sp)[:n]
        cutoff = float(min(rng.uniform(1.5, 3.0), span / 2.2))
        periodic = bool(trial % 2)
        kind = lanemd.BoundaryKind.PERIODIC if periodic else lanemd.BoundaryKind.REFLECTIVE
        box = lanemd.SimulationBox(np.zeros(3), np.full(3, span), (kind,) * 3)
        params = lanemd.LJParams(cutoff=cutoff, skin=0.2 * cutoff)
        for cfg in configs:
            buf = lanemd.ParticleBuffer.empty(n)
            buf.pos_x[:], buf.pos_y[:], buf.pos_z[:] = pos.T
            buf.id[:] = np.arange(n)
            st = force_phase(buf, box, params, cfg, 8)
            f, ost = _run(pos, span, periodic, params, cfg.label, 8)
            assert np.array_equal(f, buf.forces()), cfg.label
            assert ost.as_tuple() == (st.kernel_invocations, st.lane_slots,
                                      st.useful_interactions, st.pair_interactions)
