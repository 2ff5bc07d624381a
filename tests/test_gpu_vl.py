"""GPU Verlet lists (north-star extension) against the oracle.

Bars: the neighbor-pair set is EXACTLY the oracle's (same exact-r2 rule);
forces within forces_close of the oracle; pair counts and lane statistics
exact; energy/virial 1e-12 relative; lists reused between rebuilds track a
from-scratch linked-cell evaluation at the moved positions.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import forces_close, jittered_lattice
from oracle import oracle as O

import paper_2512_03565_b200 as B
from paper_2512_03565_b200 import Configuration, LJParams, ParticleBuffer, PatternKind, SimulationBox

pytestmark = pytest.mark.gpu


def _state(rng, n, rho):
    side = int(round((n / rho) ** (1 / 3) / 1.0))
    span = (n / rho) ** (1 / 3)
    k = int(np.ceil(n ** (1 / 3)))
    pos = jittered_lattice(rng, (k, k, k), span / k, 0.3 * span / k)[:n]
    return pos, span


@pytest.mark.parametrize("periodic", [True, False])
def test_pair_sets_exact(rng, periodic):
    pos, span = _state(rng, 3000, 0.6)
    params = LJParams(cutoff=2.5, skin=0.3)
    box = SimulationBox.cube(span, periodic=periodic)
    cont = B.VerletListContainer(box, params)
    buf = ParticleBuffer.from_positions(pos, device="cuda")
    cont.rebuild(buf)
    for n3 in (False, True):
        gi, gj, gh = (t.cpu().numpy() for t in cont.pairs(n3))
        oi, oj, oh = O.vl_pairs(pos, np.zeros(3), np.full(3, span), [periodic] * 3, 2.8, n3)
        got = sorted(zip(gi.tolist(), gj.tolist(), gh.astype(int).tolist()))
        want = sorted(zip(oi.tolist(), oj.tolist(), oh.astype(int).tolist()))
        assert got == want


@pytest.mark.parametrize("n3_mode", ["full_list", "half_list"])
@pytest.mark.parametrize("pattern", list(PatternKind))
def test_forces_stats_energy_vs_oracle(rng, pattern, n3_mode):
    pos, span = _state(rng, 4000, 0.8)
    params = LJParams(cutoff=2.5, skin=0.3)
    box = SimulationBox.cube(span, periodic=True)
    lo, hi = np.zeros(3), np.full(3, span)
    for n3 in (False, True):
        for V in (8, 16):
            of, ost = O.force_phase_vl(pos, lo, hi, [True] * 3, params, n3, pattern.value, V)
            buf = ParticleBuffer.from_positions(pos, device="cuda")
            cont = B.VerletListContainer(box, params)
            cont.n3_mode = n3_mode
            cont.rebuild(buf)
            cont.refresh(buf)
            st = cont.compute_forces("vl", n3, pattern, V, energy=True)
            cont.collect_forces(buf)
            assert st == B.KernelStats(*ost.as_tuple()), (n3, V)
            assert forces_close(buf.forces().cpu().numpy(), of), (n3, V)
            assert abs(st.epot - ost.epot) <= 1e-12 * abs(ost.epot)
            assert abs(st.virial - ost.virial) <= 1e-12 * abs(ost.virial)


def test_lists_reused_between_rebuilds_match_fresh_linked_cells(rng):
    pos, span = _state(rng, 6000, 0.8)
    params = LJParams(cutoff=2.5, skin=0.3)
    box = SimulationBox.cube(span, periodic=True)
    cont = B.VerletListContainer(box, params)
    buf = ParticleBuffer.from_positions(pos, device="cuda")
    cont.rebuild(buf)
    moved = pos + rng.uniform(-0.07, 0.07, pos.shape)   # |disp| < skin/2
    moved = np.mod(moved, span)
    buf2 = ParticleBuffer.from_positions(moved, device="cuda")
    assert not cont.needs_rebuild(buf2)
    cont.refresh(buf2)
    st = cont.compute_forces("vl", False, PatternKind.TWO_BY_HALF, 8)
    cont.collect_forces(buf2)
    of, ost = O.force_phase_lc(moved, np.zeros(3), np.full(3, span), [True] * 3,
                               LJParams(cutoff=2.5, skin=0.0), "lc_c01", False, "one_by_v", 8)
    assert st.pair_interactions == ost.pair_interactions
    assert forces_close(buf2.forces().cpu().numpy(), of)


def test_vl_overlap_raises():
    pos = np.random.default_rng(3).uniform(0, 9, (40, 3))
    pos[7] = pos[3]
    cfg = Configuration.parse("vl,vl,false,one_by_v")
    with pytest.raises(B.ParticleOverlapError):
        B.force_phase(ParticleBuffer.from_positions(pos, device="cuda"),
                      SimulationBox.cube(9.0, periodic=False), LJParams(cutoff=2.2, skin=0.4),
                      cfg, 8)


def test_lists_for_a_new_pattern_use_rebuild_positions(rng):
    """A list built lazily after the particles moved must still be the
    rebuild-time list (tile sizes were counted then)."""
    pos, span = _state(rng, 5000, 0.8)
    params = LJParams(cutoff=2.5, skin=0.3)
    box = SimulationBox.cube(span, periodic=True)
    cont = B.VerletListContainer(box, params)
    buf = ParticleBuffer.from_positions(pos, device="cuda")
    cont.rebuild(buf)
    cont.refresh(buf)
    st1 = cont.compute_forces("vl", False, PatternKind.V_BY_ONE, 8)
    moved = np.mod(pos + rng.uniform(-0.07, 0.07, pos.shape), span)
    buf2 = ParticleBuffer.from_positions(moved, device="cuda")
    cont.refresh(buf2)
    for pat in PatternKind:
        st = cont.compute_forces("vl", False, pat, 8)
        assert st.useful_interactions == st1.useful_interactions
        of, ost = O.force_phase_lc(moved, np.zeros(3), np.full(3, span), [True] * 3,
                                   LJParams(cutoff=2.5, skin=0.0), "lc_c01", False, "one_by_v", 8)
        assert st.pair_interactions == ost.pair_interactions


@pytest.mark.parametrize("n3", [False, True])
def test_fused_collect_matches_scatter(rng, n3):
    """launch_force(out=buf) writes the forces straight into the caller's
    order (collect_forces fused); bitwise equal to launch + scatter."""
    pos, span = _state(rng, 3000, 0.8)
    params = LJParams(cutoff=2.5, skin=0.3)
    box = SimulationBox.cube(span, periodic=True)
    res = []
    for fused in (False, True):
        cont = B.VerletListContainer(box, params)
        buf = ParticleBuffer.from_positions(pos, device="cuda")
        cont.rebuild(buf)
        cont.refresh(buf)
        st = cont.launch_force(PatternKind.V_BY_ONE, n3, out=buf if fused else None)
        cont.collect_forces(buf)
        res.append((buf.forces().cpu().numpy(), cont.pair_count(B._native.read_stats(st), n3)))
    assert np.array_equal(res[0][0], res[1][0]) and res[0][1] == res[1][1]


@pytest.mark.parametrize("staged,bank,index16", [
    (0, -1, True), (128, -1, True), (128, 0, True), (128, 0, False), (128, 2, False),
    (256, 0, True), (512, 0, True), (0, 2, True), (256, 0, False)])
@pytest.mark.parametrize("n3", [False, True])
def test_staged_and_bank_ordered_lists_match_oracle(rng, staged, bank, index16, n3):
    """Staged lists (TMA copies of each group's candidate runs into shared
    memory, local rows) and the bank-pair-aware entry orders: pair counts,
    statistics and energy exact / 1e-12 vs the oracle, forces within
    tolerance, runs deterministic.  A dense, non-periodic corner case (groups
    crossing z-planes stage long runs) mixes staged and global-gather
    groups in one launch."""
    pos, span = _state(rng, 6000, 0.8)
    params = LJParams(cutoff=2.5, skin=0.3)
    for periodic in (True, False):
        box = SimulationBox.cube(span, periodic=periodic)
        of, ost = O.force_phase_vl(pos, np.zeros(3), np.full(3, span), [periodic] * 3, params, n3,
                                   "v_by_one", 8)
        prev = None
        for _ in range(2):
            cont = B.VerletListContainer(box, params)
            cont.segmented = False     # the round-1 staged path (fallback)
            cont.staged_group = staged
            cont.bank_rounds = bank
            cont.index16 = index16
            buf = ParticleBuffer.from_positions(pos, device="cuda")
            cont.rebuild(buf)
            cont.refresh(buf)
            st = cont.compute_forces("vl", n3, PatternKind.V_BY_ONE, 8, energy=True)
            cont.collect_forces(buf)
            f = buf.forces().cpu().numpy()
            assert (st.kernel_invocations, st.lane_slots, st.useful_interactions,
                    st.pair_interactions) == ost.as_tuple()[:4]
            assert abs(st.epot - ost.epot) <= 1e-12 * abs(ost.epot)
            assert forces_close(f, of)
            if prev is not None:
                assert np.array_equal(prev, f)
            prev = f
        if staged:
            groups, rows, g, over, bits = next(iter(cont._staging.values()))
            assert rows >= 16 and g == staged
            assert bits == (16 if (over == 0 and index16) else 32)
