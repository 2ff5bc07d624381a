"""Reference schedules on the device containers and execute_packed.

Coverage/coloring mirrors the reference's traversal tests (acceptance
criterion 5); execute_packed must reproduce the oracle's statistics exactly
and its forces within forces_close."""

from __future__ import annotations

import itertools

import numpy as np
import pytest

from conftest import forces_close, golden
from oracle import oracle as O

import paper_2512_03565_b200 as B
from paper_2512_03565_b200 import (LJParams, ParticleBuffer, PatternKind, SimulationBox,
                                   TraversalKind, execute_packed, pack_schedule, schedule,
                                   verify_coloring)

pytestmark = pytest.mark.gpu
PARAMS = LJParams(cutoff=2.0, skin=0.5)  # cell side 2.5


def _full_grid(n):
    box = SimulationBox(np.zeros(3), np.full(3, 2.5 * n), ("reflective",) * 3)
    cont = B.LinkedCellsContainer(box, PARAMS)
    centers = (np.stack(np.meshgrid(*[np.arange(n)] * 3, indexing="ij"), -1)
               .reshape(-1, 3) * 2.5 + 1.25)
    buf = ParticleBuffer.from_positions(centers, device="cuda")
    cont.rebuild(buf)
    cont.refresh(buf, ParticleBuffer.empty(0, device="cuda"))
    return cont


def _adjacent(cont):
    tx, ty, _ = cont.total_dims
    coords = {lin: (lin % tx, (lin // tx) % ty, lin // (tx * ty))
              for lin in cont.owned_occupied.tolist()}
    return {frozenset((a, b)) for a, b in itertools.combinations(coords, 2)
            if all(abs(coords[a][k] - coords[b][k]) <= 1 for k in range(3))}, coords


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_traversal_coverage_and_coloring(n):
    cont = _full_grid(n)
    adj, coords = _adjacent(cont)
    for kind in (TraversalKind.LC_C08, TraversalKind.LC_C18):
        sched = schedule(cont, kind, True)
        assert verify_coloring(sched)
        pairs = [frozenset((u.i_index, u.j_index)) for u in sched.units if not u.same_buffer]
        assert len(pairs) == len(set(pairs)) and set(pairs) == adj
        assert sum(u.same_buffer for u in sched.units) == n ** 3
        assert verify_coloring(schedule(cont, kind, False))
    c01 = schedule(cont, TraversalKind.LC_C01, False)
    ordered = [(u.i_index, u.j_index) for u in c01.units]
    want = {(a, b) for p in adj for a, b in itertools.permutations(tuple(p), 2)}
    want |= {(c, c) for c in coords}
    assert len(ordered) == len(set(ordered)) and set(ordered) == want
    with pytest.raises(B.ConfigurationError):
        schedule(cont, TraversalKind.LC_C01, True)


def test_c08_and_c18_choose_different_i_sides():
    cont = _full_grid(4)
    c08 = {frozenset((u.i_index, u.j_index)): u.i_index
           for u in schedule(cont, TraversalKind.LC_C08, True).units if not u.same_buffer}
    c18 = {frozenset((u.i_index, u.j_index)): u.i_index
           for u in schedule(cont, TraversalKind.LC_C18, True).units if not u.same_buffer}
    assert set(c08) == set(c18)
    assert any(c08[p] != c18[p] for p in c08)
    assert all(c18[p] == min(p) for p in c18)


def test_execute_packed_matches_oracle_all_traversals():
    g = golden("instances.npz")
    for k in (1, 4, 5):
        pos = g[f"i{k}_pos"]
        span, periodic, cutoff, skin = g[f"i{k}_box"]
        box = SimulationBox.cube(float(span), periodic=bool(periodic))
        params = LJParams(cutoff=float(cutoff), skin=float(skin))
        lo, hi = np.zeros(3), np.full(3, float(span))
        for trav, n3 in (("lc_c01", False), ("lc_c08", True), ("lc_c18", True),
                         ("lc_c18", False)):
            for pat in (PatternKind.TWO_BY_HALF, PatternKind.V_BY_ONE):
                cont = B.LinkedCellsContainer(box, params)
                buf = ParticleBuffer.from_positions(pos, device="cuda")
                cont.rebuild(buf)
                cont.refresh(buf)
                sched = schedule(cont, trav, n3)
                assert verify_coloring(sched)
                packed = pack_schedule(sched)
                own, hal = cont.kernel_backings()
                st = execute_packed(packed, own, hal, params, pat, 8)
                cont.collect_forces(buf)
                of, ost = O.force_phase_lc(pos, lo, hi, [bool(periodic)] * 3, params, trav, n3,
                                           pat.value, 8)
                assert (st.kernel_invocations, st.lane_slots, st.useful_interactions,
                        st.pair_interactions) == ost.as_tuple(), (k, trav, n3, pat)
                assert forces_close(buf.forces().cpu().numpy(), of), (k, trav, n3, pat)
        for n3 in (False, True):
            cont = B.VerletClusterContainer(box, params, 8)
            buf = ParticleBuffer.from_positions(pos, device="cuda")
            cont.rebuild(buf)
            cont.refresh(buf)
            sched = schedule(cont, "vcl", n3)
            assert verify_coloring(sched)
            own, hal = cont.kernel_backings()
            st = execute_packed(pack_schedule(sched), own, hal, params, PatternKind.HALF_BY_TWO, 8)
            cont.collect_forces(buf)
            of, ost = O.force_phase_vcl(pos, lo, hi, [bool(periodic)] * 3, params, 8, n3,
                                        "half_by_two", 8)
            assert (st.kernel_invocations, st.lane_slots, st.useful_interactions,
                    st.pair_interactions) == ost.as_tuple(), (k, "vcl", n3)
            assert forces_close(buf.forces().cpu().numpy(), of), (k, "vcl", n3)
