"""Segmented staged Verlet lists (csrc/vls.cu), the default v_by_one path.

The lists hold every candidate within rc + skin of the build positions, the
inner segment those within rc + inner_skin; the force kernel runs the inner
segment alone while no particle moved inner_skin / 2 since the build, and
both segments afterwards (decided on the device).  Checked against the
oracle (the reference's force phase restated, oracle/lj_oracle.c) at the
CURRENT positions: pair counts exact, forces within the reference's
forces_close, energy / virial 1e-12 -- before any move, after moves that keep
the inner segment valid, and after moves that need the outer segment."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import forces_close, jittered_lattice
from oracle import oracle as O

import paper_2512_03565_b200 as B
from paper_2512_03565_b200 import LJParams, ParticleBuffer, PatternKind, SimulationBox

pytestmark = pytest.mark.gpu


def _state(rng, n, rho):
    span = (n / rho) ** (1 / 3)
    k = int(np.ceil(n ** (1 / 3)))
    pos = jittered_lattice(rng, (k, k, k), span / k, 0.3 * span / k)[:n]
    return pos, span


def _check(cont, buf, pos, span, periodic, params, n3):
    of, ost = O.force_phase_vl(pos, np.zeros(3), np.full(3, span), [periodic] * 3, params, n3,
                               "v_by_one", 8)
    st = cont.compute_forces("vl", n3, PatternKind.V_BY_ONE, 8, energy=True)
    cont.collect_forces(buf)
    f = buf.forces().cpu().numpy()
    assert st.pair_interactions == ost.pair_interactions
    assert forces_close(f, of)
    assert abs(st.epot - ost.epot) <= 1e-12 * abs(ost.epot)
    assert abs(st.virial - ost.virial) <= 1e-12 * abs(ost.virial)
    return st, f


@pytest.mark.parametrize("n3", [False, True])
@pytest.mark.parametrize("periodic", [True, False])
def test_segmented_lists_match_oracle_and_are_used(rng, periodic, n3):
    pos, span = _state(rng, 6000, 0.8)
    params = LJParams(cutoff=2.5, skin=0.3)
    box = SimulationBox.cube(span, periodic=periodic)
    prev = None
    for _ in range(2):
        cont = B.VerletListContainer(box, params)
        buf = ParticleBuffer.from_positions(pos, device="cuda")
        cont.rebuild(buf)
        cont.refresh(buf)
        st, f = _check(cont, buf, pos, span, periodic, params, n3)
        assert cont._vls_for("v_by_one", n3) is not None      # the segmented path ran
        _, ost = O.force_phase_vl(pos, np.zeros(3), np.full(3, span), [periodic] * 3, params,
                                  n3, "v_by_one", 8)
        assert (st.kernel_invocations, st.lane_slots, st.useful_interactions) == \
            ost.as_tuple()[:3]
        if prev is not None:
            assert np.array_equal(prev, f)                     # deterministic
        prev = f


@pytest.mark.parametrize("move", [0.02, 0.07, 0.14])
def test_segments_cover_moved_particles(rng, move):
    """Moves below inner_skin / 2 (0.05) run the inner segment, larger ones
    (up to skin / 2 = 0.15) need the outer segment -- exact either way."""
    pos, span = _state(rng, 8000, 0.8)
    params = LJParams(cutoff=2.5, skin=0.3)
    box = SimulationBox.cube(span, periodic=True)
    cont = B.VerletListContainer(box, params)
    buf = ParticleBuffer.from_positions(pos, device="cuda")
    cont.rebuild(buf)
    cont.refresh(buf)
    cont.ensure_lists("v_by_one", False)
    d = rng.normal(size=pos.shape)
    d *= (move * 0.999) / np.linalg.norm(d, axis=1, keepdims=True)
    moved = pos + d
    for ax, t in enumerate((buf.pos_x, buf.pos_y, buf.pos_z)):
        t.copy_(torch.from_numpy(np.ascontiguousarray(moved[:, ax])))
    cont.refresh(buf)
    assert cont._vls_outer() == (move >= 0.05)
    _check(cont, buf, moved, span, True, params, False)


def test_inner_skin_equal_to_skin_and_zero(rng):
    """Degenerate segmentations: everything inner (inner_skin >= skin) or
    everything outer (inner_skin = 0: the inner segment holds r < rc)."""
    pos, span = _state(rng, 5000, 0.7)
    params = LJParams(cutoff=2.5, skin=0.3)
    box = SimulationBox.cube(span, periodic=True)
    for inner in (0.3, 0.0):
        cont = B.VerletListContainer(box, params)
        cont.inner_skin = inner
        buf = ParticleBuffer.from_positions(pos, device="cuda")
        cont.rebuild(buf)
        cont.refresh(buf)
        _check(cont, buf, pos, span, True, params, False)


def test_collect_fused_and_overlap(rng):
    """Forces written straight into the caller's order (launch_force(out=)),
    and a coincident pair raises ParticleOverlapError as the reference does."""
    pos, span = _state(rng, 4000, 0.6)
    params = LJParams(cutoff=2.5, skin=0.3)
    box = SimulationBox.cube(span, periodic=True)
    of, _ = O.force_phase_vl(pos, np.zeros(3), np.full(3, span), [True] * 3, params, False,
                             "v_by_one", 8)
    cont = B.VerletListContainer(box, params)
    buf = ParticleBuffer.from_positions(pos, device="cuda")
    cont.rebuild(buf)
    cont.refresh(buf)
    cont.launch_force("v_by_one", False, out=buf)
    cont.collect_forces(buf)
    assert forces_close(buf.forces().cpu().numpy(), of)
    bad = pos.copy()
    bad[1] = bad[0]
    buf2 = ParticleBuffer.from_positions(bad, device="cuda")
    cont2 = B.VerletListContainer(box, params)
    cont2.rebuild(buf2)
    cont2.refresh(buf2)
    with pytest.raises(B.ParticleOverlapError):
        cont2.compute_forces("vl", False, PatternKind.V_BY_ONE, 8)


def test_overlapped_ghost_exchange_matches_plain_refresh(rng):
    """launch_force_overlapped (interior groups on a side stream while the
    ghost rows are produced, boundary groups after) gives bitwise the forces
    and exactly the statistics of refresh + launch with an external ghost
    layer (here: the periodic images as the ghost layer)."""
    pos, span = _state(rng, 60000, 0.8)    # 15 cells per line: interior groups exist
    params = LJParams(cutoff=2.5, skin=0.3)
    box = SimulationBox.cube(span, periodic=True)
    buf = ParticleBuffer.from_positions(pos, device="cuda")
    halo = B.build_halo(buf, box, params.interaction_length)
    rows = torch.stack([halo.pos_x, halo.pos_y, halo.pos_z], 1).contiguous()
    inner = SimulationBox.cube(span, periodic=False)   # ghosts supply the images
    res = []
    for overlapped in (False, True):
        cont = B.VerletListContainer(inner, params)
        cont.rebuild(buf, halo)
        cont.refresh(buf, rows)
        cont.ensure_lists("v_by_one", False)
        parts = cont._vls_parts(cont._vls_for("v_by_one", False)["plan"])
        assert parts["interior"].numel() > 0 and parts["boundary"].numel() > 0
        if overlapped:
            st_t = cont.launch_force_overlapped(buf, lambda: rows, "v_by_one", False, energy=True)
        else:
            cont.refresh(buf, rows)
            st_t = cont.launch_force("v_by_one", False, energy=True)
        st = B._native.read_stats(st_t)
        cont.collect_forces(buf)
        res.append((buf.forces().cpu().numpy(), st.pair_interactions, st.epot, st.virial))
    assert np.array_equal(res[0][0], res[1][0])
    assert res[0][1:] == res[1][1:]
    of, ost = O.force_phase_vl(pos, np.zeros(3), np.full(3, span), [True] * 3, params, False,
                               "v_by_one", 8)
    assert res[1][1] == ost.pair_interactions and forces_close(res[1][0], of)


def test_capacity_retry_and_reuse(rng):
    """A list capacity that is too small for the build (here forced to the
    minimum) is detected on the device and the build redone at the observed
    maximum; the next rebuild reuses the learnt capacity.  Same results."""
    pos, span = _state(rng, 5000, 0.8)
    params = LJParams(cutoff=2.5, skin=0.3)
    box = SimulationBox.cube(span, periodic=True)
    cont = B.VerletListContainer(box, params)
    cont._vls_cap = 8
    buf = ParticleBuffer.from_positions(pos, device="cuda")
    cont.rebuild(buf)
    cont.refresh(buf)
    _check(cont, buf, pos, span, True, params, False)
    assert cont._vls_for("v_by_one", False) is not None
    learnt = cont._vls_cap
    assert learnt > 8
    cont.rebuild(buf)
    cont.refresh(buf)
    _check(cont, buf, pos, span, True, params, False)
    assert cont._vls_cap == learnt


def test_lists_too_long_for_segments_fall_back(rng):
    """More than 248 candidates within rc + skin of a particle (a dense
    state with a long cutoff) do not fit the segmented lists' 8-bit lane
    counters: the container serves such a state from the round-1 staged /
    global-gather lists instead, with the same results."""
    pos, span = _state(rng, 4000, 1.0)
    params = LJParams(cutoff=3.9, skin=0.3)      # ~310 neighbours within 4.2
    box = SimulationBox.cube(span, periodic=True)
    cont = B.VerletListContainer(box, params)
    buf = ParticleBuffer.from_positions(pos, device="cuda")
    cont.rebuild(buf)
    cont.refresh(buf)
    _check(cont, buf, pos, span, True, params, False)
    assert cont._vls_for("v_by_one", False) is None


@pytest.mark.parametrize("rho", [0.02, 0.1])
def test_sparse_states_with_groups_over_many_cells(rng, rho):
    """Dilute states: a group of 128 particles spans many cells of its line
    (or whole lines hold a handful of particles); groups shrink to the
    staging budget and empty runs are skipped."""
    pos, span = _state(rng, 3000, rho)
    params = LJParams(cutoff=2.5, skin=0.3)
    box = SimulationBox.cube(span, periodic=True)
    for n3 in (False, True):
        cont = B.VerletListContainer(box, params)
        buf = ParticleBuffer.from_positions(pos, device="cuda")
        cont.rebuild(buf)
        cont.refresh(buf)
        _check(cont, buf, pos, span, True, params, n3)
        assert cont._vls_for("v_by_one", n3) is not None


def test_adaptive_single_segment_after_a_long_epoch(rng):
    """An epoch that ended with a displacement of at least inner_skin (the
    outer segment ran for most of its steps) is followed by one-segment lists;
    a short epoch by two segments again.  Same results either way."""
    pos, span = _state(rng, 5000, 0.8)
    params = LJParams(cutoff=2.5, skin=0.3)
    box = SimulationBox.cube(span, periodic=True)
    cont = B.VerletListContainer(box, params, rebuild_period=1000)
    buf = ParticleBuffer.from_positions(pos, device="cuda")
    cont.rebuild(buf)
    cont.refresh(buf)
    cont.ensure_lists("v_by_one", False)
    vls = cont._vls_for("v_by_one", False)
    ng = vls["plan"]["ngroups"]
    assert int(vls["segc"][: 8 * ng].view(-1, 2)[:, 1].sum()) > 0      # two segments
    buf.pos_x[17] += 0.16                                              # >= skin / 2: rebuild due
    assert cont.refresh_and_check(buf) is True
    cont.rebuild(buf)
    cont.refresh(buf)
    now = buf.positions().cpu().numpy()
    _check(cont, buf, now, span, True, params, False)
    vls = cont._vls_for("v_by_one", False)
    ng = vls["plan"]["ngroups"]
    assert int(vls["segc"][: 8 * ng].view(-1, 2)[:, 1].sum()) == 0     # one segment
    buf.pos_x[17] += 0.01                                              # a short epoch
    assert cont.refresh_and_check(buf) is False
    cont.steps_since_rebuild = 1000
    assert cont.refresh_and_check(buf) is True                         # the period rule
    cont.rebuild(buf)
    cont.refresh(buf)
    _check(cont, buf, buf.positions().cpu().numpy(), span, True, params, False)
    vls = cont._vls_for("v_by_one", False)
    ng = vls["plan"]["ngroups"]
    assert int(vls["segc"][: 8 * ng].view(-1, 2)[:, 1].sum()) > 0


@pytest.mark.parametrize("n3", [False, True])
@pytest.mark.parametrize("periodic", [True, False])
def test_list_free_one_shot_kernel_matches_oracle(rng, periodic, n3):
    """The one-shot path of force_phase (lmd_vls_direct: no lists written)
    gives the oracle's pair counts, list statistics, forces, energy and
    virial, and the same forces as the list path to summation order."""
    pos, span = _state(rng, 6000, 0.8)
    params = LJParams(cutoff=2.5, skin=0.3)
    box = SimulationBox.cube(span, periodic=periodic)
    of, ost = O.force_phase_vl(pos, np.zeros(3), np.full(3, span), [periodic] * 3, params, n3,
                               "v_by_one", 8)
    cont = B.VerletListContainer(box, params)
    buf = ParticleBuffer.from_positions(pos, device="cuda")
    cont.rebuild(buf)
    cont.refresh(buf)
    st = cont.compute_forces_once("vl", n3, PatternKind.V_BY_ONE, 8, energy=True)
    assert st is not None and not cont._lists and not cont._vls        # nothing was built
    cont.collect_forces(buf)
    f = buf.forces().cpu().numpy()
    assert (st.kernel_invocations, st.lane_slots, st.useful_interactions,
            st.pair_interactions) == ost.as_tuple()
    assert forces_close(f, of)
    assert abs(st.epot - ost.epot) <= 1e-12 * abs(ost.epot)
    assert abs(st.virial - ost.virial) <= 1e-12 * abs(ost.virial)
    # and through the public entry point
    buf2 = ParticleBuffer.from_positions(pos, device="cuda")
    st2 = B.force_phase(buf2, box, params, B.Configuration.parse(
        f"vl,vl,{str(n3).lower()},v_by_one"), 8)
    assert st2.pair_interactions == ost.pair_interactions
    assert np.array_equal(buf2.forces().cpu().numpy(), f)


def test_list_free_kernel_capacity_retry_and_overlap(rng):
    pos, span = _state(rng, 3000, 0.9)
    params = LJParams(cutoff=3.2, skin=0.3)            # more hits than the first guess
    box = SimulationBox.cube(span, periodic=True)
    of, ost = O.force_phase_vl(pos, np.zeros(3), np.full(3, span), [True] * 3, params, False,
                               "v_by_one", 8)
    buf = ParticleBuffer.from_positions(pos, device="cuda")
    st = B.force_phase(buf, box, params, B.Configuration.parse("vl,vl,false,v_by_one"), 8)
    assert st.pair_interactions == ost.pair_interactions
    assert forces_close(buf.forces().cpu().numpy(), of)
    pos2 = pos.copy()
    pos2[11] = pos2[10]                                # coincident particles
    buf = ParticleBuffer.from_positions(pos2, device="cuda")
    with pytest.raises(B.ParticleOverlapError):
        B.force_phase(buf, box, params, B.Configuration.parse("vl,vl,false,v_by_one"), 8)


def test_external_ghost_layer_tracks_displacement_for_the_inner_segment(rng):
    """With a decomposition's ghost layer the inner segment is used while
    neither an owned particle nor a ghost has moved inner_skin / 2 since the
    build (the ghost rows' displacements are reduced on the device as they
    are refreshed), and both segments afterwards; results equal the
    self-imaged container's either way."""
    pos, span = _state(rng, 5000, 0.8)
    params = LJParams(cutoff=2.5, skin=0.3)
    box = SimulationBox.cube(span, periodic=True)
    from paper_2512_03565_b200.domain import build_halo
    for move_ghost in (0.0, 0.02, 0.09):
        buf = ParticleBuffer.from_positions(pos, device="cuda")
        halo = build_halo(buf, box, params.interaction_length)
        ext = B.VerletListContainer(box, params)
        ext.rebuild(buf, halo)
        ext.refresh(buf, halo)
        ext.ensure_lists("v_by_one", False)
        # move one owned particle near a face together with its images
        k = int(torch.argmin(buf.pos_x))
        buf.pos_x[k] += move_ghost
        halo2 = build_halo(buf, box, params.interaction_length)
        assert len(halo2) == len(halo)
        ext.refresh(buf, halo2)
        assert ext._disp_slot >= 0
        assert ext._vls_outer() == (move_ghost >= 0.05)
        st = ext.compute_forces("vl", False, PatternKind.V_BY_ONE, 8)
        ext.collect_forces(buf)
        now = buf.positions().cpu().numpy()
        of, ost = O.force_phase_vl(now, np.zeros(3), np.full(3, span), [True] * 3, params, False,
                                   "v_by_one", 8)
        assert st.pair_interactions == ost.pair_interactions
        assert forces_close(buf.forces().cpu().numpy(), of)
