"""GPU parity of the linked-cell force path against the oracle / golden fixtures.

Bars: cell assignment, permutation and halo cells bit-exact; pair counts and
lane statistics exact; forces within the reference's forces_close predicate
(|dF| <= 1e-12 * max(|F|_inf, 1)); energy/virial within 1e-12 relative.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import brute_energy_virial, forces_close, golden, jittered_lattice
from oracle import oracle as O

import paper_2512_03565_b200 as B
from paper_2512_03565_b200 import (Configuration, ContainerKind, LJParams, ParticleBuffer,
                                   PatternKind, SimulationBox, TraversalKind)

pytestmark = pytest.mark.gpu

PATTERNS = list(PatternKind)


def _box(span, periodic):
    return SimulationBox.cube(float(span), periodic=bool(periodic))


def _buf(pos):
    return ParticleBuffer.from_positions(pos, device="cuda")


def test_cell_binning_and_halo_bit_exact():
    g = golden("config1.npz")
    pos = g["pos0"]
    box = _box(22.0, True)
    params = LJParams(cutoff=2.5, skin=0.0)
    cont = B.LinkedCellsContainer(box, params)
    buf = _buf(pos)
    cell = cont.cell_index(buf).cpu().numpy()
    assert np.array_equal(cell, g["cell0"])
    cont.rebuild(buf)
    assert np.array_equal(cont._perm.cpu().numpy(), g["perm0"])
    halo = B.build_halo(buf, box, params.interaction_length)
    hpos = halo.positions().cpu().numpy()
    hid = halo.id.cpu().numpy()
    # same image set (the device emits (owner, shift) order, the reference (shift, owner))
    got = sorted(zip(hid.tolist(), map(tuple, hpos.tolist())))
    want = sorted(zip(g["halo_id"].tolist(), map(tuple, g["halo_pos"].tolist())))
    assert got == want
    hcell = cont.cell_index(halo, clip_ring=True).cpu().numpy()
    want_cell = dict(zip(map(tuple, g["halo_pos"].tolist()), g["halo_cell"].tolist()))
    assert all(want_cell[tuple(p)] == c for p, c in zip(hpos.tolist(), hcell.tolist()))


def test_instances_all_lc_configs_match_reference():
    g = golden("instances.npz")
    labels = [str(x) for x in g["labels"]]
    for k in range(8):
        pos = g[f"i{k}_pos"]
        span, periodic, cutoff, skin = g[f"i{k}_box"]
        box = _box(span, periodic)
        params = LJParams(cutoff=float(cutoff), skin=float(skin))
        stats = g[f"i{k}_stats"]
        for ci, label in enumerate(labels):
            if not label.startswith("lc,"):
                continue
            cfg = Configuration.parse(label)
            ref = g[f"i{k}_F_{label.rsplit(',', 1)[0]}"]
            for vi, V in enumerate((4, 8, 16)):
                buf = _buf(pos)
                st = B.force_phase(buf, box, params, cfg, V)
                got = (st.kernel_invocations, st.lane_slots, st.useful_interactions,
                       st.pair_interactions)
                assert got == tuple(stats[ci, vi]), (k, label, V)
                assert forces_close(buf.forces().cpu().numpy(), ref), (k, label, V)


def test_config1_forces_stats_and_host_buffers():
    g = golden("config1.npz")
    box = _box(22.0, True)
    params = LJParams(cutoff=2.5, skin=0.0)
    cases = (("c08n3", "lc,lc_c08,true,one_by_v", 250764),
             ("c01", "lc,lc_c01,false,v_by_one", 448000))
    for key, label, pairs in cases:
        cfg = Configuration.parse(label)
        buf = _buf(g["pos0"])
        st = B.force_phase(buf, box, params, cfg, 8)
        assert st.pair_interactions == pairs
        assert (st.kernel_invocations, st.lane_slots, st.useful_interactions,
                st.pair_interactions) == tuple(g[f"stats0_{key}"])
        assert forces_close(buf.forces().cpu().numpy(), g[f"F0_{key}"])
    # host (numpy) buffers through the same entry point, as a reference caller would pass
    host = B.ParticleBuffer.from_positions(g["pos0"], device="cpu").numpy()

    class HostBuf:
        pass

    hb = HostBuf()
    for name, arr in host.items():
        setattr(hb, name, arr.copy())
    st = B.force_phase(hb, box, params, Configuration.parse(cases[0][1]), 8)
    assert st.pair_interactions == 250764
    f = np.stack([hb.force_x, hb.force_y, hb.force_z], axis=1)
    assert forces_close(f, g["F0_c08n3"])


def test_config1_ten_verlet_steps_track_reference():
    g = golden("config1.npz")
    box = _box(22.0, True)
    params = LJParams(cutoff=2.5, skin=0.0, dt=0.001)
    cfg = Configuration.parse("lc,lc_c08,true,one_by_v")
    buf = _buf(g["pos0"])
    v = torch.as_tensor(g["vel0"], device="cuda")
    buf.vel_x.copy_(v[:, 0]), buf.vel_y.copy_(v[:, 1]), buf.vel_z.copy_(v[:, 2])
    from paper_2512_03565_b200.integrator import velocity_verlet_step
    B.force_phase(buf, box, params, cfg, 8)
    pairs = []
    for _ in range(10):
        velocity_verlet_step(buf, params, "pre-force")
        pairs.append(B.force_phase(buf, box, params, cfg, 8).pair_interactions)
        velocity_verlet_step(buf, params, "post-force")
        B.apply_boundaries(buf, box)
    assert pairs == g["pairs_per_step"].tolist()
    pos = buf.positions().cpu().numpy()
    assert np.abs(pos - g["pos10"]).max() < 1e-12
    assert forces_close(buf.forces().cpu().numpy(), g["F10"], rtol=1e-10)


@pytest.mark.parametrize("periodic", [False, True])
def test_energy_virial_and_forces_vs_oracle_dense(rng, periodic):
    pos = jittered_lattice(rng, (12, 12, 12), 1.077, 0.1)
    span = 12 * 1.077
    params = LJParams(cutoff=2.5, skin=0.3)
    box = _box(span, periodic)
    lo, hi = np.zeros(3), np.full(3, span)
    of, ost = O.force_phase_lc(pos, lo, hi, [periodic] * 3, params, "lc_c18", True,
                               "two_by_half", 8)
    for label in ("lc,lc_c01,false,one_by_v", "lc,lc_c18,true,two_by_half",
                  "lc,lc_c08,false,half_by_two", "lc,lc_c08,true,v_by_one"):
        cfg = Configuration.parse(label)
        buf = _buf(pos)
        st = B.force_phase(buf, box, params, cfg, 8, energy=True)
        assert forces_close(buf.forces().cpu().numpy(), of), label
        assert abs(st.epot - ost.epot) <= 1e-12 * abs(ost.epot), label
        assert abs(st.virial - ost.virial) <= 1e-12 * abs(ost.virial), label
        if cfg.newton3:
            assert st.pair_interactions == ost.pair_interactions
    e, w = brute_energy_virial(pos, params, np.full(3, span) if periodic else None)
    assert abs(ost.epot - e) <= 1e-11 * abs(e)


def test_overlap_raises():
    pos = np.random.default_rng(3).uniform(0, 9, (20, 3))
    pos[7] = pos[3]
    for label in ("lc,lc_c08,true,one_by_v", "lc,lc_c01,false,two_by_half"):
        with pytest.raises(B.ParticleOverlapError):
            B.force_phase(_buf(pos), _box(9.0, False), LJParams(cutoff=2.2, skin=0.4),
                          Configuration.parse(label), 8)


def test_functor_matches_reference_fixtures():
    g = golden("functor.npz")
    params = LJParams(cutoff=2.5, skin=0.5)
    for k in range(int(g["count"])):
        ni, nj, same, n3, pi_, V = g[f"c{k}_meta"].tolist()
        bi = ParticleBuffer.from_positions(g[f"c{k}_pi"], ownership=g[f"c{k}_oi"], device="cuda")
        bj = bi if same else ParticleBuffer.from_positions(g[f"c{k}_pj"], ownership=g[f"c{k}_oj"],
                                                           device="cuda")
        st = B.compute_pair_vectorized(bi, bj, params, bool(n3), bool(same), PATTERNS[pi_], V)
        assert (st.kernel_invocations, st.lane_slots, st.useful_interactions,
                st.pair_interactions) == tuple(g[f"c{k}_stats"]), k
        assert forces_close(bi.forces().cpu().numpy(), g[f"c{k}_fi"]), k
        if not same:
            assert forces_close(bj.forces().cpu().numpy(), g[f"c{k}_fj"]), k


def test_functor_edge_cases():
    params = LJParams(cutoff=2.5, skin=0.5)
    # empty j buffer
    bi = ParticleBuffer.from_positions([[0.0, 0.0, 0.0]], device="cuda")
    bj = ParticleBuffer.from_positions(np.zeros((0, 3)), device="cuda")
    assert B.compute_pair_vectorized(bi, bj, params, False, False, PatternKind.ONE_BY_V, 8) \
        == B.KernelStats(1 * 0, 0, 0, 0)
    # two-body third law, bitwise antisymmetric
    b = ParticleBuffer.from_positions([[0.0, 0.0, 0.0], [1.1, 0.0, 0.0]], device="cuda")
    st = B.compute_pair_vectorized(b, b, params, True, True, PatternKind.TWO_BY_HALF, 8)
    f = b.forces().cpu().numpy()
    assert st.pair_interactions == 1 and f[0, 0] == -f[1, 0] != 0.0
    # exact cutoff distance contributes nothing
    b = ParticleBuffer.from_positions([[0.0, 0.0, 0.0], [2.5, 0.0, 0.0]], device="cuda")
    st = B.compute_pair_vectorized(b, b, params, True, True, PatternKind.ONE_BY_V, 8)
    assert st.pair_interactions == 0 and not b.forces().abs().sum().item()
    # same_buffer requires identity; invalid widths
    a = ParticleBuffer.from_positions([[0.0, 0.0, 0.0]], device="cuda")
    with pytest.raises(B.ConfigurationError):
        B.compute_pair_vectorized(a, a.copy(), params, False, True, PatternKind.ONE_BY_V, 8)
    for w in (2, 3, 6, 0):
        with pytest.raises(B.ConfigurationError):
            B.compute_pair_vectorized(a, a, params, False, True, PatternKind.ONE_BY_V, w)
    # scalar path: no blank lanes
    b = ParticleBuffer.from_positions(np.random.default_rng(1).uniform(0, 6, (40, 3)),
                                      device="cuda")
    st = B.compute_pair_scalar(b, b, params, True, True)
    assert st.lane_slots == st.useful_interactions == 40 * 39 // 2


def test_lc_random_medium_vs_oracle(rng):
    n = 20000
    span = (n / 0.5) ** (1 / 3)
    pos = jittered_lattice(rng, (28, 28, 28), span / 28, 0.3)[:n]
    params = LJParams(cutoff=2.5, skin=0.3)
    lo, hi = np.zeros(3), np.full(3, span)
    for trav, n3, pat in (("lc_c01", False, "one_by_v"), ("lc_c08", True, "half_by_two"),
                          ("lc_c18", True, "v_by_one")):
        of, ost = O.force_phase_lc(pos, lo, hi, [True] * 3, params, trav, n3, pat, 8)
        buf = _buf(pos)
        st = B.force_phase(buf, _box(span, True), params,
                           Configuration(ContainerKind.LINKED_CELLS, TraversalKind(trav), n3,
                                         PatternKind(pat)), 8)
        assert st == B.KernelStats(*ost.as_tuple())
        assert forces_close(buf.forces().cpu().numpy(), of)


@pytest.mark.parametrize("trav", ["lc_c08", "lc_c18"])
def test_colored_newton3_matches_full_shell_and_is_deterministic(rng, trav):
    pos = jittered_lattice(rng, (14, 14, 14), 1.08, 0.12)
    span = 14 * 1.08
    params = LJParams(cutoff=2.5, skin=0.0)
    box = _box(span, True)
    results = {}
    for mode in ("colored", "full_shell", "colored"):
        cont = B.LinkedCellsContainer(box, params)
        cont.n3_mode = mode
        buf = _buf(pos)
        cont.rebuild(buf)
        cont.refresh(buf)
        for pat in PATTERNS:
            st = cont.compute_forces(trav, True, pat, 8, energy=True)
            cont.collect_forces(buf)
            f = buf.forces().cpu().numpy()
            key = (mode, pat)
            if key in results:
                assert np.array_equal(results[key][0], f)        # bitwise deterministic
            results[key] = (f, st)
    for pat in PATTERNS:
        fc, sc = results[("colored", pat)]
        ff, sf = results[("full_shell", pat)]
        assert forces_close(fc, ff)
        assert sc == sf
        assert abs(sc.epot - sf.epot) <= 1e-12 * abs(sf.epot)


@pytest.mark.parametrize("tpi", [True, False])
def test_full_shell_dup_cells_energy_and_determinism(rng, tpi):
    """Full-shell kernels (warp per cell; V_BY_ONE also thread per particle)
    against the oracle with dup-weighted cells (images mid-step in owned
    cells), energy/virial, and run-to-run bitwise determinism."""
    n = 6000
    span = (n / 0.7) ** (1 / 3)
    pos = jittered_lattice(rng, (19, 19, 19), span / 19, 0.3)[:n]
    pos[:40] = np.mod(pos[:40] - 0.02 * span, span)      # a few near the faces
    pos[40:45, 0] = span + 1e-3                           # outside [lo, hi): dup anchors
    params = LJParams(cutoff=2.5, skin=0.0)
    lo, hi = np.zeros(3), np.full(3, span)
    for pat in PATTERNS:
        of, ost = O.force_phase_lc(pos, lo, hi, [True] * 3, params, "lc_c18", False, pat.value,
                                   8)
        prev = None
        for _ in range(2):
            cont = B.LinkedCellsContainer(_box(span, True), params)
            cont.thread_per_particle = tpi
            buf = _buf(pos)
            cont.rebuild(buf)
            cont.refresh(buf)
            st = cont.compute_forces("lc_c18", False, pat, 8, energy=True)
            cont.collect_forces(buf)
            f = buf.forces().cpu().numpy()
            assert st == B.KernelStats(*ost.as_tuple()), pat
            assert forces_close(f, of), pat
            assert abs(st.epot - ost.epot) <= 1e-12 * abs(ost.epot)
            assert abs(st.virial - ost.virial) <= 1e-12 * abs(ost.virial)
            if prev is not None:
                assert np.array_equal(prev, f)
            prev = f


def test_thread_per_particle_between_rebuilds_uses_rebuild_cells(rng):
    """With a skin, particles move between rebuilds while staying in their
    rebuild-time cells: the thread-per-particle kernel must sweep those cells
    (as the warp-per-cell kernel does), not cells recomputed from positions."""
    pos = jittered_lattice(rng, (16, 16, 16), 1.1, 0.2)
    span = 16 * 1.1
    params = LJParams(cutoff=2.5, skin=0.4)
    box = _box(span, True)
    moved = np.mod(pos + rng.uniform(-0.15, 0.15, pos.shape), span)
    res = {}
    for tpi in (True, False):
        cont = B.LinkedCellsContainer(box, params)
        cont.thread_per_particle = tpi
        buf = _buf(pos)
        cont.rebuild(buf)
        cont.refresh(buf)
        buf2 = _buf(moved)
        cont.refresh_positions(buf2)
        st = cont.compute_forces("lc_c01", False, PatternKind.V_BY_ONE, 8)
        cont.collect_forces(buf2)
        res[tpi] = (st.pair_interactions, buf2.forces().cpu().numpy())
    assert res[True][0] == res[False][0]
    assert forces_close(res[True][1], res[False][1])


def test_gpu_lane_stats_lc_and_vl(rng):
    """Physical lane use of the executing kernels: recomputed
    here from the cell tables / list layout independently."""
    pos = jittered_lattice(rng, (14, 14, 14), 1.05, 0.3)
    span = 14 * 1.05
    box = _box(span, True)
    cont = B.LinkedCellsContainer(box, LJParams(cutoff=2.5, skin=0.0))
    buf = _buf(pos)
    cont.rebuild(buf)
    cont.refresh(buf)
    # warp per cell: the reference's c01 formula at V = 32
    cont.thread_per_particle = False
    for pat in PATTERNS:
        steps, active = cont.gpu_lane_stats(pat)
        inv, slots, useful = cont._lc_stats(B.traversals.traversal_code(TraversalKind.LC_C01),
                                            False, pat, 32)
        assert (steps, active) == (slots, useful)
    # thread per particle: per warp of a consecutive particles and per
    # neighbour offset, ceil(n / b) for the largest neighbour cell n
    cont.thread_per_particle = True
    cells = cont._cell_of.cpu().numpy().astype(np.int64)
    count = cont._count.cpu().numpy().astype(np.int64)
    t0, t1 = int(cont.total_dims[0]), int(cont.total_dims[1])
    for pat in (PatternKind.V_BY_ONE, PatternKind.HALF_BY_TWO):   # the orders it serves
        a, b = pat.shape(32)
        steps, active = cont.gpu_lane_stats(pat)
        want = 0
        for w0 in range(0, len(cells), a):
            c = cells[w0:w0 + a]
            for d in range(27):
                off = (d // 9 - 1) + t0 * ((d // 3) % 3 - 1 + t1 * (d % 3 - 1))
                want += int((-(-count[c + off] // b)).max())
        assert steps == 32 * want and 0 < active <= steps
    # Verlet lists: tiles x kmax / B steps; active = list entries
    vl = B.VerletListContainer(box, LJParams(cutoff=2.5, skin=0.3))
    vl.rebuild(buf)
    vl.refresh(buf)
    for pat in PATTERNS:
        steps, active = vl.gpu_lane_stats(pat, False)
        inv, slots, useful = vl.vl_stats(False, pat, 32)
        a, b = pat.shape(32)
        if vl._vls_for(pat, False) is not None:
            # segmented lists (v_by_one): whole 8-step chunks per tile segment,
            # lanes dealt by length; every entry on a lane, padding bounded
            assert active == useful and steps % 256 == 0 and useful <= steps < 1.6 * useful
            continue
        cnt = vl._count(False, pat)[: vl.n_owned].cpu().numpy().astype(np.int64)
        pad = (-len(cnt)) % a
        m = np.concatenate([cnt, np.zeros(pad, np.int64)]).reshape(-1, a).max(axis=1)
        fills = -(-m // b)
        want = int((-(-fills // 4) * 4).sum())          # whole 4-step index chunks
        assert active == useful and steps == 32 * want and steps >= slots
