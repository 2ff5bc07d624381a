"""GPU Verlet cluster lists against the reference fixtures (bit-exact
cluster structure and pair lists; forces within forces_close; exact stats)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import forces_close, golden
from oracle import oracle as O

import paper_2512_03565_b200 as B
from paper_2512_03565_b200 import Configuration, LJParams, ParticleBuffer, SimulationBox

pytestmark = pytest.mark.gpu


def test_cluster_structure_and_lists_match_reference():
    g = golden("clusters.npz")
    pos = g["pos"]
    box = SimulationBox.cube(9.0, periodic=True)
    params = LJParams(cutoff=2.2, skin=0.4)
    for M in (4, 8):
        from paper_2512_03565_b200.clusters import VerletClusterContainer
        cont = VerletClusterContainer(box, params, M)
        buf = ParticleBuffer.from_positions(pos, device="cuda")
        cont.rebuild(buf)
        cont.refresh(buf)
        s = cont.structure()
        assert np.array_equal(s["perm"], g[f"M{M}_perm"])
        assert np.array_equal(s["slots"], g[f"M{M}_slots"])
        assert np.array_equal(s["counts"], g[f"M{M}_counts"])
        assert np.array_equal(s["aabb_min"], g[f"M{M}_amin"])
        assert np.array_equal(s["aabb_max"], g[f"M{M}_amax"])
        assert np.array_equal(s["padded"], g[f"M{M}_padded"])
        for n3 in (False, True):
            lists = cont.neighbor_lists[n3]
            flat = [(k, z) for k, zs in enumerate(lists) for z in zs]
            want = [tuple(r) for r in g[f"M{M}_pairs_n3{int(n3)}"].tolist()]
            assert flat == want, (M, n3)
        # images are emitted in (owner, shift) order on the device; the (col, z)
        # sort makes the halo clusters independent of that order (no z ties)
        links = [(k, h) for k, hs in enumerate(cont.halo_links) for h in hs]
        assert links == [tuple(r) for r in g[f"M{M}_halo_links"].tolist()]


def test_vcl_force_phase_matches_reference_instances():
    g = golden("instances.npz")
    labels = [str(x) for x in g["labels"]]
    for k in range(8):
        pos = g[f"i{k}_pos"]
        span, periodic, cutoff, skin = g[f"i{k}_box"]
        box = SimulationBox.cube(float(span), periodic=bool(periodic))
        params = LJParams(cutoff=float(cutoff), skin=float(skin))
        stats = g[f"i{k}_stats"]
        for ci, label in enumerate(labels):
            if not label.startswith("vcl,"):
                continue
            cfg = Configuration.parse(label)
            for vi, V in enumerate((4, 8, 16)):
                buf = ParticleBuffer.from_positions(pos, device="cuda")
                st = B.force_phase(buf, box, params, cfg, V)
                got = (st.kernel_invocations, st.lane_slots, st.useful_interactions,
                       st.pair_interactions)
                assert got == tuple(stats[ci, vi]), (k, label, V)
                ref = g[f"i{k}_F_{label.rsplit(',', 1)[0]},M{V}"]
                assert forces_close(buf.forces().cpu().numpy(), ref), (k, label, V)


@pytest.mark.parametrize("M", [4, 8, 32])
def test_vcl_medium_vs_oracle_lc(rng, M):
    n = 6000
    span = (n / 0.7) ** (1 / 3)
    k = int(np.ceil(n ** (1 / 3)))
    grid = np.stack(np.meshgrid(*[np.arange(k)] * 3, indexing="ij"), -1).reshape(-1, 3)[:n]
    pos = (grid + 0.5) * (span / k) + rng.uniform(-0.2, 0.2, (n, 3))
    params = LJParams(cutoff=2.5, skin=0.3)
    of, ost = O.force_phase_lc(pos, np.zeros(3), np.full(3, span), [True] * 3,
                               LJParams(cutoff=2.5, skin=0.3), "lc_c01", False, "one_by_v", 8)
    buf = ParticleBuffer.from_positions(pos, device="cuda")
    st = B.force_phase(buf, SimulationBox.cube(span, periodic=True), params,
                       Configuration.parse("vcl,vcl,false,half_by_two"), 8, cluster_size=M,
                       energy=True)
    assert st.pair_interactions == ost.pair_interactions
    assert forces_close(buf.forces().cpu().numpy(), of)
    assert abs(st.epot - ost.epot) <= 1e-12 * abs(ost.epot)
