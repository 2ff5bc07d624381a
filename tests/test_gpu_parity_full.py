"""Parity at BASELINE.json's full sizes, through the exact path bench.py times.

The persistent containers are built as bench.py builds them (default knobs:
staged groups, bank-ordered 16-bit lists for Verlet lists), refreshed, run
through ``compute_forces`` and collected; the results are compared with the
oracle's bitwise restatement of the reference force phase (LC c01, energy and
virial on) on the same seeded state:

* pair counts exactly equal (N3 off: the oracle's LC c01 count; N3 on: the
  oracle's Verlet-list Newton3 count -- owned pairs once, image pairs once
  per owned side, the reference's convention, executor.py:104-111);
* forces within the reference's ``forces_close`` (1e-12 relative to each
  particle's own force scale, reference tests/conftest.py:73-79);
* potential energy and virial within 1e-12 relative.

Workloads: C2 (1,000,000 particles, RSA, rho 0.2 / 0.5 / 0.8), C4
(16,777,216-particle perturbed lattice; the bench's headline workload, also
through the both-segment launch and the one-shot force_phase path), C5
(8,388,608-particle gas at rho 0.3, the weak-scaling brick), C3
(2,000,000-particle droplet, rc 3.0) for the cluster lists at M = 4 / 8 / 32.
The oracle costs ~1.5 s per 1M particles and ~25 s at 16.8M (1 core)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import forces_close
from oracle import oracle as O

pytestmark = pytest.mark.gpu

ORDERS = ("v_by_one", "one_by_v", "two_by_half", "half_by_two")
RTOL = 1e-12


class Case:
    def __init__(self, w, skin=0.3):
        import paper_2512_03565_b200 as B
        self.w = w
        self.pos = w.positions.cpu().numpy() if hasattr(w.positions, "cpu") \
            else np.asarray(w.positions)
        self.L = w.box_length
        self.box = B.SimulationBox.cube(self.L, periodic=True)
        lo, hi = np.zeros(3), np.full(3, self.L)
        self.f, self.st = O.force_phase_lc(self.pos, lo, hi, [True] * 3,
                                           B.LJParams(cutoff=w.cutoff, skin=0.0), "lc_c01",
                                           False, "one_by_v", 8, omp=True)
        self.skin = skin
        self._n3_pairs = None

    def n3_pairs(self):
        """The oracle's Newton3 pair count on Verlet lists (same pairs as LC)."""
        if self._n3_pairs is None:
            import paper_2512_03565_b200 as B
            _, st = O.force_phase_vl(self.pos, np.zeros(3), np.full(3, self.L), [True] * 3,
                                     B.LJParams(cutoff=self.w.cutoff, skin=self.skin), True,
                                     "v_by_one", 8)
            self._n3_pairs = st.pair_interactions
        return self._n3_pairs


def _bench_container(case, kind, cluster_size=8):
    """The container exactly as bench.build_phase makes it."""
    import paper_2512_03565_b200 as B
    params = B.LJParams(cutoff=case.w.cutoff, skin=0.0 if kind == "lc" else case.skin)
    buf = B.ParticleBuffer.from_positions(case.pos, device="cuda")
    cont = B.make_container(kind, case.box, params, cluster_size=cluster_size)
    cont.rebuild(buf)
    cont.refresh(buf)
    return cont, buf


def _check(case, cont, buf, label, newton3, pattern, expect_pairs):
    st = cont.compute_forces(label, newton3, pattern, 8, energy=True)
    cont.collect_forces(buf)
    f = buf.forces().cpu().numpy()
    assert st.pair_interactions == expect_pairs, (label, pattern, newton3)
    assert forces_close(f, case.f, RTOL), (label, pattern, newton3)
    assert abs(st.epot - case.st.epot) <= RTOL * abs(case.st.epot)
    assert abs(st.virial - case.st.virial) <= RTOL * abs(case.st.virial)
    # Newton's third law over the whole periodic system
    assert np.abs(f.sum(axis=0)).max() <= 1e-10 * np.abs(f).sum()


def _vl_all(case):
    cont, buf = _bench_container(case, "vl")
    for pattern in ORDERS:
        _check(case, cont, buf, "vl", False, pattern, case.st.pair_interactions)
    for pattern in ("v_by_one", "half_by_two"):
        _check(case, cont, buf, "vl", True, pattern, case.n3_pairs())
    del cont, buf
    torch.cuda.empty_cache()


@pytest.fixture(scope="module", params=[0.2, 0.5, 0.8], ids=lambda r: f"rho{r}")
def c2(request):
    from paper_2512_03565_b200 import workloads
    torch.cuda.set_device(0)
    return Case(workloads.config2(request.param, n=1_000_000, device="cuda"))


def test_c2_verlet_lists_every_order_and_newton3(c2):
    _vl_all(c2)


def test_c2_linked_cells(c2):
    cont, buf = _bench_container(c2, "lc")
    for trav, pattern in (("lc_c01", "v_by_one"), ("lc_c01", "one_by_v"),
                          ("lc_c08", "half_by_two")):
        st = cont.compute_forces(trav, False, pattern, 8, energy=True)
        cont.collect_forces(buf)
        assert st.pair_interactions == c2.st.pair_interactions
        assert forces_close(buf.forces().cpu().numpy(), c2.f, RTOL), (trav, pattern)
        assert abs(st.epot - c2.st.epot) <= RTOL * abs(c2.st.epot)


def test_c4_headline_workload():
    """BASELINE config 4 at full size (16,777,216 particles)."""
    from paper_2512_03565_b200 import workloads
    torch.cuda.set_device(0)
    case = Case(workloads.config4(256, device="cpu"))
    assert case.st.pair_interactions == 907_284_108   # profiles/r01_parity_full.jsonl
    _vl_all(case)


def _one_shot_and_both_segments(case):
    """The same state through (i) the launch that runs both list segments
    (no displacement record: what a launch does once a particle has moved
    inner_skin / 2) and (ii) the public one-shot force_phase (the list-free
    path, lmd_vls_direct), which bench.py's e2e times."""
    import paper_2512_03565_b200 as B
    cont, buf = _bench_container(case, "vl")
    cont.ensure_lists(B.PatternKind.V_BY_ONE, False)
    cont._disp_slot = -1
    _check(case, cont, buf, "vl", False, "v_by_one", case.st.pair_interactions)
    del cont, buf
    torch.cuda.empty_cache()
    params = B.LJParams(cutoff=case.w.cutoff, skin=case.skin)
    buf = B.ParticleBuffer.from_positions(case.pos, device="cuda")
    st = B.force_phase(buf, case.box, params, B.Configuration.parse("vl,vl,false,v_by_one"), 8,
                       energy=True)
    f = buf.forces().cpu().numpy()
    assert st.pair_interactions == case.st.pair_interactions
    assert forces_close(f, case.f, RTOL)
    assert abs(st.epot - case.st.epot) <= RTOL * abs(case.st.epot)
    assert abs(st.virial - case.st.virial) <= RTOL * abs(case.st.virial)
    del buf
    torch.cuda.empty_cache()


def test_c4_one_shot_path_and_both_segments():
    from paper_2512_03565_b200 import workloads
    torch.cuda.set_device(0)
    _one_shot_and_both_segments(Case(workloads.config4(256, device="cpu")))


def test_c5_weak_scaling_brick():
    """BASELINE config 5's per-GPU system (8,388,608 particles, rho 0.3)."""
    from paper_2512_03565_b200 import workloads
    torch.cuda.set_device(0)
    case = Case(workloads.config5(device="cuda"))
    cont, buf = _bench_container(case, "vl")
    _check(case, cont, buf, "vl", False, "v_by_one", case.st.pair_interactions)
    _check(case, cont, buf, "vl", True, "v_by_one", case.n3_pairs())
    del cont, buf
    torch.cuda.empty_cache()
    _one_shot_and_both_segments(case)


@pytest.mark.parametrize("m", [4, 8, 32])
def test_c3_cluster_lists(m, c3):
    cont, buf = _bench_container(c3, "vcl", cluster_size=m)
    for pattern in ("v_by_one", "one_by_v"):
        _check(c3, cont, buf, "vcl", False, pattern, c3.st.pair_interactions)


@pytest.fixture(scope="module")
def c3():
    from paper_2512_03565_b200 import workloads
    torch.cuda.set_device(0)
    return Case(workloads.config3(device="cuda"))
