"""Known-answer tests on every GPU force kernel (the reference's
KATs, tests/test_kernels.py:24-42 and the exact-cutoff exclusion of
tests/test_kernels.py:226-238), through the containers:

* a pair at exactly r = rc contributes no pair and no force, directly and
  across the periodic boundary;
* a pair one ulp inside rc is a pair;
* F(2^(1/6) sigma) ~ 0 and F(d = (1, 0, 0)) = (24, 0, 0).

Every container / kernel variant (LC warp per cell, LC thread per particle,
colored Newton3, VL, VCL with M = 4 and 8), every interaction order and
Newton3 on/off, against the oracle's exact statistics.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import forces_close
from oracle import oracle as O

import paper_2512_03565_b200 as B
from paper_2512_03565_b200 import (Configuration, ContainerKind, LJParams, ParticleBuffer,
                                   PatternKind, SimulationBox, TraversalKind)

pytestmark = pytest.mark.gpu

L = 30.0
RC = 2.5


def _pairs():
    """Isolated pairs (> rc + skin apart from everything else) in a periodic box."""
    inside = np.nextafter(RC, 0.0)
    p = [
        (5.0, 5.0, 5.0), (5.0 + RC, 5.0, 5.0),                 # exactly rc: excluded
        (1.0, 15.0, 5.0), (1.0 + inside, 15.0, 5.0),           # one ulp inside: a pair
        (15.0, 5.0, 15.0), (15.0 + 2.0 ** (1 / 6), 5.0, 15.0),  # force minimum: F ~ 0
        (15.0, 15.0, 15.0), (16.0, 15.0, 15.0),                # d = 1: F = 24
        (0.5, 25.0, 25.0), (L - 2.0, 25.0, 25.0),              # exactly rc across x = L
        (25.0, 0.25, 10.0), (25.0, L - 2.0, 10.0),             # 2.25 across y = L: a pair
    ]
    p = np.array(p, dtype=np.float64)
    assert p[3, 0] - p[2, 0] == inside and p[1, 0] - p[0, 0] == RC
    return p


def _check_kats(f, st, n3):
    # pairs: one-ulp, minimum, unit distance, across-boundary 2.25 -> 4
    # (unordered); owned-image pairs count once per owned side even under N3
    assert np.all(f[0:2] == 0.0), "exact-cutoff pair must contribute nothing"
    assert np.all(f[8:10] == 0.0), "exact-cutoff image pair must contribute nothing"
    assert np.all(np.abs(f[4:6]) < 1e-12)
    assert f[6][0] == pytest.approx(-24.0, rel=1e-12) and f[7][0] == pytest.approx(24.0, rel=1e-12)
    assert f[3][0] < 0 < f[2][0]                     # attractive near rc
    assert st.pair_interactions == (5 if n3 else 8)


CASES = []
for pat in PatternKind:
    for trav, n3 in (("lc_c01", False), ("lc_c08", True), ("lc_c18", False), ("lc_c18", True)):
        CASES.append(("lc", trav, n3, pat, None))
    for n3 in (False, True):
        CASES.append(("vl", "vl", n3, pat, None))
        for m in (4, 8):
            CASES.append(("vcl", "vcl", n3, pat, m))


@pytest.mark.parametrize("cont,trav,n3,pat,m", CASES,
                         ids=[f"{c[0]}-{c[1]}-{int(c[2])}-{c[3].value}-{c[4]}" for c in CASES])
def test_known_answers(cont, trav, n3, pat, m):
    pos = _pairs()
    params = LJParams(cutoff=RC, skin=0.3 if cont != "lc" else 0.0)
    box = SimulationBox.cube(L, periodic=True)
    lo, hi = np.zeros(3), np.full(3, L)
    if cont == "lc":
        of, ost = O.force_phase_lc(pos, lo, hi, [True] * 3, params, trav, n3, pat.value, 8)
    elif cont == "vl":
        of, ost = O.force_phase_vl(pos, lo, hi, [True] * 3, params, n3, pat.value, 8)
    else:
        of, ost = O.force_phase_vcl(pos, lo, hi, [True] * 3, params, m, n3, pat.value, 8)
    cfg = Configuration(ContainerKind(cont), TraversalKind(trav), n3, pat,
                        cluster_size=m)
    variants = [{}]
    if cont == "lc":
        variants = [{"thread_per_particle": False}, {"thread_per_particle": True}]
        if n3 and trav != "lc_c01":
            variants.append({"n3_mode": "colored"})
    for knobs in variants:
        buf = ParticleBuffer.from_positions(pos, device="cuda")
        c = B.make_container(cfg.container, box, params, cluster_size=m)
        for k, v in knobs.items():
            setattr(c, k, v)
        c.rebuild(buf)
        c.refresh(buf)
        st = c.compute_forces(cfg.traversal, n3, pat, 8)
        c.collect_forces(buf)
        f = buf.forces().cpu().numpy()
        assert st == B.KernelStats(*ost.as_tuple()), knobs
        assert forces_close(f, of), knobs
        _check_kats(f, st, n3)
