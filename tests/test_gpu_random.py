"""Randomised parity (hypothesis): every container / order / Newton3 against
the oracle on small seeded systems with the edge cases the reference's tests
exercise -- mixed per-axis periodicity, grids only 1-3 cells wide, particles
exactly on the lower box faces, dense and dilute fills, several cutoff /
skin combinations.  Exact statistics, forces within forces_close."""

from __future__ import annotations

import os

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from conftest import forces_close
from oracle import oracle as O

import paper_2512_03565_b200 as B
from paper_2512_03565_b200 import (Configuration, ContainerKind, LJParams, ParticleBuffer,
                                   PatternKind, SimulationBox, TraversalKind)

pytestmark = pytest.mark.gpu

CONFIGS = [("lc", "lc_c01", False), ("lc", "lc_c08", True), ("lc", "lc_c18", False),
           ("lc", "lc_c18", True), ("vl", "vl", False), ("vl", "vl", True),
           ("vcl", "vcl", False), ("vcl", "vcl", True)]


def _system(seed, n, extent, min_d):
    """n particles in [0, extent) with pairwise distance >= min_d (greedy
    rejection), a few of them on the lower faces."""
    rng = np.random.default_rng(seed)
    pts = []
    tries = 0
    while len(pts) < n and tries < 50 * n:
        tries += 1
        p = rng.uniform(0.0, extent)
        if len(pts) < 3:
            p[len(pts)] = 0.0                 # exactly on a lower face
        if pts and np.min(np.linalg.norm(np.array(pts) - p, axis=1)) < min_d:
            continue
        pts.append(p)
    return np.array(pts)


@settings(max_examples=int(os.environ.get("LMD_RANDOM_EXAMPLES", "30")), deadline=None,
          suppress_health_check=list(HealthCheck))
@given(seed=st.integers(0, 10_000), n=st.integers(20, 400),
       extent=st.tuples(*[st.floats(5.2, 14.0)] * 3),
       periodic=st.tuples(*[st.booleans()] * 3),
       cutoff=st.sampled_from([1.8, 2.5]), skin=st.sampled_from([0.0, 0.2, 0.4]),
       cfg=st.sampled_from(CONFIGS), pattern=st.sampled_from(list(PatternKind)),
       m=st.sampled_from([4, 8]))
def test_random_systems_match_oracle(seed, n, extent, periodic, cutoff, skin, cfg, pattern, m):
    extent = np.array(extent)
    if np.any(extent < 2 * (cutoff + skin)):
        return                                 # images need a box >= 2 (rc + skin)
    pos = _system(seed, n, extent, 0.8)
    params = LJParams(cutoff=cutoff, skin=skin if cfg[0] != "lc" else 0.0)
    kinds = tuple("periodic" if p else "reflective" for p in periodic)
    box = SimulationBox(np.zeros(3), extent, kinds)
    lo, hi = np.zeros(3), extent
    cont, trav, n3 = cfg
    if cont == "lc":
        of, ost = O.force_phase_lc(pos, lo, hi, list(periodic), params, trav, n3, pattern.value, 8)
    elif cont == "vl":
        of, ost = O.force_phase_vl(pos, lo, hi, list(periodic), params, n3, pattern.value, 8)
    else:
        of, ost = O.force_phase_vcl(pos, lo, hi, list(periodic), params, m, n3, pattern.value, 8)
    buf = ParticleBuffer.from_positions(pos, device="cuda")
    config = Configuration(ContainerKind(cont), TraversalKind(trav), n3, pattern,
                           cluster_size=m if cont == "vcl" else None)
    stt = B.force_phase(buf, box, params, config, 8, energy=True)
    assert stt == B.KernelStats(*ost.as_tuple())
    assert forces_close(buf.forces().cpu().numpy(), of)
    if ost.epot != 0.0:
        assert abs(stt.epot - ost.epot) <= 1e-12 * abs(ost.epot) + 1e-300
