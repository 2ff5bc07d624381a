"""Host-side logic that needs no GPU: patterns, statistics formulas, the
configuration space and the tuner state machine (reference tests
test_kernels.py / test_tuning.py / test_acceptance.py criteria 3, 4, 6)."""

from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2512_03565_b200 import (PATTERN_ORDER, Configuration, ConfigurationError,
                                   ContainerKind, KernelStats, LaneOpsMetric, PatternKind,
                                   ReplayMetric, TraversalKind, Tuner, TuningPolicy,
                                   blanks_expected, enumerate_search_space, lj_pair_force,
                                   needs_rebuild, reduce_samples, select_optimum)
from paper_2512_03565_b200.tuning import Evidence
from conftest import P

REF_CONTAINERS = [ContainerKind.LINKED_CELLS, ContainerKind.VERLET_CLUSTER_LISTS]
REF_TRAVERSALS = [TraversalKind.LC_C01, TraversalKind.LC_C08, TraversalKind.LC_C18,
                  TraversalKind.VCL]


def test_reference_search_space_has_28_configs():
    space = enumerate_search_space(REF_CONTAINERS, REF_TRAVERSALS, [False, True],
                                   list(PATTERN_ORDER))
    assert len(space) == 28
    assert space[0].label == "lc,lc_c01,false,one_by_v"
    assert all(c.is_valid() for c in space)


def test_extended_search_space_adds_verlet_lists():
    space = enumerate_search_space(list(ContainerKind), list(TraversalKind), [False, True],
                                   list(PATTERN_ORDER))
    assert len(space) == 36
    vl = [c for c in space if c.container is ContainerKind.VERLET_LISTS]
    assert len(vl) == 8 and all(c.traversal is TraversalKind.VL for c in vl)


def test_configuration_parse_and_validity():
    c = Configuration.parse("lc,lc_c08,on,two_by_half")
    assert c.newton3 and c.pattern is PatternKind.TWO_BY_HALF
    assert c.label == "lc,lc_c08,true,two_by_half"
    for bad in ("lc,lc_c01,true,one_by_v", "vcl,lc_c08,false,one_by_v", "lc,vl,false,one_by_v",
                "lc,lc_c08,maybe,one_by_v", "lc,lc_c08"):
        with pytest.raises(ConfigurationError):
            Configuration.parse(bad)


@pytest.mark.parametrize("width", [4, 8, 16, 32])
def test_pattern_shapes(width):
    for p in PATTERN_ORDER:
        a, b = p.shape(width)
        assert a * b == width


def test_blanks_expected_values():
    assert blanks_expected(PatternKind.ONE_BY_V, 5, 8, 8) == 0
    assert blanks_expected(PatternKind.ONE_BY_V, 5, 5, 8) == 15
    assert blanks_expected(PatternKind.HALF_BY_TWO, 4, 6, 8) == 0
    for width in (4, 8, 16):
        half = width // 2
        for nb in range(1, 7):
            assert blanks_expected(PatternKind.HALF_BY_TWO, half, nb * half, width) == 0
            for p in (PatternKind.V_BY_ONE, PatternKind.ONE_BY_V):
                assert blanks_expected(p, width, nb * width, width) == 0
        assert blanks_expected(PatternKind.V_BY_ONE, half, half, width) > 0
    with pytest.raises(ConfigurationError):
        blanks_expected(PatternKind.ONE_BY_V, -1, 2, 8)
    with pytest.raises(ConfigurationError):
        blanks_expected(PatternKind.ONE_BY_V, 1, 2, 6)


def test_lj_pair_force_known_answers():
    p = P(cutoff=2.5)
    assert np.abs(lj_pair_force(np.array([2.0 ** (1 / 6), 0, 0]), p)).max() < 1e-12
    assert np.allclose(lj_pair_force(np.array([1.0, 0, 0]), p), [24.0, 0, 0])
    assert np.array_equal(lj_pair_force(np.array([2.5, 0, 0]), p), np.zeros(3))


def test_needs_rebuild_thresholds():
    ref = np.zeros((3, 3))
    assert not needs_rebuild(ref.copy(), ref, skin=1.0, steps_since_rebuild=5)
    assert needs_rebuild(ref.copy(), ref, skin=1.0, steps_since_rebuild=20)
    moved = ref.copy()
    moved[1, 0] = 0.5
    assert needs_rebuild(moved, ref, skin=1.0, steps_since_rebuild=0)
    nearly = ref.copy()
    nearly[1, 0] = 0.5 - 1e-9
    assert not needs_rebuild(nearly, ref, skin=1.0, steps_since_rebuild=0)
    assert needs_rebuild(ref, None, skin=1.0, steps_since_rebuild=0)
    import torch
    t = torch.as_tensor(moved)
    assert needs_rebuild(t, torch.as_tensor(ref), skin=1.0, steps_since_rebuild=0)
    assert not needs_rebuild(torch.as_tensor(nearly), torch.as_tensor(ref), 1.0, 0)


def test_kernel_stats_equality_ignores_energy():
    a = KernelStats(1, 8, 5, 2, epot=-3.0)
    b = KernelStats(1, 8, 5, 2, epot=0.0)
    assert a == b and a.blank_lanes == 3


def test_reduce_and_select():
    assert reduce_samples([1.0, 3.0], "mean") == 2.0
    assert reduce_samples([1.0, 3.0, 2.0], "median") == 2.0
    assert reduce_samples([4.0, 3.0], "min") == 3.0
    with pytest.raises(ConfigurationError):
        reduce_samples([], "mean")
    space = enumerate_search_space(REF_CONTAINERS, REF_TRAVERSALS, [False], [PatternKind.ONE_BY_V])
    ev = [Evidence(space[0], [2.0], 2.0), Evidence(space[1], [math.inf], math.inf),
          Evidence(space[2], [1.0], 1.0), Evidence(space[3], [1.0], 1.0)]
    assert select_optimum(ev) == space[2]


def test_tuner_full_search_and_selection():
    space = enumerate_search_space([ContainerKind.LINKED_CELLS],
                                   [TraversalKind.LC_C01, TraversalKind.LC_C08], [False, True],
                                   list(PATTERN_ORDER))
    assert len(space) == 12
    tuner = Tuner(space, TuningPolicy(samples_per_config=2, tuning_interval=30))
    target = space[7]
    seen = {}
    selections = []
    for it in range(90):
        cfg, phase = tuner.next_configuration(it)
        if phase == "tuning":
            seen[cfg.label] = seen.get(cfg.label, 0) + 1
        tuner.record_sample(1.0 if cfg == target else 10.0 + space.index(cfg))
    assert set(seen.values()) == {6}
    assert [c.label for c in tuner.phase_selection] == [target.label] * 3
    with pytest.raises(ConfigurationError):
        Tuner(space, TuningPolicy(samples_per_config=3, tuning_interval=10))


def test_tuner_displaced_samples_are_retaken_and_retune():
    space = enumerate_search_space([ContainerKind.LINKED_CELLS], [TraversalKind.LC_C08],
                                   [False, True], [PatternKind.ONE_BY_V])
    tuner = Tuner(space, TuningPolicy(samples_per_config=1, tuning_interval=100))
    cfg, phase = tuner.next_configuration(0)
    tuner.record_sample(5.0, displaced=True)
    cfg2, _ = tuner.next_configuration(1)
    assert cfg2 == cfg
    tuner.record_sample(5.0)
    tuner.next_configuration(2)
    tuner.record_sample(1.0)
    assert tuner.selected == space[1]
    tuner.request_retune()
    _, phase = tuner.next_configuration(3)
    assert phase == "tuning"


def test_lane_ops_and_replay_metrics(tmp_path):
    counter = [0]
    m = LaneOpsMetric(lambda: counter[0])
    m.begin_region()
    counter[0] += 48
    assert m.end_region() == 48.0
    path = tmp_path / "r.txt"
    path.write_text("1.5\n\n2\n")
    r = ReplayMetric(str(path))
    assert r.end_region() == 1.5 and r.end_region() == 2.0


def test_cluster_size_is_a_tuning_dimension():
    space = enumerate_search_space([ContainerKind.LINKED_CELLS, ContainerKind.VERLET_CLUSTER_LISTS],
                                   [TraversalKind.LC_C08, TraversalKind.VCL], [False],
                                   [PatternKind.ONE_BY_V], cluster_sizes=[4, 8, 32])
    assert [c.label for c in space] == ["lc,lc_c08,false,one_by_v",
                                        "vcl,vcl,false,one_by_v,m4", "vcl,vcl,false,one_by_v,m8",
                                        "vcl,vcl,false,one_by_v,m32"]
    assert Configuration.parse("vcl,vcl,true,half_by_two,m8").cluster_size == 8
    with pytest.raises(ConfigurationError):
        Configuration.parse("lc,lc_c08,true,half_by_two,m8")


def test_energy_metric_needs_a_device():
    """The NVML energy metric (the paper's PMT analogue) refuses to run
    without a CUDA device instead of falling back to a host clock."""
    import torch

    import paper_2512_03565_b200 as B
    if torch.cuda.is_available():
        pytest.skip("host-only check")
    with pytest.raises(B.ConfigurationError):
        B.make_metric_provider("energy", lambda: 0)
