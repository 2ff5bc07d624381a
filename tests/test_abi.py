"""The C-ABI library loads on a CPU-only host and exports every symbol the
public header declares; host-side geometry entry points agree with the
reference arithmetic (no GPU needed)."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_2512_03565_b200 import _native as N
from paper_2512_03565_b200 import LJParams, SimulationBox
from paper_2512_03565_b200.errors import DegenerateDomainError


def test_library_exports_every_declared_symbol():
    lib = N.load()
    names = N.declared_symbols()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert missing == []
    # every declared function has a ctypes signature in the binding
    assert set(names) <= set(N._SIGNATURES)


def test_binding_arity_matches_header():
    arity = N.declared_arity()
    assert set(arity) == set(N.declared_symbols())
    bad = {name: (arity[name], len(N._SIGNATURES[name][1])) for name in arity
           if arity[name] != len(N._SIGNATURES[name][1])}
    assert bad == {}


def test_version_and_status_strings():
    lib = N.load()
    assert lib.lmd_version() >= 1
    for code in range(5):
        assert lib.lmd_status_string(code)


def test_struct_sizes_match_header():
    assert C.sizeof(N.Stats) == 8 * 4 + 8 * 2 + 8 + 4 + 4
    assert C.sizeof(N.Box) == 8 * 6 + 4 * 4
    assert C.sizeof(N.Grid) == 8 * 13


@pytest.mark.parametrize("L,length,dims", [(22.0, 2.5, 8), (10.0, 5.0, 2), (200.0, 5.0, 40),
                                           (6.0, 5.0, 1), (107.72, 2.8, 38)])
def test_grid_init_matches_reference_rule(L, length, dims):
    box = N.make_box(SimulationBox.cube(L))
    g = N.Grid()
    assert N.load().lmd_grid_init(C.byref(box), length, C.byref(g)) == 0
    assert list(g.dims) == [dims] * 3
    assert list(g.tdims) == [dims + 2] * 3
    assert g.cell_len[0] == L / dims
    assert g.ncell == (dims + 2) ** 3


def test_grid_init_degenerate():
    from paper_2512_03565_b200 import LinkedCellsContainer
    with pytest.raises(DegenerateDomainError):
        LinkedCellsContainer(SimulationBox(np.zeros(3), np.array([4.0, 10, 10]),
                                           ("reflective",) * 3), LJParams(cutoff=4.0, skin=1.0))


def test_container_geometry_on_cpu():
    from paper_2512_03565_b200 import LinkedCellsContainer
    c = LinkedCellsContainer(SimulationBox.cube(22.0), LJParams(cutoff=2.5, skin=0.0))
    assert c.dims.tolist() == [8, 8, 8]
    assert c.total_dims.tolist() == [10, 10, 10]
    assert c.linear_index(np.array([1, 2, 3])) == 1 + 10 * (2 + 10 * 3)


def test_no_cpu_fallback_for_device_entry_points():
    import torch
    from paper_2512_03565_b200.errors import NativeLibraryError
    with pytest.raises(NativeLibraryError):
        N.ptr(torch.zeros(3))


def test_force_phase_refuses_to_run_without_a_device():
    """The public entry point has no CPU fallback: without a CUDA device it
    raises instead of computing anything on the host."""
    import torch

    import paper_2512_03565_b200 as B
    from paper_2512_03565_b200.errors import NativeLibraryError
    if torch.cuda.is_available():
        pytest.skip("host-only check")

    class Host:
        pass

    h = Host()
    pos = np.random.default_rng(0).uniform(0, 10, (50, 3))
    for k, v in zip(("pos_x", "pos_y", "pos_z"), pos.T):
        setattr(h, k, np.ascontiguousarray(v))
    for k in ("force_x", "force_y", "force_z"):
        setattr(h, k, np.zeros(50))
    h.ownership = np.zeros(50, dtype=np.int8)
    with pytest.raises(NativeLibraryError):
        B.force_phase(h, B.SimulationBox.cube(10.0), B.LJParams(cutoff=2.5, skin=0.3),
                      B.Configuration.parse("vl,vl,false,v_by_one"), 8)


def test_missing_library_is_an_error(monkeypatch, tmp_path):
    """A missing libb200md.so raises NativeLibraryError (no silent fallback)."""
    from paper_2512_03565_b200.errors import NativeLibraryError
    monkeypatch.setattr(N, "_lib", None)
    monkeypatch.setattr(N, "lib_path", lambda: str(tmp_path / "absent.so"))
    with pytest.raises(NativeLibraryError):
        N.load()


def test_staged_list_host_entry_points():
    """Host-side sizing entry points of the staged Verlet lists (no GPU):
    the staged-row capacity per group size (the dummy row and a 16-row
    margin below the shared-memory rows), invalid sizes rejected, and the
    bank-order workspace per warp."""
    lib = N.load()
    assert lib.lmd_vl_staged_capacity(128) == 2304 - 16
    assert lib.lmd_vl_staged_capacity(256) == 4096 - 16
    assert lib.lmd_vl_staged_capacity(512) == 7168 - 16
    for bad in (0, 64, 100, 1024):
        assert lib.lmd_vl_staged_capacity(bad) == 0
    assert lib.lmd_vl_bank_smem_per_warp(100) == (64 * 16 + 100 * 32) * 4
