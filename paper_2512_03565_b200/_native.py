"""ctypes binding of libb200md.so -- the C ABI declared in include/b200md.h.

Loading fails loudly: there is no CPU fallback for any entry point.  Every
pointer handed to the library is a CUDA tensor's ``data_ptr()`` and every
call is issued on the current torch stream.
"""

from __future__ import annotations

import ctypes as C
import os
import re

import torch

from . import _build
from .errors import (ConfigurationError, DegenerateDomainError, NativeLibraryError,
                     ParticleOverlapError)

OK, ERR_CONFIG, ERR_DEGENERATE, ERR_CUDA, ERR_OVERLAP = 0, 1, 2, 3, 4

OWNED, HALO, DUMMY = 0, 1, 2

ONE_BY_V, V_BY_ONE, TWO_BY_HALF, HALF_BY_TWO = 0, 1, 2, 3
LC_C01, LC_C08, LC_C18, VCL, VL = 0, 1, 2, 3, 4
FLAG_ENERGY = 1
FLAG_DEFER_EV = 2


class Stats(C.Structure):
    _fields_ = [("kernel_invocations", C.c_int64), ("lane_slots", C.c_int64),
                ("useful_interactions", C.c_int64), ("pair_interactions", C.c_int64),
                ("epot", C.c_double), ("virial", C.c_double),
                ("pairs_owned_halo", C.c_int64),
                ("overlap", C.c_int32), ("overflow", C.c_int32)]


class Box(C.Structure):
    _fields_ = [("lo", C.c_double * 3), ("hi", C.c_double * 3),
                ("periodic", C.c_int32 * 3), ("pad", C.c_int32)]


class LJ(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("sigma", C.c_double),
                ("cutoff", C.c_double), ("skin", C.c_double)]


class Grid(C.Structure):
    _fields_ = [("dims", C.c_int64 * 3), ("tdims", C.c_int64 * 3),
                ("cell_len", C.c_double * 3), ("lo", C.c_double * 3),
                ("ncell", C.c_int64)]


STATS_BYTES = C.sizeof(Stats)

_VP = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_INT = C.c_int
_D = C.c_double
_SZ = C.c_size_t

# name -> (restype, argtypes); must match include/b200md.h
_SIGNATURES: dict[str, tuple] = {}


def _parse_header() -> list[str]:
    """Names of every function the public header declares."""
    hdr = os.path.join(_build.ROOT, "include", "b200md.h")
    with open(hdr, encoding="utf-8") as fh:
        text = fh.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lmd_[a-z0-9_]+)\s*\(", text)))


def declared_symbols() -> list[str]:
    return _parse_header()


def declared_arity() -> dict[str, int]:
    """Parameter count of every function the public header declares."""
    hdr = os.path.join(_build.ROOT, "include", "b200md.h")
    with open(hdr, encoding="utf-8") as fh:
        text = fh.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    out = {}
    for m in re.finditer(r"\b(lmd_[a-z0-9_]+)\s*\(([^)]*)\)\s*;", text):
        params = m.group(2).strip()
        out[m.group(1)] = 0 if params in ("", "void") else params.count(",") + 1
    return out


_lib: C.CDLL | None = None


def lib_path() -> str:
    return _build.lib_path()


def load(build_if_missing: bool = False) -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not os.path.exists(path):
        if build_if_missing:
            _build.build()
        else:
            raise NativeLibraryError(
                f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                " (the B200 force path has no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _sig(name, res, *args):
    _SIGNATURES[name] = (res, list(args))


_sig("lmd_version", _INT)
_sig("lmd_status_string", C.c_char_p, _INT)
_sig("lmd_device_sm_count", _INT)
_sig("lmd_grid_init", _INT, C.POINTER(Box), _D, C.POINTER(Grid))
_sig("lmd_cell_index", _INT, C.POINTER(Grid), _INT, _I64, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_sort_temp_bytes", _SZ, _I64)
_sig("lmd_sort_by_cell", _INT, _I64, _I64, _VP, _VP, _VP, _VP, _VP, _SZ, _VP)
_sig("lmd_cell_ranges", _INT, _I64, _I64, _I32, _VP, _VP, _VP, _VP)
_sig("lmd_merge_cell_tables", _INT, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_gather_pos4", _INT, _I64, _VP, _VP, _VP, _VP, _VP, _D, _VP, _VP)
_sig("lmd_halo_count", _INT, C.POINTER(Box), _D, _I64, _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_scan_temp_bytes", _SZ, _I64)
_sig("lmd_exclusive_scan_i32", _INT, _I64, _VP, _VP, _VP, _SZ, _VP)
_sig("lmd_halo_emit", _INT, C.POINTER(Box), _D, _I64, _VP, _VP, _VP, _VP, _VP,
     _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_halo_refresh_pos4", _INT, C.POINTER(Box), _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_lc_ev_slots", _I64, C.POINTER(Grid))
_sig("lmd_force_lc", _INT, C.POINTER(Grid), C.POINTER(LJ), _INT, _INT, _VP, _VP, _VP,
     _VP, _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_lc_stats", _INT, C.POINTER(Grid), _INT, _INT, _INT, _INT, _INT, _VP, _VP, _VP, _VP)
_sig("lmd_apply_boundaries", _INT, C.POINTER(Box), _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_verlet_step", _INT, _I64, _INT, _D, _D, *([_VP] * 13), _VP)
_sig("lmd_pair_sweep_ev_slots", _I64, _I64, _INT)
_sig("lmd_pair_sweep", _INT, _I64, _VP, _I64, _VP, _INT, _INT, _INT, _INT, C.POINTER(LJ),
     *([_VP] * 6), _VP, _VP, _VP)
_sig("lmd_buffer_counts", _INT, _I64, _VP, _VP, _VP)
_sig("lmd_dfma_burn", _INT, _INT, _INT, _INT, _VP, _VP)
_sig("lmd_gather_pos4_soa", _INT, _I64, _VP, _VP, _VP, _VP, _D, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_halo_refresh_pos4_soa", _INT, C.POINTER(Box), _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
     _VP, _VP, _VP)
_sig("lmd_halo_refresh_soa", _INT, C.POINTER(Box), _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
     _VP, _VP)
_sig("lmd_halo_refresh_rows", _INT, C.POINTER(Box), _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_gather_soa", _INT, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_vl_num_tiles", _I64, _I64, _INT)
_sig("lmd_vl_build", _INT, C.POINTER(Grid), _D, _INT, _INT, _I64, _I32, _VP, _VP, _VP, _VP, _VP,
     _I32, _VP, _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_vl_ev_slots", _I64, _I64, _INT)
_sig("lmd_ghost_pack", _INT, _I64, _VP, _I64, _VP, _VP, _VP, _VP, _INT, _D, _VP, _VP)
_sig("lmd_gather_pos4_rows", _INT, _I64, _VP, _VP, _D, _VP, _VP)
_sig("lmd_gather_rows_soa", _INT, _I64, _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_max_displacement2", _INT, _I64, _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_lc_tpi_ev_slots", _I64, _I64, _INT)
_sig("lmd_force_lc_particles", _INT, C.POINTER(Grid), C.POINTER(LJ), _INT, _INT, _VP, _I64, _VP,
     _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_vl_bank_smem_per_warp", C.c_size_t, _I32)
_sig("lmd_vl_groups", _INT, C.POINTER(Grid), _I64, _I32, _I32, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
     _VP)
_sig("lmd_vl_build_staged", _INT, C.POINTER(Grid), _D, _INT, _I64, _VP, _VP, _VP, _VP, _VP, _I32,
     _VP, _I32, _I32, _VP, _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_vl_staged_capacity", _I32, _I32)
_sig("lmd_force_vl_staged", _INT, _INT, _INT, C.POINTER(LJ), _I64, _VP, _VP, _I64, _I32, _I32, _VP,
     _I32, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_vl_bank_schedule", _INT, _INT, _I64, _I32, _INT, _I32, _I32, _I32, _VP, _VP, _VP, _VP)
_sig("lmd_vls_max_groups", _I64, C.POINTER(Grid), _I64)
_sig("lmd_vls_rows_for", _I32, _I32)
_sig("lmd_vls_plan_temp_bytes", _SZ, C.POINTER(Grid))
_sig("lmd_vls_plan", _INT, C.POINTER(Grid), _I64, *([_VP] * 9), _SZ, _VP, _VP, _VP)
_sig("lmd_vls_build_smem", _SZ, _I32, _I32)
_sig("lmd_vls_build", _INT, C.POINTER(Grid), _D, _D, _I64, _I32, _VP, _VP, _VP, _VP, _VP, _VP,
     _I64, _I32, _I32, _I32, _VP, _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_vls_ev_slots", _I64, _I64)
_sig("lmd_vls_force", _INT, _INT, _INT, C.POINTER(LJ), _I64, _I32, _VP, _VP, _I64, _VP, _I64,
     _VP, _VP, _VP, _I32, _VP, _D, _VP, _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_vls_direct", _INT, C.POINTER(Grid), _INT, _INT, C.POINTER(LJ), _I64, _I32, _VP, _VP,
     _VP, _VP, _VP, _VP, _I64, _I32, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_vls_reduce_ev", _INT, _I64, _VP, _VP, _VP)
_sig("lmd_vls_refresh", _INT, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _I32, C.POINTER(Box), _I64,
     _VP, _VP, _VP)
_sig("lmd_vls_gather_rows", _INT, _I64, _VP, _VP, _VP, _VP, _VP, _I32, _VP)
_sig("lmd_vls_rows_to_legacy", _INT, _I64, _I64, _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_force_vl", _INT, _INT, _INT, _INT, C.POINTER(LJ), _I64, _VP, _VP, _I64, _VP, _VP,
     _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_vl_stats", _INT, _I64, _INT, _INT, _INT, _VP, _VP, _VP)
_sig("lmd_vcl_temp_bytes", _SZ, _I64)
_sig("lmd_vcl_order", _INT, _I64, _VP, _VP, _VP, _D, _D, _D, _I64, *([_VP] * 8), _SZ, _VP)
_sig("lmd_vcl_chunk", _INT, _I64, _INT, *([_VP] * 8), C.POINTER(_I64), _VP, _SZ, _VP)
_sig("lmd_vcl_backing", _INT, _I64, _I64, _INT, _VP, _VP, _VP, _VP, _VP, _D, _VP, _VP, _VP, _VP)
_sig("lmd_vcl_column_table", _INT, _I64, _VP, _VP, _VP, _I64, _VP)
_sig("lmd_vcl_pairs", _INT, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _I64, _I64, _INT, _D, _D,
     _VP, _VP, _VP, _VP, _VP)
_sig("lmd_vcl_ev_slots", _I64, _I64)
_sig("lmd_force_vcl_order", _INT, _I64, _INT, _INT, _INT, C.POINTER(LJ), *([_VP] * 16), _VP)
_sig("lmd_force_vcl", _INT, _I64, _INT, _INT, C.POINTER(LJ), *([_VP] * 12), _I64, _VP, _D, _VP)
_sig("lmd_vcl_stats", _INT, _I64, _INT, _INT, _INT, _INT, _INT, *([_VP] * 8), _I64, _VP, _VP,
     _VP)
_sig("lmd_vcl_collect", _INT, _I64, *([_VP] * 8), _VP)
_sig("lmd_lc_n3_ev_slots", _I64, C.POINTER(Grid))
_sig("lmd_force_lc_n3", _INT, C.POINTER(Grid), C.POINTER(LJ), _INT, _INT, _INT, _VP, _I64,
     _VP, _VP, _VP, _VP, _VP, _INT, _VP, _VP, _VP, _VP, _VP, _VP)
_sig("lmd_execute_packed", _INT, _I64, *([_VP] * 7), _INT, C.POINTER(C.c_int64), _VP, _VP, _INT,
     C.POINTER(LJ),
     *([_VP] * 9), _VP)
_sig("lmd_scatter_forces", _INT, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP)


def check(status: int, what: str = "") -> None:
    """Map a C-ABI status onto the reference's exception hierarchy."""
    if status == OK:
        return
    msg = load().lmd_status_string(status).decode()
    where = f"{what}: " if what else ""
    if status == ERR_CONFIG:
        raise ConfigurationError(where + msg)
    if status == ERR_DEGENERATE:
        raise DegenerateDomainError(where + msg)
    if status == ERR_OVERLAP:
        raise ParticleOverlapError(where + msg)
    raise NativeLibraryError(where + msg)


_FUNCS: dict = {}


def call(name: str, *args) -> None:
    f = _FUNCS.get(name)
    if f is None:
        f = _FUNCS[name] = getattr(load(), name)
    check(f(*args), name)


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise NativeLibraryError("the B200 force path needs CUDA tensors (no CPU fallback)")
    return t.data_ptr()


def stream() -> int:
    """The current CUDA stream of the current device (raw handle): kernels go
    wherever torch's work goes, including a graph-capture stream."""
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


# per-object caches of the ctypes structs (boxes and LJ parameters are frozen
# dataclasses; the cache holds the object, so its id is not reused)
_STRUCT_CACHE: dict = {}


def make_box(box) -> Box:
    hit = _STRUCT_CACHE.get(("box", id(box)))
    if hit is not None and hit[0] is box:
        return hit[1]
    b = Box()
    for ax in range(3):
        b.lo[ax] = float(box.min[ax])
        b.hi[ax] = float(box.max[ax])
        b.periodic[ax] = 1 if ax in box.periodic_axes else 0
    if len(_STRUCT_CACHE) < 4096:
        _STRUCT_CACHE[("box", id(box))] = (box, b)
    return b


def make_lj(params) -> LJ:
    hit = _STRUCT_CACHE.get(("lj", id(params)))
    if hit is not None and hit[0] is params:
        return hit[1]
    lj = LJ(float(params.epsilon), float(params.sigma), float(params.cutoff),
            float(params.skin))
    if len(_STRUCT_CACHE) < 4096:
        _STRUCT_CACHE[("lj", id(params))] = (params, lj)
    return lj


def new_stats(device) -> torch.Tensor:
    return torch.zeros(STATS_BYTES, dtype=torch.uint8, device=device)


def read_stats(t: torch.Tensor) -> Stats:
    raw = t.cpu().numpy().tobytes()
    return Stats.from_buffer_copy(raw)


def I64_out() -> C.c_int64:
    """An int64 out-parameter (passed by reference through POINTER argtypes)."""
    return C.c_int64(0)
