"""ctypes front-end of the CPU oracle (TEST INFRASTRUCTURE -- checker only).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this module.  The product package
(``paper_2512_03565_b200``) never does; it fails loudly without its CUDA
library instead of falling back here.

Every entry point restates a function of the reference package ``lanemd``
(``/root/reference/pkg/src/lanemd``); see the file:line citations in
``lj_oracle.c``.  Parity of the restatement against the unmodified reference is
pinned by ``tests/golden`` (fixtures generated with ``make_golden.py``).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))

TRAVERSAL_CODES = {"lc_c01": 0, "lc_c08": 1, "lc_c18": 2, "vcl": 3, "vl": 4}
PATTERN_SHAPES = {
    "one_by_v": lambda v: (1, v),
    "v_by_one": lambda v: (v, 1),
    "two_by_half": lambda v: (2, v // 2),
    "half_by_two": lambda v: (v // 2, 2),
}

OK, OVERLAP, DEGENERATE, CONFIG, NOMEM = 0, 1, 2, 3, 4


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"oracle {what} failed with code {code}")
        self.code = code


class _Stats(C.Structure):
    _fields_ = [("kernel_invocations", C.c_int64), ("lane_slots", C.c_int64),
                ("useful_interactions", C.c_int64), ("pair_interactions", C.c_int64),
                ("epot", C.c_double), ("virial", C.c_double),
                ("overlap", C.c_int32), ("pad", C.c_int32)]


@dataclass
class OracleStats:
    kernel_invocations: int
    lane_slots: int
    useful_interactions: int
    pair_interactions: int
    epot: float
    virial: float

    @property
    def blank_lanes(self) -> int:
        return self.lane_slots - self.useful_interactions

    def as_tuple(self):
        return (self.kernel_invocations, self.lane_slots,
                self.useful_interactions, self.pair_interactions)


def _stats(s: _Stats) -> OracleStats:
    return OracleStats(s.kernel_invocations, s.lane_slots, s.useful_interactions,
                       s.pair_interactions, s.epot, s.virial)


_LIBS: dict[str, C.CDLL] = {}


def build(quiet: bool = True) -> None:
    """Compile the oracle with its Makefile (gcc only)."""
    subprocess.run(["make", "-C", _HERE, "all"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def lib(omp: bool = False) -> C.CDLL:
    name = "liblj_oracle_omp.so" if omp else "liblj_oracle.so"
    if name not in _LIBS:
        path = os.path.join(_HERE, name)
        if not os.path.exists(path):
            build()
        _LIBS[name] = C.CDLL(path)
    return _LIBS[name]


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a, ctype=C.c_double):
    return a.ctypes.data_as(C.POINTER(ctype))


def _box_args(lo, hi, periodic):
    lo = _d(lo)
    hi = _d(hi)
    per = np.ascontiguousarray([1 if p else 0 for p in periodic], dtype=np.int32)
    return lo, hi, per


def _xyz(pos):
    pos = np.asarray(pos, dtype=np.float64).reshape(-1, 3)
    return _d(pos[:, 0]), _d(pos[:, 1]), _d(pos[:, 2])


def _own(n, ownership):
    if ownership is None:
        return np.zeros(n, dtype=np.int8)
    return np.ascontiguousarray(ownership, dtype=np.int8)


def force_phase_lc(pos, lo, hi, periodic, params, traversal: str, newton3: bool,
                   pattern: str, vector_width: int, ownership=None, omp=False):
    """driver.force_phase for linked cells: returns (forces (n,3), stats)."""
    x, y, z = _xyz(pos)
    n = len(x)
    own = _own(n, ownership)
    lo, hi, per = _box_args(lo, hi, periodic)
    a, b = PATTERN_SHAPES[pattern](vector_width)
    f = np.zeros((3, n))
    st = _Stats()
    L = lib(omp)
    rc = L.orc_force_phase_lc(
        C.c_int64(n), _p(x), _p(y), _p(z), _p(own, C.c_int8), _p(lo), _p(hi), _p(per, C.c_int32),
        C.c_double(params.epsilon), C.c_double(params.sigma), C.c_double(params.cutoff),
        C.c_double(params.skin), C.c_int(TRAVERSAL_CODES[traversal]), C.c_int(int(newton3)),
        C.c_int(a), C.c_int(b), C.c_int(vector_width),
        _p(f[0]), _p(f[1]), _p(f[2]), C.byref(st))
    if rc:
        raise OracleError(rc, "force_phase_lc")
    return f.T.copy(), _stats(st)


def force_phase_vcl(pos, lo, hi, periodic, params, cluster_size: int, newton3: bool,
                    pattern: str, vector_width: int, ownership=None):
    x, y, z = _xyz(pos)
    n = len(x)
    own = _own(n, ownership)
    lo, hi, per = _box_args(lo, hi, periodic)
    a, b = PATTERN_SHAPES[pattern](vector_width)
    f = np.zeros((3, n))
    st = _Stats()
    ncl = C.c_int64(0)
    ncol = C.c_int32(0)
    rc = lib().orc_force_phase_vcl(
        C.c_int64(n), _p(x), _p(y), _p(z), _p(own, C.c_int8), _p(lo), _p(hi), _p(per, C.c_int32),
        C.c_double(params.epsilon), C.c_double(params.sigma), C.c_double(params.cutoff),
        C.c_double(params.skin), C.c_int(cluster_size), C.c_int(int(newton3)),
        C.c_int(a), C.c_int(b), C.c_int(vector_width),
        _p(f[0]), _p(f[1]), _p(f[2]), C.byref(st), C.byref(ncl), C.byref(ncol))
    if rc:
        raise OracleError(rc, "force_phase_vcl")
    return f.T.copy(), _stats(st)


def force_phase_vl(pos, lo, hi, periodic, params, newton3: bool, pattern: str,
                   vector_width: int, ownership=None):
    """Verlet-list force phase (extension; see DESIGN.md for the stats rule)."""
    x, y, z = _xyz(pos)
    n = len(x)
    own = _own(n, ownership)
    lo, hi, per = _box_args(lo, hi, periodic)
    a, b = PATTERN_SHAPES[pattern](vector_width)
    f = np.zeros((3, n))
    st = _Stats()
    ne = C.c_int64(0)
    rc = lib().orc_force_phase_vl(
        C.c_int64(n), _p(x), _p(y), _p(z), _p(own, C.c_int8), _p(lo), _p(hi), _p(per, C.c_int32),
        C.c_double(params.epsilon), C.c_double(params.sigma), C.c_double(params.cutoff),
        C.c_double(params.skin), C.c_int(int(newton3)),
        C.c_int(a), C.c_int(b), C.c_int(vector_width),
        _p(f[0]), _p(f[1]), _p(f[2]), C.byref(st), C.byref(ne))
    if rc:
        raise OracleError(rc, "force_phase_vl")
    return f.T.copy(), _stats(st)


def lc_bin(pos, lo, hi, length: float, ring: bool = False):
    """(cell linear index per particle, stable perm, dims)."""
    x, y, z = _xyz(pos)
    n = len(x)
    cell = np.zeros(n, dtype=np.int64)
    perm = np.zeros(n, dtype=np.int64)
    dims = np.zeros(3, dtype=np.int64)
    lo, hi, _ = _box_args(lo, hi, (0, 0, 0))
    rc = lib().orc_lc_bin(C.c_int64(n), _p(x), _p(y), _p(z), _p(lo), _p(hi),
                          C.c_double(length), C.c_int(int(ring)), _p(cell, C.c_int64),
                          _p(perm, C.c_int64), _p(dims, C.c_int64))
    if rc:
        raise OracleError(rc, "lc_bin")
    return cell, perm, dims


def build_halo(pos, lo, hi, periodic, margin: float, ownership=None):
    """(halo positions (h,3), owner index per image) in the reference order."""
    x, y, z = _xyz(pos)
    n = len(x)
    own = _own(n, ownership)
    lo, hi, per = _box_args(lo, hi, periodic)
    cap = 7 * n + 1
    hx, hy, hz = np.zeros(cap), np.zeros(cap), np.zeros(cap)
    hid = np.zeros(cap, dtype=np.int64)
    L = lib()
    L.orc_build_halo.restype = C.c_int64
    cnt = L.orc_build_halo(C.c_int64(n), _p(x), _p(y), _p(z), _p(own, C.c_int8), _p(lo), _p(hi),
                           _p(per, C.c_int32), C.c_double(margin), _p(hx), _p(hy), _p(hz),
                           _p(hid, C.c_int64))
    if cnt < 0:
        raise OracleError(int(cnt), "build_halo")
    return np.stack([hx[:cnt], hy[:cnt], hz[:cnt]], axis=1), hid[:cnt]


def pair_sweep(pos_i, pos_j, params, newton3: bool, same: bool, pattern: str,
               vector_width: int, own_i=None, own_j=None, f_i=None, f_j=None):
    """compute_pair_vectorized on two buffers; returns (f_i, f_j, stats)."""
    xi, yi, zi = _xyz(pos_i)
    ni = len(xi)
    oi = _own(ni, own_i)
    fi = np.zeros((3, ni)) if f_i is None else np.ascontiguousarray(np.asarray(f_i, float).T)
    if same:
        xj, yj, zj, oj, fj, nj = xi, yi, zi, oi, fi, ni
    else:
        xj, yj, zj = _xyz(pos_j)
        nj = len(xj)
        oj = _own(nj, own_j)
        fj = np.zeros((3, nj)) if f_j is None else np.ascontiguousarray(np.asarray(f_j, float).T)
    a, b = PATTERN_SHAPES[pattern](vector_width)
    st = _Stats()
    rc = lib().orc_pair_sweep(
        C.c_int64(ni), _p(xi), _p(yi), _p(zi), _p(oi, C.c_int8), _p(fi[0]), _p(fi[1]), _p(fi[2]),
        C.c_int64(nj), _p(xj), _p(yj), _p(zj), _p(oj, C.c_int8), _p(fj[0]), _p(fj[1]), _p(fj[2]),
        C.c_double(params.epsilon), C.c_double(params.sigma), C.c_double(params.cutoff),
        C.c_int(int(newton3)), C.c_int(int(same)), C.c_int(a), C.c_int(b), C.c_int(vector_width),
        C.byref(st))
    if rc:
        raise OracleError(rc, "pair_sweep")
    return fi.T.copy(), fj.T.copy(), _stats(st)


def vcl_structure(pos, lo, hi, length: float, cluster_size: int):
    x, y, z = _xyz(pos)
    n = len(x)
    order = np.zeros(n, dtype=np.int64)
    slots = np.zeros(n, dtype=np.int64)
    counts = np.zeros(n + 1, dtype=np.int64)
    ncl = C.c_int64(0)
    cap = (n + 1) * cluster_size
    amin = np.zeros(3 * (n + 1))
    amax = np.zeros(3 * (n + 1))
    px, py, pz = np.zeros(cap), np.zeros(cap), np.zeros(cap)
    lo, hi, _ = _box_args(lo, hi, (0, 0, 0))
    rc = lib().orc_vcl_structure(C.c_int64(n), _p(x), _p(y), _p(z), _p(lo), _p(hi),
                                 C.c_double(length), C.c_int(cluster_size),
                                 _p(order, C.c_int64), _p(slots, C.c_int64), _p(counts, C.c_int64),
                                 C.byref(ncl), _p(amin), _p(amax), _p(px), _p(py), _p(pz))
    if rc:
        raise OracleError(rc, "vcl_structure")
    k = ncl.value
    m = k * cluster_size
    return dict(order=order, slots=slots, counts=counts[:k],
                aabb_min=amin[:3 * k].reshape(k, 3), aabb_max=amax[:3 * k].reshape(k, 3),
                padded=np.stack([px[:m], py[:m], pz[:m]], axis=1))


def vl_pairs(pos, lo, hi, periodic, length: float, newton3: bool):
    """Verlet-list pairs as (id_i, id_j, j_is_halo) arrays."""
    x, y, z = _xyz(pos)
    n = len(x)
    lo, hi, per = _box_args(lo, hi, periodic)
    L = lib()
    L.orc_vl_pairs.restype = C.c_int64
    cap = max(1024, 200 * n)
    while True:
        pi = np.zeros(cap, dtype=np.int64)
        pj = np.zeros(cap, dtype=np.int64)
        ph = np.zeros(cap, dtype=np.int8)
        cnt = L.orc_vl_pairs(C.c_int64(n), _p(x), _p(y), _p(z), _p(lo), _p(hi), _p(per, C.c_int32),
                             C.c_double(length), C.c_int(int(newton3)), C.c_int64(cap),
                             _p(pi, C.c_int64), _p(pj, C.c_int64), _p(ph, C.c_int8))
        if cnt == -3:
            cap *= 4
            continue
        if cnt < 0:
            raise OracleError(int(cnt), "vl_pairs")
        return pi[:cnt], pj[:cnt], ph[:cnt]


def verlet(state: dict, phase: int, dt: float, mass: float) -> None:
    """integrator.velocity_verlet_step on a dict of (n,) float64 arrays, in place."""
    keys = ("x", "y", "z", "vx", "vy", "vz", "fx", "fy", "fz", "ox", "oy", "oz")
    arrs = [state[k] for k in keys]
    for a in arrs:
        assert a.dtype == np.float64 and a.flags.c_contiguous
    lib().orc_verlet(C.c_int64(len(state["x"])), C.c_int(phase), C.c_double(dt), C.c_double(mass),
                     *[_p(a) for a in arrs])


def apply_boundaries(state: dict, lo, hi, periodic) -> bool:
    """domain.apply_boundaries in place; returns True on divergence."""
    lo, hi, per = _box_args(lo, hi, periodic)
    arrs = [state[k] for k in ("x", "y", "z", "vx", "vy", "vz")]
    rc = lib().orc_apply_boundaries(C.c_int64(len(state["x"])), _p(lo), _p(hi), _p(per, C.c_int32),
                                    *[_p(a) for a in arrs])
    return bool(rc)


class PreparedLC:
    """orc_lc_prepare / orc_lc_execute: the reference's execute_packed timed
    apart from rebuild/halo/schedule (driver.py:203-207).  ``threads > 1``
    (Newton3 off only) runs per-i-cell unit groups in parallel, bitwise
    identical to the sequential sweep."""

    def __init__(self, pos, lo, hi, periodic, params, traversal: str, newton3: bool,
                 pattern: str, vector_width: int, omp: bool = True):
        x, y, z = _xyz(pos)
        self._keep = (x, y, z)
        n = len(x)
        self.n = n
        own = np.zeros(n, dtype=np.int8)
        self._own = own
        lo, hi, per = _box_args(lo, hi, periodic)
        a, b = PATTERN_SHAPES[pattern](vector_width)
        self.L = lib(omp)
        self.L.orc_lc_prepare.restype = C.c_void_p
        self.L.orc_lc_execute.argtypes = [C.c_void_p, C.c_int, C.POINTER(_Stats),
                                          C.c_void_p, C.c_void_p, C.c_void_p]
        self.L.orc_lc_free.argtypes = [C.c_void_p]
        status = C.c_int(0)
        self.h = self.L.orc_lc_prepare(
            C.c_int64(n), _p(x), _p(y), _p(z), _p(own, C.c_int8), _p(lo), _p(hi),
            _p(per, C.c_int32), C.c_double(params.epsilon), C.c_double(params.sigma),
            C.c_double(params.cutoff), C.c_double(params.skin), C.c_int(TRAVERSAL_CODES[traversal]),
            C.c_int(int(newton3)), C.c_int(a), C.c_int(b), C.c_int(vector_width), C.byref(status))
        if status.value:
            self.close()
            raise OracleError(status.value, "orc_lc_prepare")

    def execute(self, threads: int = 1, want_forces: bool = False):
        st = _Stats()
        f = np.zeros((3, self.n)) if want_forces else None
        ptrs = [f[k].ctypes.data for k in range(3)] if want_forces else [None] * 3
        rc = self.L.orc_lc_execute(self.h, int(threads), C.byref(st), *ptrs)
        if rc:
            raise OracleError(rc, "orc_lc_execute")
        return (f.T.copy() if want_forces else None), _stats(st)

    def close(self):
        if getattr(self, "h", None):
            self.L.orc_lc_free(self.h)
            self.h = None

    def __del__(self):
        self.close()


def max_threads() -> int:
    return int(lib(True).orc_omp_max_threads())
