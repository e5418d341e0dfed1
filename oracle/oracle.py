"""ctypes front end of the CPU oracle (oracle/zsvd_oracle.c).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package.
It restates the reference rangesvd hot path (svd.hpp, store.hpp, query.hpp);
see zsvd_oracle.h for the file:line map.
"""
from __future__ import annotations

import ctypes as C
import glob
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

ENERGY, FIXED_RANK = 0, 1
INCREMENTAL, DIRECT = 0, 1

OK, INVALID_INPUT, INVALID_PARAMETER, RANGE_ERROR, LOGIC_ERROR, NO_MEMORY = range(6)


class OracleError(Exception):
    def __init__(self, code: int, what: str = ""):
        super().__init__(f"oracle status {code} {what}")
        self.code = code


class _Factors(C.Structure):
    _fields_ = [("m", C.c_size_t), ("n", C.c_size_t), ("k", C.c_size_t),
                ("u", C.POINTER(C.c_double)), ("s", C.POINTER(C.c_double)),
                ("v", C.POINTER(C.c_double))]


class _Range(C.Structure):
    _fields_ = [(n, C.c_size_t) for n in ("first_row", "last_row", "start_block", "end_block",
                                          "skip_front", "keep_front", "keep_back", "skip_back")]


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(
                os.path.join(HERE, "zsvd_oracle.c")):
            build()
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        dp = P(C.c_double)
        fp = P(_Factors)
        L.zo_thin_svd.argtypes = [dp, C.c_size_t, C.c_size_t, fp]
        L.zo_truncate.argtypes = [fp, C.c_int, C.c_double, C.c_size_t, fp]
        L.zo_canonical_sign.argtypes = [fp]
        L.zo_orthonormality_defect.argtypes = [dp, C.c_size_t, C.c_size_t]
        L.zo_orthonormality_defect.restype = C.c_double
        L.zo_factors_free.argtypes = [fp]
        L.zo_trim_block.argtypes = [fp, C.c_size_t, C.c_size_t, C.c_int, C.c_double, C.c_size_t, fp]
        L.zo_stitch.argtypes = [fp, C.c_size_t, C.c_int, C.c_double, C.c_size_t, fp]
        L.zo_store_create.argtypes = [C.c_size_t, C.c_size_t, C.c_int, C.c_double, C.c_size_t,
                                      C.c_int, P(C.c_int)]
        L.zo_store_create.restype = C.c_void_p
        L.zo_store_destroy.argtypes = [C.c_void_p]
        L.zo_store_append.argtypes = [C.c_void_p, dp, C.c_size_t]
        for f in ("zo_store_total_rows", "zo_store_sealed_count", "zo_store_open_rows"):
            getattr(L, f).argtypes = [C.c_void_p]
            getattr(L, f).restype = C.c_size_t
        L.zo_store_block.argtypes = [C.c_void_p, C.c_size_t, fp]
        L.zo_resolve.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, P(_Range)]
        L.zo_range_query.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, C.c_int, C.c_double,
                                     C.c_size_t, fp]
        L.zo_open_block_from_row.argtypes = [dp, C.c_size_t, fp]
        L.zo_incremental_update.argtypes = [fp, C.c_size_t, dp, C.c_size_t, fp]
        L.zo_reorthonormalize.argtypes = [fp, fp]
        L.zo_set_backend.argtypes = [C.c_int, C.c_char_p]
        _lib = L
    return _lib


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _check(code: int, what: str = ""):
    if code != OK:
        raise OracleError(code, what)


@dataclass
class Factors:
    """SvdFactors (svd.hpp:30-40): u m x k, s (k,), v n x k."""
    u: np.ndarray
    s: np.ndarray
    v: np.ndarray

    @property
    def rank(self) -> int:
        return int(self.s.shape[0])

    def reconstruct(self) -> np.ndarray:
        return (self.u * self.s) @ self.v.T


def _take(f: _Factors) -> Factors:
    m, n, k = f.m, f.n, f.k
    u = np.ctypeslib.as_array(f.u, shape=(m * k,)).reshape(m, k).copy() if m * k else np.zeros((m, k))
    s = np.ctypeslib.as_array(f.s, shape=(k,)).copy() if k else np.zeros((0,))
    v = np.ctypeslib.as_array(f.v, shape=(n * k,)).reshape(n, k).copy() if n * k else np.zeros((n, k))
    lib().zo_factors_free(C.byref(f))
    return Factors(u, s, v)


def _give(fa: Factors):
    """Build a borrowed _Factors view (arrays kept alive by the returned tuple)."""
    u = np.ascontiguousarray(fa.u, dtype=np.float64)
    s = np.ascontiguousarray(fa.s, dtype=np.float64)
    v = np.ascontiguousarray(fa.v, dtype=np.float64)
    st = _Factors(u.shape[0], v.shape[0], s.shape[0], _dptr(u), _dptr(s), _dptr(v))
    return st, (u, s, v)


def set_backend(name: str) -> None:
    """'jacobi' (default) or 'lapack' (OpenBLAS dgesdd, single thread)."""
    if name == "jacobi":
        _check(lib().zo_set_backend(0, None))
        return
    import scipy
    cands = glob.glob(os.path.join(os.path.dirname(os.path.dirname(scipy.__file__)),
                                   "scipy.libs", "libscipy_openblas*.so"))
    if not cands:
        raise OracleError(INVALID_PARAMETER, "no OpenBLAS found for the lapack backend")
    _check(lib().zo_set_backend(1, cands[0].encode()))


def thin_svd(a: np.ndarray) -> Factors:
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("2-D input expected")
    f = _Factors()
    _check(lib().zo_thin_svd(_dptr(a), a.shape[0], a.shape[1], C.byref(f)), "thin_svd")
    return _take(f)


def truncate(f: Factors, policy=ENERGY, xi=1.0, k=0) -> Factors:
    src, keep = _give(f)
    out = _Factors()
    _check(lib().zo_truncate(C.byref(src), policy, xi, k, C.byref(out)), "truncate")
    return _take(out)


def canonical_sign(f: Factors) -> Factors:
    src, keep = _give(Factors(f.u.copy(), f.s.copy(), f.v.copy()))
    lib().zo_canonical_sign(C.byref(src))
    return Factors(keep[0], keep[1], keep[2])


def orthonormality_defect(m: np.ndarray) -> float:
    m = np.ascontiguousarray(m, dtype=np.float64)
    d = lib().zo_orthonormality_defect(_dptr(m), m.shape[0], m.shape[1])
    if d < 0:
        raise OracleError(INVALID_INPUT, "orthonormality_defect: wide matrix")
    return d


def trim_block(block: Factors, keep_from: int, keep_to: int, policy=ENERGY, xi=1.0, k=0) -> Factors:
    src, keep = _give(block)
    out = _Factors()
    _check(lib().zo_trim_block(C.byref(src), keep_from, keep_to, policy, xi, k, C.byref(out)),
           "trim_block")
    return _take(out)


def stitch(parts, policy=ENERGY, xi=1.0, k=0) -> Factors:
    arr = (_Factors * max(1, len(parts)))()
    keeps = []
    for i, p in enumerate(parts):
        st, kp = _give(p)
        arr[i] = st
        keeps.append(kp)
    out = _Factors()
    _check(lib().zo_stitch(arr, len(parts), policy, xi, k, C.byref(out)), "stitch")
    return _take(out)


def open_block_from_row(row) -> Factors:
    row = np.ascontiguousarray(row, dtype=np.float64)
    out = _Factors()
    _check(lib().zo_open_block_from_row(_dptr(row), row.shape[0], C.byref(out)))
    return _take(out)


def incremental_update(block: Factors, rows_seen: int, row, capacity: int) -> Factors:
    row = np.ascontiguousarray(row, dtype=np.float64)
    src, keep = _give(block)
    out = _Factors()
    _check(lib().zo_incremental_update(C.byref(src), rows_seen, _dptr(row), capacity, C.byref(out)))
    return _take(out)


def reorthonormalize(block: Factors) -> Factors:
    src, keep = _give(block)
    out = _Factors()
    _check(lib().zo_reorthonormalize(C.byref(src), C.byref(out)))
    return _take(out)


class Store:
    """BlockStore (store.hpp:161-249) in INCREMENTAL (reference) or DIRECT mode."""

    def __init__(self, b: int, c: int, xi: float = 1.0, policy: int = ENERGY, k: int = 0,
                 mode: int = INCREMENTAL):
        st = C.c_int(0)
        self._h = lib().zo_store_create(b, c, policy, xi, k, mode, C.byref(st))
        _check(st.value, "store_create")
        self.b, self.c, self.xi, self.policy, self.k = b, c, xi, policy, k

    def __del__(self):
        if getattr(self, "_h", None):
            lib().zo_store_destroy(self._h)
            self._h = None

    def append(self, rows) -> None:
        rows = np.ascontiguousarray(rows, dtype=np.float64)
        if rows.ndim == 1:
            rows = rows.reshape(1, -1)
        if rows.shape[1] != self.c:
            raise OracleError(INVALID_INPUT, "row has wrong number of columns")
        _check(lib().zo_store_append(self._h, _dptr(rows), rows.shape[0]), "append")

    @property
    def total_rows(self) -> int:
        return lib().zo_store_total_rows(self._h)

    @property
    def sealed_count(self) -> int:
        return lib().zo_store_sealed_count(self._h)

    @property
    def open_rows(self) -> int:
        return lib().zo_store_open_rows(self._h)

    def block(self, i: int) -> Factors:
        out = _Factors()
        _check(lib().zo_store_block(self._h, i, C.byref(out)), "block")
        return _take(out)

    def resolve(self, first: int, last: int) -> dict:
        r = _Range()
        _check(lib().zo_resolve(self._h, first, last, C.byref(r)), "resolve")
        return {n: getattr(r, n) for n, _ in _Range._fields_}

    def range_query(self, first: int, last: int, xi=None, policy=None, k=None) -> Factors:
        policy = self.policy if policy is None else policy
        xi = self.xi if xi is None else xi
        k = self.k if k is None else k
        out = _Factors()
        _check(lib().zo_range_query(self._h, first, last, policy, xi, k, C.byref(out)), "range_query")
        return _take(out)
