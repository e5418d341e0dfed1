"""Host-side mirror of the reference rangesvd API over the B200 C-ABI.

Same names, argument meaning and error types as the reference headers, so the
parity tests read like the reference's own GoogleTest suites:

    reference (proj/include/rangesvd)        here
    -------------------------------------    ------------------------------------
    BlockStore(b, c, xi)  store.hpp:163      BlockStore(b, c, xi, policy=, k=)
    BlockStore::append    store.hpp:182      BlockStore.append(rows)  (1 row or many)
    BlockStore::snapshot  store.hpp:200      BlockStore.snapshot()
    sealed()/open()       store.hpp:178-179  BlockStore.block(i) / .sealed() / .open()
    StoreSnapshot         store.hpp:135-156  StoreSnapshot
    TimeRange::resolve    query.hpp:34-51    StoreSnapshot.resolve(first, last)
    range_query           query.hpp:163-201  range_query(store_or_snapshot, first, last, xi)
    trim_block            query.hpp:64-89    trim_block(f, keep_from, keep_to, xi)
    stitch                query.hpp:150-157  stitch(parts, xi)
    thin_svd              svd.hpp:90-131     thin_svd(a)
    truncate_rank         svd.hpp:135-164    truncate_rank(f, xi)
    canonical_sign        svd.hpp:179-203    canonical_sign(f)
    errors.hpp:9-68                          Error, InvalidInputError, ...

Every numerical step runs in libzsvd.so on the GPU.  This module only moves
arguments and results; it never computes factors itself.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence, Union

import numpy as np

from . import _capi
from ._capi import lib


# ------------------------------------------------------------------ errors
class Error(RuntimeError):
    """rangesvd::Error (errors.hpp:10)."""


class InvalidInputError(Error):
    """errors.hpp:16."""


class InvalidParameterError(Error):
    """errors.hpp:22."""


class RangeError(Error):
    """errors.hpp:28."""


class LogicError(Error):
    """std::logic_error (store.hpp:65-67)."""


class CudaError(Error):
    """Device or runtime failure (no reference analogue)."""


class UnsupportedError(Error):
    """Shape outside this build's kernels (min(b, c) above 1024)."""


class IoError(Error):
    """errors.hpp:52: a file cannot be read or written."""


class FormatError(Error):
    """errors.hpp:58: not a ZSVD v1 store file (magic, version)."""


class CorruptionError(Error):
    """errors.hpp:65: a store file is structurally damaged."""


class ParseError(Error):
    """errors.hpp:34-45: malformed CSV text; ``line`` is 1-based."""

    def __init__(self, what: str, line: int = 0):
        super().__init__(what)
        self.line = int(line)


class SchemaError(Error):
    """errors.hpp:47: the CSV has a different column layout than requested."""


_ERRORS = {
    _capi.INVALID_INPUT: InvalidInputError,
    _capi.INVALID_PARAMETER: InvalidParameterError,
    _capi.RANGE: RangeError,
    _capi.LOGIC: LogicError,
    _capi.CUDA: CudaError,
    _capi.NO_MEMORY: CudaError,
    _capi.UNSUPPORTED: UnsupportedError,
    _capi.IO: IoError,
    _capi.FORMAT: FormatError,
    _capi.CORRUPTION: CorruptionError,
    _capi.SCHEMA: SchemaError,
}


def _check(code: int) -> None:
    if code == _capi.OK:
        return
    buf = C.create_string_buffer(4096)
    lib().zsvd_last_error(buf, 4096)
    msg = buf.value.decode("latin-1")
    if code == _capi.PARSE:
        raise ParseError(msg, int(lib().zsvd_last_error_line()))
    raise _ERRORS.get(code, Error)(msg)


# --------------------------------------------------------------- policies
TruncArg = Union[float, "Truncation", None]


@dataclass(frozen=True)
class Truncation:
    """ENERGY(xi) = truncate_rank; FIXED_RANK(k) = min(k, numerical rank)
    (SURVEY App. A #1)."""
    policy: int = _capi.POLICY_ENERGY
    xi: float = 1.0
    k: int = 0

    @staticmethod
    def energy(xi: float) -> "Truncation":
        return Truncation(_capi.POLICY_ENERGY, float(xi), 0)

    @staticmethod
    def fixed_rank(k: int) -> "Truncation":
        return Truncation(_capi.POLICY_FIXED_RANK, 1.0, int(k))

    def c(self) -> _capi.Truncation:
        return _capi.Truncation(self.policy, self.xi, max(0, self.k))


def _trunc(t: TruncArg, default: Optional[Truncation] = None) -> Truncation:
    if t is None:
        if default is None:
            raise InvalidParameterError("a truncation threshold is required")
        return default
    if isinstance(t, Truncation):
        return t
    return Truncation.energy(float(t))


# ---------------------------------------------------------------- factors
@dataclass
class SvdFactors:
    """rangesvd::SvdFactors (svd.hpp:30-40), host copy: u m x k, sigma (k,), v n x k."""
    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray

    def rank(self) -> int:
        return int(self.sigma.shape[0])

    def left_rows(self) -> int:
        return int(self.u.shape[0])

    def right_rows(self) -> int:
        return int(self.v.shape[0])


class DeviceFactors:
    """A device-resident SvdFactors (zsvd_factors*).  download() copies it out."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _capi._lib is not None:
            lib().zsvd_factors_release(h)
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def shape(self):
        m, n, k = C.c_size_t(), C.c_size_t(), C.c_size_t()
        _check(lib().zsvd_factors_shape(self._h, C.byref(m), C.byref(n), C.byref(k)))
        return m.value, n.value, k.value

    def rank(self) -> int:
        return self.shape()[2]

    def download(self) -> SvdFactors:
        m, n, k = self.shape()
        u = np.zeros((m, k))
        s = np.zeros((k,))
        v = np.zeros((n, k))
        _check(lib().zsvd_factors_copy(self._h, u.ctypes.data, s.ctypes.data, v.ctypes.data))
        return SvdFactors(u, s, v)

    @staticmethod
    def upload(f: SvdFactors) -> "DeviceFactors":
        u = np.ascontiguousarray(f.u, dtype=np.float64)
        s = np.ascontiguousarray(f.sigma, dtype=np.float64)
        v = np.ascontiguousarray(f.v, dtype=np.float64)
        out = C.c_void_p()
        _check(lib().zsvd_factors_upload(u.ctypes.data, s.ctypes.data, v.ctypes.data, u.shape[0],
                                         v.shape[0], s.shape[0], C.byref(out)))
        return DeviceFactors(out.value)


def _as_device(f: Union[SvdFactors, DeviceFactors]) -> DeviceFactors:
    return f if isinstance(f, DeviceFactors) else DeviceFactors.upload(f)


# ------------------------------------------------------ L1: svd.hpp ops
def thin_svd(a) -> SvdFactors:
    """svd.hpp:90-131."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise InvalidInputError("thin_svd: 2-D matrix expected")
    a = np.ascontiguousarray(a)
    if a.shape[0] < 1 or a.shape[1] < 1:
        raise InvalidInputError("thin_svd: matrix must have at least one row and one column")
    out = C.c_void_p()
    _check(lib().zsvd_thin_svd(a.ctypes.data, a.shape[0], a.shape[1], _capi.MEM_HOST, C.byref(out)))
    return DeviceFactors(out.value).download()


def truncate_rank(f: Union[SvdFactors, DeviceFactors], xi: TruncArg) -> SvdFactors:
    """svd.hpp:135-164 (xi float) or a Truncation policy."""
    t = _trunc(xi)
    d = _as_device(f)
    out = C.c_void_p()
    _check(lib().zsvd_truncate(d.handle, t.c(), C.byref(out)))
    return DeviceFactors(out.value).download()


def canonical_sign(f: Union[SvdFactors, DeviceFactors]) -> SvdFactors:
    """svd.hpp:179-203."""
    d = _as_device(f)
    out = C.c_void_p()
    _check(lib().zsvd_canonical_sign(d.handle, C.byref(out)))
    return DeviceFactors(out.value).download()


# ---------------------------------------------------- L3: query.hpp ops
def trim_block(block: Union[SvdFactors, DeviceFactors], keep_from: int, keep_to: int,
               xi: TruncArg) -> SvdFactors:
    """query.hpp:64-89."""
    t = _trunc(xi)
    if keep_from < 0 or keep_to < 0:
        raise InvalidParameterError("trim_block: empty or out-of-bounds keep range")
    d = _as_device(block)
    out = C.c_void_p()
    _check(lib().zsvd_trim_block(d.handle, keep_from, keep_to, t.c(), C.byref(out)))
    return DeviceFactors(out.value).download()


def stitch(parts: Sequence[Union[SvdFactors, DeviceFactors]], xi: TruncArg) -> SvdFactors:
    """query.hpp:150-157."""
    t = _trunc(xi)
    devs = [_as_device(p) for p in parts]
    arr = (C.c_void_p * max(1, len(devs)))(*[d.handle.value for d in devs])
    out = C.c_void_p()
    _check(lib().zsvd_stitch(arr, len(devs), t.c(), C.byref(out)))
    return DeviceFactors(out.value).download()


# ------------------------------------------------------------- L2: store
@dataclass
class TimeRange:
    """query.hpp:19-31."""
    first_row: int
    last_row: int
    start_block: int
    end_block: int
    skip_front: int
    keep_front: int
    keep_back: int
    skip_back: int

    def length(self) -> int:
        return self.last_row - self.first_row + 1


@dataclass
class RangeSvd:
    """query.hpp:55-60."""
    factors: SvdFactors

    def rows(self) -> int:
        return self.factors.left_rows()

    def rank(self) -> int:
        return self.factors.rank()


class StoreSnapshot:
    """store.hpp:135-156.  Valid while its store lives."""

    def __init__(self, store: "BlockStore"):
        self._store = store
        h = C.c_void_p()
        _check(lib().zsvd_snapshot_create(store._h, C.byref(h)))
        self._h = h
        info = _capi.StoreInfo()
        _check(lib().zsvd_snapshot_info_get(self._h, C.byref(info)))
        self.block_size = info.block_size
        self.num_columns = info.num_columns
        self.total_rows = info.total_rows
        self.sealed_count = info.sealed_count
        self.open_rows = info.open_rows
        self.energy_threshold = store.energy_threshold()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _capi._lib is not None:
            lib().zsvd_snapshot_release(h)
            self._h = None

    def block_count(self) -> int:
        return self.sealed_count + (1 if self.open_rows else 0)

    def block_rows(self, i: int) -> int:
        return self.block_size if i < self.sealed_count else self.open_rows

    def resolve(self, first: int, last: int) -> TimeRange:
        if first < 0 or last < 0:
            raise RangeError("time range out of bounds")
        r = _capi.TimeRangeC()
        _check(lib().zsvd_resolve(self._h, first, last, C.byref(r)))
        return TimeRange(*[getattr(r, n) for n, _ in _capi.TimeRangeC._fields_])

    def stream(self) -> int:
        s = C.c_void_p()
        _check(lib().zsvd_snapshot_stream(self._h, C.byref(s)))
        return s.value or 0

    def query_device(self, first: int, last: int, xi: TruncArg = None) -> DeviceFactors:
        """Enqueues range_query; the answer stays on the device (no wait)."""
        t = _trunc(xi, self._store.truncation)
        if first < 0 or last < 0:
            raise RangeError("time range out of bounds")
        out = C.c_void_p()
        _check(lib().zsvd_range_query(self._h, first, last, t.c(), C.byref(out)))
        return DeviceFactors(out.value)


class BlockStore:
    """store.hpp:161-249 over zsvd_store*.  ``xi`` alone = the reference's
    energy policy; ``policy=Truncation.fixed_rank(k)`` = the BASELINE configs."""

    def __init__(self, block_size: int, num_columns: int, energy_threshold: Optional[float] = None,
                 *, policy: Optional[Truncation] = None, device: int = 0):
        if policy is None:
            policy = Truncation.energy(1.0 if energy_threshold is None else energy_threshold)
        if block_size < 1 or num_columns < 1:
            raise InvalidParameterError("block size and column count must be at least 1")
        self.truncation = policy
        h = C.c_void_p()
        self._h = None
        _check(lib().zsvd_store_create_ex(block_size, num_columns, policy.c(), device, C.byref(h)))
        self._h = h
        self._b, self._c = int(block_size), int(num_columns)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _capi._lib is not None:
            lib().zsvd_store_destroy(h)
            self._h = None

    # accessors (store.hpp:173-179)
    def block_size(self) -> int:
        return self._b

    def num_columns(self) -> int:
        return self._c

    def energy_threshold(self) -> float:
        return self.truncation.xi

    def info(self) -> _capi.StoreInfo:
        i = _capi.StoreInfo()
        _check(lib().zsvd_store_info_get(self._h, C.byref(i)))
        return i

    def total_rows(self) -> int:
        return self.info().total_rows

    def sealed_count(self) -> int:
        return self.info().sealed_count

    def open_rows(self) -> int:
        return self.info().open_rows

    # storage phase
    def append(self, rows) -> None:
        """BlockStore::append (store.hpp:182): one row (1-D) or many (2-D)."""
        a = np.asarray(rows, dtype=np.float64)
        if a.ndim == 1:
            a = a.reshape(1, -1)
        if a.ndim != 2 or a.shape[1] != self._c:
            raise InvalidInputError("row has wrong number of columns")
        a = np.ascontiguousarray(a)
        _check(lib().zsvd_store_append(self._h, a.ctypes.data, a.shape[0], a.shape[1], _capi.MEM_HOST))

    def append_csv(self, path, options: Optional["CsvOptions"] = None) -> int:
        """Appends every row of a CSV file (cmd_ingest's loop, commands.hpp:
        119-123), parsed on the GPU and appended from HBM.  All or nothing: a
        ParseError / SchemaError leaves the store untouched.  Returns the rows
        appended."""
        csv = _CsvFile(path, options, self.info().device)
        n = C.c_size_t()
        _check(lib().zsvd_store_append_csv(self._h, csv.h, C.byref(n)))
        return n.value

    def append_ptr(self, ptr: int, nrows: int, ld: int, memory: int) -> None:
        """Appends rows from a raw host or device pointer (HBM-resident input)."""
        _check(lib().zsvd_store_append(self._h, ptr, nrows, ld, memory))

    def sync(self) -> None:
        _check(lib().zsvd_store_sync(self._h))

    def stream(self) -> int:
        s = C.c_void_p()
        _check(lib().zsvd_store_stream(self._h, C.byref(s)))
        return s.value or 0

    def block(self, i: int) -> SvdFactors:
        """Factors of block i (sealed, or the open tail at i == sealed_count)."""
        k = C.c_size_t()
        _check(lib().zsvd_store_block_rank(self._h, i, C.byref(k)))
        info = self.info()
        rows = self._b if i < info.sealed_count else info.open_rows
        k = k.value
        u = np.zeros((rows, k))
        s = np.zeros((k,))
        v = np.zeros((self._c, k))
        _check(lib().zsvd_store_block_copy(self._h, i, u.ctypes.data, s.ctypes.data, v.ctypes.data))
        return SvdFactors(u, s, v)

    def sealed(self):
        return [self.block(i) for i in range(self.sealed_count())]

    def open(self) -> Optional[SvdFactors]:
        info = self.info()
        return self.block(info.sealed_count) if info.open_rows else None

    def snapshot(self) -> StoreSnapshot:
        return StoreSnapshot(self)

    # profiling of the storage kernel (bench.py)
    def profile(self, enable: bool) -> None:
        _check(lib().zsvd_store_profile(self._h, 1 if enable else 0))

    def profile_read(self):
        a, b, ms = C.c_uint64(), C.c_uint64(), C.c_double()
        _check(lib().zsvd_store_profile_read(self._h, C.byref(a), C.byref(b), C.byref(ms)))
        return a.value, b.value, ms.value


def range_query(src: Union[BlockStore, StoreSnapshot], first: int, last: int,
                xi: TruncArg = None) -> RangeSvd:
    """query.hpp:163-201: SVD of rows [first, last], sign-canonicalised."""
    snap = src.snapshot() if isinstance(src, BlockStore) else src
    if xi is None:
        xi = snap._store.truncation
    return RangeSvd(snap.query_device(first, last, xi).download())


def naive_range_svd(src: Union[BlockStore, StoreSnapshot], first: int, last: int) -> SvdFactors:
    """analysis.hpp:49-66: the range's rows rebuilt from the stored factors,
    decomposed from scratch (on the GPU)."""
    snap = src.snapshot() if isinstance(src, BlockStore) else src
    out = C.c_void_p()
    _check(lib().zsvd_naive_range_svd(snap._h, int(first), int(last), C.byref(out)))
    return DeviceFactors(out.value).download()


def reconstruction_error(raw, f: Union[SvdFactors, DeviceFactors]) -> float:
    """analysis.hpp:20-37: ||X - U S V^T||_F^2 / ||X||_F^2 (GPU)."""
    x = np.ascontiguousarray(np.asarray(raw, dtype=np.float64))
    if x.ndim != 2:
        raise InvalidInputError("reconstruction_error: 2-D matrix expected")
    d = _as_device(f)
    e = C.c_double()
    _check(lib().zsvd_reconstruction_error(x.ctypes.data, x.shape[0], x.shape[1], _capi.MEM_HOST, d.handle,
                                           C.byref(e)))
    return float(e.value)


def save_store(store: BlockStore, path: str) -> None:
    """serialize.hpp:162-194: the ZSVD v1 file (energy stores; fixed-rank stores
    as the version-2 extension, see zsvd_store_save)."""
    _check(lib().zsvd_store_save(store._h, str(path).encode()))


def _adopt_store(h) -> BlockStore:
    st = BlockStore.__new__(BlockStore)
    st._h = h
    info = _capi.StoreInfo()
    _check(lib().zsvd_store_info_get(h, C.byref(info)))
    st._b, st._c = int(info.block_size), int(info.num_columns)
    if int(info.truncation.policy) == _capi.POLICY_FIXED_RANK:
        st.truncation = Truncation.fixed_rank(int(info.truncation.k))
    else:
        st.truncation = Truncation.energy(float(info.truncation.xi))
    return st


def load_store(path: str, device: int = 0) -> BlockStore:
    """serialize.hpp:196-254: a store resumed from a ZSVD v1 (or v2) file."""
    h = C.c_void_p()
    _check(lib().zsvd_store_load(str(path).encode(), device, C.byref(h)))
    return _adopt_store(h)


def store_from_parts(block_size: int, num_columns: int, policy: "Truncation", sealed, open_block=None,
                     device: int = 0) -> BlockStore:
    """BlockStore::from_parts (store.hpp:206-231): ``sealed`` is a list of
    Factors (block_size x k U, sigma, num_columns x k V) in block order;
    ``open_block`` is (rows_seen, Factors) or None.  Inconsistent counts or
    shapes raise InvalidInputError, like the reference."""
    keep = []

    def part(index, rows, f):
        u = np.ascontiguousarray(f.u, dtype=np.float64)
        sv = np.ascontiguousarray(getattr(f, "sigma", None) if hasattr(f, "sigma") else f.s, dtype=np.float64)
        v = np.ascontiguousarray(f.v, dtype=np.float64)
        if u.shape != (rows, sv.size) or v.shape != (num_columns, sv.size):
            raise InvalidInputError("from_parts: inconsistent block")
        keep.extend((u, sv, v))
        return _capi.BlockFactorsC(index, rows, sv.size, u.ctypes.data, sv.ctypes.data, v.ctypes.data)

    arr = (_capi.BlockFactorsC * max(1, len(sealed)))(*[part(i, block_size, f) for i, f in enumerate(sealed)])
    op = None
    if open_block is not None:
        rows_seen, f = open_block
        op = C.byref(part(len(sealed), int(rows_seen), f))
    h = C.c_void_p()
    _check(lib().zsvd_store_from_parts(block_size, num_columns, policy.c(), device, arr, len(sealed), op,
                                       C.byref(h)))
    return _adopt_store(h)


@dataclass
class SearchHit:
    """analysis.hpp:70-74: window start and |cos| of the leading left singular vectors."""
    window_start: int
    similarity: float


def similar_range_search(src: Union[BlockStore, StoreSnapshot], base_first: int, base_last: int,
                         stride: int, top_n: int, xi: TruncArg = None) -> List[SearchHit]:
    """analysis.hpp:78-148: the top_n windows [w, w + L - 1] (w = 0, stride, ...,
    ending before the base) most similar to the base range, all windows
    queried in batches on the GPU."""
    snap = src.snapshot() if isinstance(src, BlockStore) else src
    if xi is None:
        xi = snap._store.truncation
    t = _trunc(xi)
    if int(base_last) < int(base_first) or int(base_last) - int(base_first) + 1 < 2:
        raise InvalidParameterError("similar_range_search: base must span at least 2 rows")
    if int(stride) < 1:
        raise InvalidParameterError("similar_range_search: stride must be at least 1")
    cap = max(int(top_n), 0)
    starts = np.zeros(max(cap, 1), dtype=np.uint64)
    sims = np.zeros(max(cap, 1), dtype=np.float64)
    n = C.c_size_t()
    _check(lib().zsvd_similar_range_search(snap._h, int(base_first), int(base_last), int(stride), cap, t.c(),
                                           starts.ctypes.data, sims.ctypes.data, C.byref(n)))
    return [SearchHit(int(starts[i]), float(sims[i])) for i in range(n.value)]


# ------------------------------------------------------------ CSV (csv.hpp)
@dataclass
class CsvOptions:
    """csv.hpp:22-27."""
    expected_cols: Optional[int] = None
    drop_timestamp: bool = False

    def c(self) -> _capi.CsvOptionsC:
        return _capi.CsvOptionsC(-1 if self.expected_cols is None else int(self.expected_cols),
                                 1 if self.drop_timestamp else 0)


class _CsvFile:
    """A parsed file (zsvd_csv*): the rows on the device plus the pending error."""

    def __init__(self, path, options: Optional[CsvOptions], device: int = 0):
        self.h = None
        h = C.c_void_p()
        _check(lib().zsvd_csv_read(str(path).encode(), (options or CsvOptions()).c(), device, C.byref(h)))
        self.h = h
        r, c, e, ln = C.c_size_t(), C.c_size_t(), C.c_int(), C.c_size_t()
        _check(lib().zsvd_csv_info(h, C.byref(r), C.byref(c), C.byref(e), C.byref(ln)))
        self.rows, self.cols, self.error, self.error_line = r.value, c.value, e.value, ln.value
        buf = C.create_string_buffer(4096)
        _check(lib().zsvd_csv_error_message(h, buf, 4096))
        self.message = buf.value.decode("latin-1")

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value and _capi._lib is not None:
            lib().zsvd_csv_release(h)
            self.h = None

    def matrix(self) -> np.ndarray:
        out = np.empty((self.rows, self.cols), dtype=np.float64)
        if self.rows:
            _check(lib().zsvd_csv_rows_copy(self.h, 0, self.rows, out.ctypes.data))
        return out

    def device_ptr(self) -> int:
        p = C.c_void_p()
        _check(lib().zsvd_csv_rows_device(self.h, C.byref(p)))
        return p.value or 0

    def raise_error(self) -> None:
        if self.error == _capi.PARSE:
            raise ParseError(self.message, self.error_line)
        if self.error == _capi.SCHEMA:
            raise SchemaError(self.message)


class CsvReader:
    """csv.hpp:67-160: yields the file's rows in order, then raises the
    reader's ParseError / SchemaError (if any) where the reference would.  The
    whole file is parsed on the GPU when the reader is opened; an unopenable
    file raises IoError there (csv.hpp:71-76)."""

    def __init__(self, path, options: Optional[CsvOptions] = None, device: int = 0):
        self._f = _CsvFile(path, options, device)
        self._rows = self._f.matrix()
        self._i = 0

    def next(self) -> Optional[np.ndarray]:
        if self._i < self._rows.shape[0]:
            self._i += 1
            return self._rows[self._i - 1]
        self._f.raise_error()
        return None

    def cols(self) -> int:
        """Columns per row; 0 until the first data row has been read (csv.hpp:135-136)."""
        return self._f.cols if self._i > 0 else 0

    def __iter__(self):
        while True:
            r = self.next()
            if r is None:
                return
            yield r


def read_csv_rows(path, options: Optional[CsvOptions] = None, device: int = 0) -> List[np.ndarray]:
    """csv.hpp:153-161."""
    f = _CsvFile(path, options, device)
    f.raise_error()
    return list(f.matrix())


def read_csv_matrix(path, options: Optional[CsvOptions] = None, device: int = 0) -> np.ndarray:
    """csv.hpp:164-177: the whole file as a matrix; no data rows -> InvalidInputError."""
    f = _CsvFile(path, options, device)
    f.raise_error()
    if f.rows == 0:
        raise InvalidInputError(f"'{path}' contains no data rows")
    return f.matrix()


def ingest_csv(path, block_size: int, xi: float = 0.98, drop_timestamp: bool = False, *,
               policy: Optional[Truncation] = None, device: int = 0) -> BlockStore:
    """cmd_ingest's core (commands.hpp:106-127): a new store whose width is the
    CSV's, holding every row.  Errors as the reference: bad block size / xi ->
    InvalidParameterError, no data rows -> InvalidInputError, parse errors."""
    if block_size < 1:
        raise InvalidParameterError("--block-size must be at least 1")
    if policy is None and (not xi > 0.0 or xi > 1.0):
        raise InvalidParameterError("--xi must lie in (0, 1]")
    f = _CsvFile(path, CsvOptions(None, drop_timestamp), device)
    if f.rows == 0 and f.error == _capi.OK:
        raise InvalidInputError(f"'{path}' contains no data rows")
    f.raise_error()
    st = BlockStore(block_size, f.cols, xi, policy=policy, device=device)
    n = C.c_size_t()
    _check(lib().zsvd_store_append_csv(st._h, f.h, C.byref(n)))
    return st


def launch_count() -> int:
    """Kernels launched by libzsvd.so in this process."""
    return int(lib().zsvd_launch_count())


def direct_count() -> int:
    """FIXED_RANK factorisations finished by a direct route (waits for the device)."""
    return int(lib().zsvd_direct_count())


def fallback_count() -> int:
    """Factorisations the robust fallback path re-did (waits for the device)."""
    return int(lib().zsvd_fallback_count())


def device_count() -> int:
    n = C.c_int()
    code = lib().zsvd_device_count(C.byref(n))
    return n.value if code == _capi.OK else 0
