"""ctypes binding of libzsvd.so (include/zsvd.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a).  There is no fallback: importing this module without the library
raises, and every computing call fails loudly without a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libzsvd.so")

# zsvd_status
(OK, INVALID_INPUT, INVALID_PARAMETER, RANGE, LOGIC, CUDA, NO_MEMORY, UNSUPPORTED, IO, FORMAT, CORRUPTION, PARSE,
 SCHEMA) = range(13)
# zsvd_policy / zsvd_memory
POLICY_ENERGY, POLICY_FIXED_RANK = 0, 1
MEM_HOST, MEM_DEVICE = 0, 1


class Truncation(C.Structure):
    _fields_ = [("policy", C.c_int32), ("xi", C.c_double), ("k", C.c_uint64)]


class StoreInfo(C.Structure):
    _fields_ = [("block_size", C.c_uint64), ("num_columns", C.c_uint64), ("total_rows", C.c_uint64),
                ("sealed_count", C.c_uint64), ("open_rows", C.c_uint64), ("truncation", Truncation),
                ("device", C.c_int32)]


class CsvOptionsC(C.Structure):
    _fields_ = [("expected_cols", C.c_int64), ("drop_timestamp", C.c_int32)]


class BlockFactorsC(C.Structure):  # zsvd_block_factors
    _fields_ = [("index", C.c_uint64), ("rows", C.c_uint64), ("k", C.c_uint64),
                ("u", C.c_void_p), ("s", C.c_void_p), ("v", C.c_void_p)]


class TimeRangeC(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("first_row", "last_row", "start_block", "end_block",
                                          "skip_front", "keep_front", "keep_back", "skip_back")]


# Every symbol include/zsvd.h declares: name -> (restype, argtypes)
_vp = C.c_void_p
_pp = C.POINTER(C.c_void_p)
_dp = C.POINTER(C.c_double)
_sz = C.c_size_t
_szp = C.POINTER(C.c_size_t)
SIGNATURES = {
    "zsvd_version": (C.c_char_p, []),
    "zsvd_last_error": (C.c_int, [C.c_char_p, _sz]),
    "zsvd_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "zsvd_launch_count": (C.c_uint64, []),
    "zsvd_fallback_count": (C.c_uint64, []),
    "zsvd_direct_count": (C.c_uint64, []),
    "zsvd_store_create": (C.c_int, [_sz, _sz, C.c_double, _pp]),
    "zsvd_store_create_ex": (C.c_int, [_sz, _sz, Truncation, C.c_int, _pp]),
    "zsvd_store_destroy": (C.c_int, [_vp]),
    "zsvd_store_append": (C.c_int, [_vp, _vp, _sz, _sz, C.c_int]),
    "zsvd_store_info_get": (C.c_int, [_vp, C.POINTER(StoreInfo)]),
    "zsvd_store_block_rank": (C.c_int, [_vp, _sz, _szp]),
    "zsvd_store_block_copy": (C.c_int, [_vp, _sz, _vp, _vp, _vp]),
    "zsvd_store_sync": (C.c_int, [_vp]),
    "zsvd_store_reset": (C.c_int, [_vp]),
    "zsvd_store_spectrum": (C.c_int, [_vp, _sz, _sz, _vp, _sz, _vp]),
    "zsvd_store_stream": (C.c_int, [_vp, _pp]),
    "zsvd_store_profile": (C.c_int, [_vp, C.c_int]),
    "zsvd_store_profile_read": (C.c_int, [_vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                          C.POINTER(C.c_double)]),
    "zsvd_snapshot_create": (C.c_int, [_vp, _pp]),
    "zsvd_snapshot_release": (C.c_int, [_vp]),
    "zsvd_snapshot_info_get": (C.c_int, [_vp, C.POINTER(StoreInfo)]),
    "zsvd_snapshot_stream": (C.c_int, [_vp, _pp]),
    "zsvd_snapshot_block": (C.c_int, [_vp, _sz, _pp]),
    "zsvd_resolve": (C.c_int, [_vp, _sz, _sz, C.POINTER(TimeRangeC)]),
    "zsvd_range_query": (C.c_int, [_vp, _sz, _sz, Truncation, _pp]),
    "zsvd_store_save": (C.c_int, [_vp, C.c_char_p]),
    "zsvd_naive_range_svd": (C.c_int, [_vp, _sz, _sz, _pp]),
    "zsvd_reconstruction_error": (C.c_int, [_vp, _sz, _sz, C.c_int, _vp, C.POINTER(C.c_double)]),
    "zsvd_store_load": (C.c_int, [C.c_char_p, C.c_int, _pp]),
    "zsvd_store_from_parts": (C.c_int, [_sz, _sz, Truncation, C.c_int, _vp, _sz, _vp, _pp]),
    "zsvd_comm_unique_id": (C.c_int, [_vp]),
    "zsvd_comm_create": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _pp]),
    "zsvd_comm_destroy": (C.c_int, [_vp]),
    "zsvd_sharded_range_query": (C.c_int, [_vp, _vp, C.c_uint64, _sz, _sz, Truncation, _pp,
                                           C.POINTER(C.c_uint64)]),
    "zsvd_reconstruct": (C.c_int, [_vp, _vp, C.c_int]),
    "zsvd_orthonormality_defect": (C.c_int, [_vp, _sz, _sz, _sz, C.c_int, _dp]),
    "zsvd_factors_defect": (C.c_int, [_vp, _dp, _dp]),
    "zsvd_refactor": (C.c_int, [_vp, _pp]),
    "zsvd_similar_range_search": (C.c_int, [_vp, _sz, _sz, _sz, _sz, Truncation, _vp, _vp, C.POINTER(C.c_size_t)]),
    "zsvd_csv_read": (C.c_int, [C.c_char_p, CsvOptionsC, C.c_int, _pp]),
    "zsvd_csv_info": (C.c_int, [_vp, _szp, _szp, C.POINTER(C.c_int), _szp]),
    "zsvd_csv_error_message": (C.c_int, [_vp, C.c_char_p, _sz]),
    "zsvd_csv_rows_device": (C.c_int, [_vp, _pp]),
    "zsvd_csv_rows_copy": (C.c_int, [_vp, _sz, _sz, _vp]),
    "zsvd_csv_release": (C.c_int, [_vp]),
    "zsvd_store_append_csv": (C.c_int, [_vp, _vp, _szp]),
    "zsvd_last_error_line": (C.c_size_t, []),
    "zsvd_factors_shape": (C.c_int, [_vp, _szp, _szp, _szp]),
    "zsvd_factors_copy": (C.c_int, [_vp, _vp, _vp, _vp]),
    "zsvd_factors_device": (C.c_int, [_vp, _pp, _pp, _pp, _pp]),
    "zsvd_factors_release": (C.c_int, [_vp]),
    "zsvd_factors_upload": (C.c_int, [_vp, _vp, _vp, _sz, _sz, _sz, _pp]),
    "zsvd_thin_svd": (C.c_int, [_vp, _sz, _sz, C.c_int, _pp]),
    "zsvd_truncate": (C.c_int, [_vp, Truncation, _pp]),
    "zsvd_canonical_sign": (C.c_int, [_vp, _pp]),
    "zsvd_trim_block": (C.c_int, [_vp, _sz, _sz, Truncation, _pp]),
    "zsvd_stitch": (C.c_int, [_pp, _sz, Truncation, _pp]),
    "zsvd_device_alloc": (C.c_int, [_sz, C.c_int, _pp]),
    "zsvd_device_free": (C.c_int, [_vp]),
    "zsvd_host_alloc": (C.c_int, [_sz, _pp]),
    "zsvd_host_free": (C.c_int, [_vp]),
    "zsvd_memcpy": (C.c_int, [_vp, _vp, _sz, _vp]),
    "zsvd_stream_sync": (C.c_int, [_vp]),
    "zsvd_event_create": (C.c_int, [_pp]),
    "zsvd_event_destroy": (C.c_int, [_vp]),
    "zsvd_event_record": (C.c_int, [_vp, _vp]),
    "zsvd_event_elapsed_ms": (C.c_int, [_vp, _vp, C.POINTER(C.c_float)]),
}

_lib = None


def lib() -> C.CDLL:
    """Loads libzsvd.so; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(the CUDA extension is required; there is no CPU path)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
