"""B200-native Zoom-SVD storage/query hot path (drop-in for rangesvd's
BlockStore / range_query path).  See DESIGN.md.

The numerical work lives in libzsvd.so (CUDA, sm_100a); this package is the
host-side mirror of the reference API over its C ABI (include/zsvd.h).
"""
from .api import (BlockStore, CorruptionError, CsvOptions, CsvReader, ParseError, SchemaError, ingest_csv,
                  read_csv_matrix, read_csv_rows, CudaError, DeviceFactors, Error, FormatError, InvalidInputError, IoError,
                  InvalidParameterError, LogicError, RangeError, RangeSvd, SearchHit, StoreSnapshot,
                  SvdFactors, TimeRange, Truncation, UnsupportedError, canonical_sign, device_count, direct_count, fallback_count,
                  launch_count, load_store, naive_range_svd, range_query, reconstruction_error, save_store,
                  similar_range_search, stitch, store_from_parts, thin_svd, trim_block, truncate_rank)

__all__ = [
    "BlockStore", "StoreSnapshot", "SvdFactors", "DeviceFactors", "RangeSvd", "TimeRange",
    "Truncation", "range_query", "similar_range_search", "SearchHit", "trim_block", "stitch", "thin_svd",
    "truncate_rank",
    "canonical_sign", "launch_count", "device_count", "fallback_count", "direct_count", "Error", "InvalidInputError",
    "InvalidParameterError", "RangeError", "LogicError", "CudaError", "UnsupportedError", "IoError",
    "FormatError", "CorruptionError", "save_store", "load_store", "naive_range_svd", "reconstruction_error",
    "CsvOptions", "CsvReader", "read_csv_rows", "read_csv_matrix", "ingest_csv", "ParseError", "SchemaError",
    "store_from_parts",
]
