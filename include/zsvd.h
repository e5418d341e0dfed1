/*
 * zsvd.h — C ABI of the B200-native Zoom-SVD storage/query hot path.
 *
 * This is the drop-in boundary for the reference library rangesvd
 * (/root/reference/proj/include/rangesvd, header-only C++20 over Eigen).  The
 * reference has no FFI of its own: its callers include the headers.  Each
 * entry point below names the reference interface it replaces (file:line);
 * include/zsvd.hpp re-creates that C++ API (BlockStore, StoreSnapshot,
 * range_query, trim_block, stitch, thin_svd, truncate_rank, canonical_sign)
 * on top of these functions, re-throwing the same exception types.
 *
 * Plain pointers and sizes only.  All numerical work runs on the GPU
 * (sm_100a); there is no CPU fallback — with no usable device every call
 * that computes fails with ZSVD_ERR_CUDA.
 *
 * Matrices are row-major fp64, like rangesvd::DenseMatrix (matrix.hpp:19-133).
 */
#ifndef ZSVD_H
#define ZSVD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: one per reference exception type (errors.hpp:9-68), plus the
 * device failures the reference cannot have. */
typedef enum {
    ZSVD_OK = 0,
    ZSVD_ERR_INVALID_INPUT = 1,     /* rangesvd::InvalidInputError     (errors.hpp:16) */
    ZSVD_ERR_INVALID_PARAMETER = 2, /* rangesvd::InvalidParameterError (errors.hpp:22) */
    ZSVD_ERR_RANGE = 3,             /* rangesvd::RangeError            (errors.hpp:28) */
    ZSVD_ERR_LOGIC = 4,             /* std::logic_error                (store.hpp:65-67) */
    ZSVD_ERR_CUDA = 5,              /* device / runtime failure */
    ZSVD_ERR_NO_MEMORY = 6,
    ZSVD_ERR_UNSUPPORTED = 7,       /* shape outside this build's kernels (min(b, c) > 1024) */
    ZSVD_ERR_IO = 8,                /* rangesvd::IoError               (errors.hpp:52) */
    ZSVD_ERR_FORMAT = 9,            /* rangesvd::FormatError           (errors.hpp:58) */
    ZSVD_ERR_CORRUPTION = 10,       /* rangesvd::CorruptionError       (errors.hpp:65) */
    ZSVD_ERR_PARSE = 11,            /* rangesvd::ParseError            (errors.hpp:34), carries a line */
    ZSVD_ERR_SCHEMA = 12            /* rangesvd::SchemaError           (errors.hpp:47) */
} zsvd_status;

/* Truncation policy.  ENERGY(xi) is truncate_rank (svd.hpp:135-164); FIXED_RANK(k)
 * keeps min(k, numerical rank) at the same three sites (seal store.hpp:236,
 * trim query.hpp:83, stitch query.hpp:124) — SURVEY App. A #1. */
typedef enum { ZSVD_POLICY_ENERGY = 0, ZSVD_POLICY_FIXED_RANK = 1 } zsvd_policy;

/* Where a caller-supplied pointer lives. */
typedef enum { ZSVD_MEM_HOST = 0, ZSVD_MEM_DEVICE = 1 } zsvd_memory;

typedef struct {
    int32_t policy; /* zsvd_policy */
    double xi;      /* ENERGY threshold in (0, 1] */
    uint64_t k;     /* FIXED_RANK rank >= 1 */
} zsvd_truncation;

typedef struct zsvd_store zsvd_store;       /* rangesvd::BlockStore    (store.hpp:161-249) */
typedef struct zsvd_snapshot zsvd_snapshot; /* rangesvd::StoreSnapshot (store.hpp:135-156) */
typedef struct zsvd_factors zsvd_factors;   /* rangesvd::SvdFactors    (svd.hpp:30-40), device-resident */

typedef struct {
    uint64_t block_size, num_columns, total_rows, sealed_count, open_rows;
    zsvd_truncation truncation;
    int32_t device;
} zsvd_store_info;

typedef struct { /* rangesvd::TimeRange (query.hpp:19-31) */
    uint64_t first_row, last_row, start_block, end_block;
    uint64_t skip_front, keep_front, keep_back, skip_back;
} zsvd_time_range;

/* ---- library ------------------------------------------------------------ */
const char* zsvd_version(void);
/* Copies the calling thread's last error message; returns its status. */
int zsvd_last_error(char* buf, size_t len);
int zsvd_device_count(int* count);
/* Number of kernels this library has launched in the process (all threads). */
uint64_t zsvd_launch_count(void);
/* Factorisations re-done by the robust fallback path on the current device
 * (ill-conditioned or rank-deficient inputs); waits for the device. */
uint64_t zsvd_fallback_count(void);
/* FIXED_RANK factorisations finished by a direct route on the current device
 * (leading eigenvectors of the Gram, then a k-column one-sided Jacobi: DESIGN
 * 4.1 / 4.1b); diagnostics, waits for the device. */
uint64_t zsvd_direct_count(void);

/* ---- storage phase (store.hpp) ------------------------------------------- */
/* BlockStore(b, c, xi) (store.hpp:163-171): ENERGY policy on device 0. */
int zsvd_store_create(size_t block_size, size_t num_columns, double xi, zsvd_store** out);
/* Same with an explicit policy and CUDA device. */
int zsvd_store_create_ex(size_t block_size, size_t num_columns, zsvd_truncation trunc,
                         int device, zsvd_store** out);
int zsvd_store_destroy(zsvd_store* store);
/* BlockStore::append (store.hpp:182-198), batched: nrows rows of num_columns
 * values, row stride ld (>= num_columns) doubles, host or device memory.  All
 * rows are validated (finite) before any state changes; a rejected call leaves
 * the store untouched.  Full blocks are factorised on the device on fill
 * (batched, possibly deferred until the next snapshot/sync). */
int zsvd_store_append(zsvd_store* store, const double* rows, size_t nrows, size_t ld,
                      int memory);
int zsvd_store_info_get(zsvd_store* store, zsvd_store_info* info);
/* Rank of block i (i < sealed: sealed block; i == sealed: open block, full
 * numerical rank).  Factor download for sealed()/open() (store.hpp:178-179). */
int zsvd_store_block_rank(zsvd_store* store, size_t i, size_t* rank);
/* Host copies: u (rows x k), s (k), v (num_columns x k), rows = block_size for
 * sealed blocks or open_rows for the open one; any pointer may be NULL. */
int zsvd_store_block_copy(zsvd_store* store, size_t i, double* u, double* s, double* v);
/* Waits for all queued storage work. */
int zsvd_store_sync(zsvd_store* store);
/* Drops all blocks (keeps device allocations): the store is empty again. */
int zsvd_store_reset(zsvd_store* store);
/* Singular values of sealed blocks [first, first+count): sigma is count x ld
 * (zero-padded past each block's rank), ranks (count) may be NULL. */
int zsvd_store_spectrum(zsvd_store* store, size_t first, size_t count, double* sigma, size_t ld,
                        uint32_t* ranks);
/* The storage (writer) stream, a cudaStream_t. */
int zsvd_store_stream(zsvd_store* store, void** stream);
/* Kernel-level timing of the storage factorisation kernel (CUDA events around
 * each launch on the storage stream) — enable, then read launches and total
 * device milliseconds.  Used by bench.py for the roofline. */
int zsvd_store_profile(zsvd_store* store, int enable);
int zsvd_store_profile_read(zsvd_store* store, uint64_t* launches, uint64_t* blocks,
                            double* total_ms);

/* ---- snapshots (store.hpp:135-156, 200-203) ------------------------------ */
/* save_store / load_store (serialize.hpp:147-256): the ZSVD v1 file format,
 * little-endian, byte-identical across saves of the same store.  FIXED_RANK
 * stores (no reference counterpart) are written as version 2: the v1 layout with
 * the rank (u64) after the threshold field; the reference reader refuses them
 * with FormatError.  Loading accepts both versions.  A loaded
 * store keeps the file's open-block factors bit for bit until the next append,
 * then continues from the open block's rows (reconstructed as U S V^T).
 * Errors: IO, FORMAT (bad magic / version), CORRUPTION (truncation, counts,
 * ordering, trailing bytes, factor invariants at 1e-8). */
int zsvd_store_save(zsvd_store* store, const char* path);
int zsvd_store_load(const char* path, int device, zsvd_store** out);

/* One block's factors in host memory (compact row-major: u rows x k, s k,
 * v num_columns x k), for BlockStore::from_parts. */
typedef struct {
    uint64_t index;     /* SealedBlock::index / OpenBlock::index */
    uint64_t rows;      /* block_size (sealed) or rows_seen (open) */
    uint64_t k;
    const double* u;
    const double* s;
    const double* v;
} zsvd_block_factors;

/* BlockStore::from_parts (store.hpp:206-231): rebuilds a store from persisted
 * parts.  Indices must run 0..nsealed-1, sealed blocks must be block_size x
 * num_columns, the open block (NULL: none) must have index nsealed and
 * 1 <= rows <= block_size; otherwise INVALID_INPUT.  Parameters as
 * zsvd_store_create_ex.  The open block's factors are kept bit for bit until
 * the next append (like zsvd_store_load). */
int zsvd_store_from_parts(size_t block_size, size_t num_columns, zsvd_truncation trunc, int device,
                          const zsvd_block_factors* sealed, size_t nsealed, const zsvd_block_factors* open,
                          zsvd_store** out);

/* StoreSnapshot snapshot() const: pins the sealed count and factorises the
 * open block (untruncated, numerical-rank cutoff only — store.hpp:59-62). */
int zsvd_snapshot_create(zsvd_store* store, zsvd_snapshot** out);
int zsvd_snapshot_release(zsvd_snapshot* snap);
int zsvd_snapshot_info_get(zsvd_snapshot* snap, zsvd_store_info* info);
/* The snapshot's query stream, a cudaStream_t. */
int zsvd_snapshot_stream(zsvd_snapshot* snap, void** stream);
/* Device copy of block i of the snapshot (sealed, or the open tail at
 * i == sealed_count): StoreSnapshot::block_factors (store.hpp:150-155). */
int zsvd_snapshot_block(zsvd_snapshot* snap, size_t i, zsvd_factors** out);

/* ---- query phase (query.hpp) --------------------------------------------- */
/* TimeRange::resolve (query.hpp:34-51). */
int zsvd_resolve(zsvd_snapshot* snap, size_t first, size_t last, zsvd_time_range* out);
/* range_query(snapshot, first, last, xi) (query.hpp:163-191), generalised to a
 * truncation policy; the answer is sign-canonicalised (query.hpp:190).  The
 * result stays on the device; it is enqueued on the snapshot's stream and this
 * call does not wait for it. */
int zsvd_range_query(zsvd_snapshot* snap, size_t first, size_t last, zsvd_truncation trunc,
                     zsvd_factors** out);

/* similar_range_search (analysis.hpp:78-148): scores every window
 * [w, w + L - 1], w = 0, stride, ..., that ends before the base range
 * [base_first, base_last] (L = its length) by the |cosine| of the leading left
 * singular vectors of range_query(window) and range_query(base); writes the
 * top_n (similarity descending, ties to the earlier window) to starts / sims
 * (capacity top_n) and their count to *nhits.  A rank-0 base gives no hits.
 * Errors: base shorter than 2 rows or stride 0 -> INVALID_PARAMETER; base out
 * of range -> RANGE.  Waits for the result. */
int zsvd_similar_range_search(zsvd_snapshot* snap, size_t base_first, size_t base_last, size_t stride,
                              size_t top_n, zsvd_truncation trunc, uint64_t* starts, double* sims,
                              size_t* nhits);

/* naive_range_svd (analysis.hpp:49-66): the paper's reconstruct-then-SVD
 * baseline — the range's rows are rebuilt from the stored factors on the
 * device and decomposed from scratch (thin_svd semantics). */
int zsvd_naive_range_svd(zsvd_snapshot* snap, size_t first, size_t last, zsvd_factors** out);
/* reconstruction_error (analysis.hpp:20-37): ||X - U S V^T||_F^2 / ||X||_F^2
 * of an m x n matrix (host or device) against factors of the same shape;
 * all-zero data gives 0 against rank-0 factors, +infinity otherwise. */
int zsvd_reconstruction_error(const double* raw, size_t m, size_t n, int memory, zsvd_factors* f,
                              double* err);

/* ---- CSV ingestion (csv.hpp) --------------------------------------------- */
/* CsvOptions (csv.hpp:22-27): expected_cols < 0 means "any". */
typedef struct {
    int64_t expected_cols;
    int32_t drop_timestamp;
} zsvd_csv_options;

typedef struct zsvd_csv zsvd_csv; /* a parsed file: CsvReader's rows, device-resident */

/* Reads and parses a whole CSV file on the device: the text is streamed through
 * pinned host buffers to HBM and tokenised and converted there, bit-exact with
 * std::from_chars (csv.hpp:42-50).  It follows the CsvReader rules (csv.hpp:69-179):
 * blank lines skipped, the first content line skipped if none of its cells is
 * numeric, timestamp column dropped, column count fixed by expected_cols or the
 * first data row.  An unopenable file fails with IO (the CsvReader constructor,
 * csv.hpp:71-76).  A parse or schema error does NOT fail this call: the handle
 * keeps the rows the reader yields before it, and zsvd_csv_info reports it. */
int zsvd_csv_read(const char* path, zsvd_csv_options options, int device, zsvd_csv** out);
/* rows before the error (all rows if none), columns (0 if no data row), the
 * pending error (ZSVD_OK, ZSVD_ERR_PARSE or ZSVD_ERR_SCHEMA) and its 1-based line
 * (ParseError::line; 0 for a schema error).  Any pointer may be NULL. */
int zsvd_csv_info(zsvd_csv* csv, size_t* rows, size_t* cols, int* error, size_t* error_line);
/* The pending error's message, exactly the reference's what() ("line N: ..."). */
int zsvd_csv_error_message(zsvd_csv* csv, char* buf, size_t len);
/* The rows, row-major rows x cols on the device (valid until release). */
int zsvd_csv_rows_device(zsvd_csv* csv, const double** rows);
/* Host copy of rows [first, first + count). */
int zsvd_csv_rows_copy(zsvd_csv* csv, size_t first, size_t count, double* out);
int zsvd_csv_release(zsvd_csv* csv);
/* BlockStore::append of a parsed file's rows straight from HBM (cmd_ingest's
 * append loop, commands.hpp:119-123).  A pending parse/schema error is raised
 * (PARSE / SCHEMA, message in zsvd_last_error) without appending anything:
 * the append is atomic, unlike the reference's row-by-row loop.  *appended may
 * be NULL. */
int zsvd_store_append_csv(zsvd_store* store, zsvd_csv* csv, size_t* appended);
/* The 1-based line of this thread's last ZSVD_ERR_PARSE (0 otherwise). */
size_t zsvd_last_error_line(void);

/* ---- multi-GPU: one process per GPU ------------------------ */
/* An NCCL communicator over the ranks' devices (NCCL is loaded at run time;
 * without it these calls fail with ZSVD_ERR_UNSUPPORTED).  Rank 0 makes the id,
 * the caller hands it to every rank (e.g. a torch.distributed broadcast). */
#define ZSVD_COMM_ID_BYTES 128
typedef struct zsvd_comm zsvd_comm;
int zsvd_comm_unique_id(void* id /* ZSVD_COMM_ID_BYTES */);
int zsvd_comm_create(const void* id, int nranks, int rank, int device, zsvd_comm** out);
int zsvd_comm_destroy(zsvd_comm* comm);
/* range_query (query.hpp:163-191) over a stream sharded by contiguous row
 * ranges: rank r's store holds global rows [r R, r R + its total_rows), R =
 * rows_per_rank a multiple of block_size (storage shards with no collective).
 * Every rank calls it with the same global [first, last] and truncation.  Each
 * rank forms the Gram of its share of the stitched stack on its GPU; the c x c
 * Grams are all-gathered over NCCL and added in rank order, so every rank runs
 * the same stitch SVD and holds the same sigma and V; each rank's result holds
 * the U rows of its own share (m = those rows, possibly 0), *row_offset = their
 * first row within the answer.  A range not covered by the shards -> RANGE on
 * every rank; a range the Gram stitch cannot take (energy truncation, c > 64,
 * a spread retained spectrum) -> UNSUPPORTED on every rank (callers fall back
 * to gathering the parts on one device). */
int zsvd_sharded_range_query(zsvd_snapshot* local, zsvd_comm* comm, uint64_t rows_per_rank, size_t first,
                             size_t last, zsvd_truncation trunc, zsvd_factors** out, uint64_t* row_offset);

/* ---- factors (svd.hpp:30-40) --------------------------------------------- */
/* Shape of a result (waits for it): u is m x k, v is n x k. */
int zsvd_factors_shape(zsvd_factors* f, size_t* m, size_t* n, size_t* k);
/* Host copies (waits); any pointer may be NULL. */
int zsvd_factors_copy(zsvd_factors* f, double* u, double* s, double* v);
/* Device pointers (valid until release; read after the producing stream). */
int zsvd_factors_device(zsvd_factors* f, const double** u, const double** s, const double** v,
                        void** stream);
int zsvd_factors_release(zsvd_factors* f);
/* Uploads host factors (u m x k, s k, v n x k) as a device-resident SvdFactors.
 * m = 0 makes a row-less part (sigma and V only) for sharded stitching: it
 * contributes its bands to the stack but no rows to the stitched U; m < k is
 * accepted for the row-partial answers of a sharded query.  k <= n. */
int zsvd_factors_upload(const double* u, const double* s, const double* v, size_t m, size_t n,
                        size_t k, zsvd_factors** out);

/* reconstruct (svd.hpp:167-174): U diag(sigma) V^T, m x n row-major, written
 * to host or device memory `out` (rank 0 gives zeros).  Waits. */
int zsvd_reconstruct(zsvd_factors* f, double* out, int memory);
/* orthonormality_defect (svd.hpp:48-58): max |M^T M - I| of a rows x cols
 * matrix (row stride ld >= cols), host or device; 0 for cols == 0;
 * rows < cols -> INVALID_INPUT.  Computed on the device; waits. */
int zsvd_orthonormality_defect(const double* m, size_t rows, size_t cols, size_t ld, int memory,
                               double* out);
/* thin_svd of U diag(sigma) V^T rebuilt on the device (numerical-rank cutoff
 * only): reorthonormalize's repair (store.hpp:102-127) of drifted factors. */
int zsvd_refactor(zsvd_factors* f, zsvd_factors** out);
/* Both defects of a device-resident result (either pointer may be NULL). */
int zsvd_factors_defect(zsvd_factors* f, double* defect_u, double* defect_v);

/* ---- L1 primitives: free functions of svd.hpp / query.hpp ---------------- */
/* thin_svd (svd.hpp:90-131): rank cutoff 1e-12*sigma_max, no truncation. */
int zsvd_thin_svd(const double* a, size_t m, size_t n, int memory, zsvd_factors** out);
/* truncate_rank (svd.hpp:135-164) / FIXED_RANK. */
int zsvd_truncate(zsvd_factors* f, zsvd_truncation trunc, zsvd_factors** out);
/* canonical_sign (svd.hpp:179-203). */
int zsvd_canonical_sign(zsvd_factors* f, zsvd_factors** out);
/* trim_block (query.hpp:64-89), rows [keep_from, keep_to]. */
int zsvd_trim_block(zsvd_factors* block, size_t keep_from, size_t keep_to,
                    zsvd_truncation trunc, zsvd_factors** out);
/* stitch (query.hpp:150-157). */
int zsvd_stitch(zsvd_factors* const* parts, size_t nparts, zsvd_truncation trunc,
                zsvd_factors** out);

/* ---- device memory and timing helpers (for HBM-resident inputs) ---------- */
int zsvd_device_alloc(size_t bytes, int device, void** ptr);
int zsvd_device_free(void* ptr);
int zsvd_host_alloc(size_t bytes, void** ptr); /* pinned */
int zsvd_host_free(void* ptr);
int zsvd_memcpy(void* dst, const void* src, size_t bytes, void* stream); /* async on stream, any direction */
int zsvd_stream_sync(void* stream);
int zsvd_event_create(void** ev);
int zsvd_event_destroy(void* ev);
int zsvd_event_record(void* ev, void* stream);
int zsvd_event_elapsed_ms(void* start, void* stop, float* ms); /* waits for stop */

#ifdef __cplusplus
}
#endif
#endif /* ZSVD_H */
