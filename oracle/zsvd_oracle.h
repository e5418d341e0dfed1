/*
 * zsvd_oracle.h — CPU restatement of the Zoom-SVD reference (rangesvd) hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1805_00754_b200/)
 * links, loads or calls this library; only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs use it, and only as the
 * checker / the timed CPU arm.
 *
 * The reference (/root/reference/proj, header-only C++20 over Eigen3) cannot be
 * compiled in this image (Eigen3, GoogleTest and CLI11 are absent), so this is
 * a restatement of its semantics in plain C, function by function:
 *
 *   zo_thin_svd            svd.hpp:90-131   (rank cutoff 1e-12*sigma_max, sigma>0)
 *   zo_truncate (ENERGY)   svd.hpp:135-164  (sequential cumulative energy, early break)
 *   zo_truncate (FIXED)    SURVEY App.A #1  (min(k, numerical rank), same three sites)
 *   zo_reconstruct         svd.hpp:167-174
 *   zo_canonical_sign      svd.hpp:179-203  (first strict argmax |V(:,j)|)
 *   zo_orthonormality_defect svd.hpp:48-58
 *   store (incremental)    store.hpp:55-57 open_block_from_row, :63-97 incremental_update,
 *                          :102-127 reorthonormalize, :182-198 append, :234-240 seal
 *   store (direct)         SURVEY App.A #2: thin_svd of the raw block on fill
 *   zo_resolve             query.hpp:34-51
 *   zo_trim_block          query.hpp:64-89
 *   zo_stitch              query.hpp:95-157
 *   zo_range_query         query.hpp:163-191
 *
 * Eigen's JacobiSVD/BDCSVD are replaced by Householder QR + one-sided (Hestenes)
 * Jacobi on R, which meets the same contract (SPEC.md core-linalg "SVD backend:
 * any numerically stable bidiagonalization or one-sided Jacobi routine").
 *
 * Matrices are row-major double, like rangesvd::DenseMatrix (matrix.hpp:19-133).
 */
#ifndef ZSVD_ORACLE_H
#define ZSVD_ORACLE_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes, one per reference exception type (errors.hpp:9-68) */
enum {
    ZO_OK = 0,
    ZO_INVALID_INPUT = 1,     /* InvalidInputError */
    ZO_INVALID_PARAMETER = 2, /* InvalidParameterError */
    ZO_RANGE_ERROR = 3,       /* RangeError */
    ZO_LOGIC_ERROR = 4,       /* std::logic_error */
    ZO_NO_MEMORY = 5
};

/* truncation policy: ENERGY(xi) is the reference's truncate_rank; FIXED_RANK(k)
 * is the BASELINE configs' fixed k (SURVEY App.A #1). */
enum { ZO_ENERGY = 0, ZO_FIXED_RANK = 1 };

/* store mode: INCREMENTAL follows store.hpp row by row; DIRECT decomposes
 * each full block once (the GPU design). */
enum { ZO_INCREMENTAL = 0, ZO_DIRECT = 1 };

typedef struct {
    size_t m, n, k; /* U is m x k, V is n x k, both row-major */
    double* u;
    double* s;
    double* v;
} zo_factors;

typedef struct {
    size_t first_row, last_row, start_block, end_block;
    size_t skip_front, keep_front, keep_back, skip_back;
} zo_range;

void zo_factors_free(zo_factors* f);
int zo_factors_copy(const zo_factors* in, zo_factors* out);

int zo_thin_svd(const double* a, size_t m, size_t n, zo_factors* out);
int zo_truncate(const zo_factors* in, int policy, double xi, size_t k, zo_factors* out);
void zo_canonical_sign(zo_factors* f);
int zo_reconstruct(const zo_factors* f, double* out);
/* returns -1 for a wide matrix (the reference throws InvalidInputError) */
double zo_orthonormality_defect(const double* m, size_t rows, size_t cols);

int zo_trim_block(const zo_factors* block, size_t keep_from, size_t keep_to, int policy, double xi,
                  size_t k, zo_factors* out);
int zo_stitch(const zo_factors* parts, size_t nparts, int policy, double xi, size_t k,
              zo_factors* out);

typedef struct zo_store zo_store;
zo_store* zo_store_create(size_t b, size_t c, int policy, double xi, size_t k, int mode,
                          int* status);
void zo_store_destroy(zo_store* s);
/* appends rows one at a time exactly like BlockStore::append; stops at the
 * first rejected row (rows before it stay appended, as in the reference). */
int zo_store_append(zo_store* s, const double* rows, size_t nrows);
size_t zo_store_total_rows(const zo_store* s);
size_t zo_store_sealed_count(const zo_store* s);
/* rows in the open block, 0 if none */
size_t zo_store_open_rows(const zo_store* s);
/* copies block i's factors: i < sealed -> sealed block; i == sealed -> open block */
int zo_store_block(zo_store* s, size_t i, zo_factors* out);
/* open-block incremental internals for the store_test KATs (store.hpp:55-127) */
int zo_open_block_from_row(const double* row, size_t c, zo_factors* out);
int zo_incremental_update(const zo_factors* blk, size_t rows_seen, const double* row,
                          size_t capacity, zo_factors* out);
int zo_reorthonormalize(const zo_factors* blk, zo_factors* out);

int zo_resolve(const zo_store* s, size_t first, size_t last, zo_range* out);
int zo_range_query(zo_store* s, size_t first, size_t last, int policy, double xi, size_t k,
                   zo_factors* out);

/* select the thin_svd backend: 0 = built-in QR + one-sided Jacobi (default),
 * 1 = LAPACK dgesdd through a dlopen'ed OpenBLAS (only for CPU timing). */
int zo_set_backend(int backend, const char* lapack_path);

#ifdef __cplusplus
}
#endif
#endif
