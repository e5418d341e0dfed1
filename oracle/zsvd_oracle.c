/*
 * zsvd_oracle.c — CPU restatement of the rangesvd hot path (see zsvd_oracle.h).
 * TEST INFRASTRUCTURE ONLY: the checker for the CUDA product path and the
 * timed CPU arm of bench.py.  Never linked into the product.
 *
 * Every function cites the reference file:line it restates.
 */
#include "zsvd_oracle.h"

#include <dlfcn.h>
#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define CUTOFF 1e-12       /* kNumericalRankCutoff, svd.hpp:22 */
#define ORTHO_TOL 1e-10    /* kOrthonormalityTol,   svd.hpp:25 */
#define REORTH_CADENCE 64  /* kReorthCadence,       store.hpp:23 */

/* ------------------------------------------------------------------ utils */

static double* dalloc(size_t n) {
    return (double*)calloc(n ? n : 1, sizeof(double));
}

void zo_factors_free(zo_factors* f) {
    if (!f) return;
    free(f->u);
    free(f->s);
    free(f->v);
    f->u = f->s = f->v = NULL;
    f->k = 0;
}

static int factors_alloc(zo_factors* f, size_t m, size_t n, size_t k) {
    f->m = m;
    f->n = n;
    f->k = k;
    f->u = dalloc(m * k);
    f->s = dalloc(k);
    f->v = dalloc(n * k);
    if (!f->u || !f->s || !f->v) {
        zo_factors_free(f);
        return ZO_NO_MEMORY;
    }
    return ZO_OK;
}

/* make_empty_factors, svd.hpp:42-44 */
static int factors_empty(zo_factors* f, size_t m, size_t n) { return factors_alloc(f, m, n, 0); }

int zo_factors_copy(const zo_factors* in, zo_factors* out) {
    int st = factors_alloc(out, in->m, in->n, in->k);
    if (st) return st;
    memcpy(out->u, in->u, in->m * in->k * sizeof(double));
    memcpy(out->s, in->s, in->k * sizeof(double));
    memcpy(out->v, in->v, in->n * in->k * sizeof(double));
    return ZO_OK;
}

static int all_finite(const double* a, size_t n) {
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(a[i])) return 0;
    return 1;
}

/* ------------------------------------------------- Householder QR (col-major) */

/* In-place QR of the m x n (m >= n) column-major matrix A (lda = m).  On exit
 * the upper triangle holds R and the strict lower part the Householder vectors
 * (v_j(j) = 1 implicit), tau[j] their scalars.  Restates the role of
 * Eigen::HouseholderQR (store.hpp:108-114). */
static void house_qr(double* A, size_t m, size_t n, double* tau) {
    for (size_t j = 0; j < n; ++j) {
        double* x = A + j * m + j;
        size_t len = m - j;
        double alpha = x[0];
        double sig = 0.0;
        for (size_t i = 1; i < len; ++i) sig += x[i] * x[i];
        if (sig == 0.0) {
            tau[j] = 0.0;
            continue;
        }
        double nrm = sqrt(alpha * alpha + sig);
        double beta = alpha <= 0.0 ? nrm : -nrm;
        tau[j] = (beta - alpha) / beta;
        double scale = 1.0 / (alpha - beta);
        for (size_t i = 1; i < len; ++i) x[i] *= scale;
        x[0] = beta;
        /* apply H = I - tau v v^T to the trailing columns */
        for (size_t c = j + 1; c < n; ++c) {
            double* y = A + c * m + j;
            double w = y[0];
            for (size_t i = 1; i < len; ++i) w += x[i] * y[i];
            w *= tau[j];
            y[0] -= w;
            for (size_t i = 1; i < len; ++i) y[i] -= w * x[i];
        }
    }
}

/* B (m x p col-major, ldb = m) := Q * B, Q from house_qr's reflectors. */
static void house_apply_q(const double* A, size_t m, size_t n, const double* tau, double* B,
                          size_t p) {
    for (size_t jj = n; jj-- > 0;) {
        if (tau[jj] == 0.0) continue;
        const double* x = A + jj * m + jj;
        size_t len = m - jj;
        for (size_t c = 0; c < p; ++c) {
            double* y = B + c * m + jj;
            double w = y[0];
            for (size_t i = 1; i < len; ++i) w += x[i] * y[i];
            w *= tau[jj];
            y[0] -= w;
            for (size_t i = 1; i < len; ++i) y[i] -= w * x[i];
        }
    }
}

/* --------------------------------------------- one-sided Jacobi (Hestenes) */

static double dot(const double* a, const double* b, size_t n) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* Orthogonalises the n columns of W (p x n col-major) by plane rotations,
 * accumulating them in V (n x n col-major, starts at I).  Cyclic by rows,
 * convergence when every pair's cosine is below p*eps. */
static void jacobi(double* W, size_t p, size_t n, double* V) {
    memset(V, 0, n * n * sizeof(double));
    for (size_t i = 0; i < n; ++i) V[i * n + i] = 1.0;
    const double tol = (double)(p > 1 ? p : 1) * DBL_EPSILON;
    for (int sweep = 0; sweep < 80; ++sweep) {
        int rotated = 0;
        for (size_t i = 0; i + 1 < n; ++i) {
            for (size_t j = i + 1; j < n; ++j) {
                double* wi = W + i * p;
                double* wj = W + j * p;
                double alpha = dot(wi, wi, p);
                double beta = dot(wj, wj, p);
                double gamma = dot(wi, wj, p);
                if (alpha == 0.0 || beta == 0.0) continue;
                if (fabs(gamma) <= tol * sqrt(alpha) * sqrt(beta)) continue;
                rotated = 1;
                double zeta = (beta - alpha) / (2.0 * gamma);
                double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                double c = 1.0 / sqrt(1.0 + t * t);
                double s = c * t;
                for (size_t r = 0; r < p; ++r) {
                    double x = wi[r], y = wj[r];
                    wi[r] = c * x - s * y;
                    wj[r] = s * x + c * y;
                }
                double* vi = V + i * n;
                double* vj = V + j * n;
                for (size_t r = 0; r < n; ++r) {
                    double x = vi[r], y = vj[r];
                    vi[r] = c * x - s * y;
                    vj[r] = s * x + c * y;
                }
            }
        }
        if (!rotated) break;
    }
}

/* ----------------------------------------------------- LAPACK (optional) */

typedef void (*dgesdd_fn)(const char*, const int*, const int*, double*, const int*, double*,
                          double*, const int*, double*, const int*, double*, const int*, int*,
                          int*);
static dgesdd_fn g_dgesdd = NULL;
static int g_backend = 0;

int zo_set_backend(int backend, const char* lapack_path) {
    if (backend == 0) {
        g_backend = 0;
        return ZO_OK;
    }
    if (!g_dgesdd) {
        void* h = dlopen(lapack_path, RTLD_NOW | RTLD_LOCAL);
        if (!h) return ZO_INVALID_PARAMETER;
        g_dgesdd = (dgesdd_fn)dlsym(h, "scipy_dgesdd_");
        if (!g_dgesdd) g_dgesdd = (dgesdd_fn)dlsym(h, "dgesdd_");
        void (*set_threads)(int) = (void (*)(int))dlsym(h, "scipy_openblas_set_num_threads");
        if (!set_threads) set_threads = (void (*)(int))dlsym(h, "openblas_set_num_threads");
        if (set_threads) set_threads(1);
        if (!g_dgesdd) return ZO_INVALID_PARAMETER;
    }
    g_backend = 1;
    return ZO_OK;
}

/* Full SVD core: fills U (m x r row-major), s (r), V (n x r row-major), r = min(m,n),
 * sorted non-increasing. */
static int svd_core_lapack(const double* a, size_t m, size_t n, double* U, double* s, double* V) {
    /* a row-major m x n == column-major a^T (n x m). */
    int M = (int)n, N = (int)m, r = (int)(m < n ? m : n);
    double* A = dalloc(m * n);
    double* Up = dalloc((size_t)M * r);
    double* VT = dalloc((size_t)r * N);
    int* iwork = (int*)malloc(sizeof(int) * 8 * (size_t)r);
    memcpy(A, a, m * n * sizeof(double));
    int lwork = -1, info = 0, ldu = M, ldvt = r;
    double wq;
    g_dgesdd("S", &M, &N, A, &M, s, Up, &ldu, VT, &ldvt, &wq, &lwork, iwork, &info);
    lwork = (int)wq + 1;
    double* work = dalloc((size_t)lwork);
    g_dgesdd("S", &M, &N, A, &M, s, Up, &ldu, VT, &ldvt, work, &lwork, iwork, &info);
    /* A^T = Up S VT  =>  A = VT^T S Up^T : U_A (m x r) row-major == VT col-major */
    memcpy(U, VT, (size_t)r * m * sizeof(double));
    for (size_t i = 0; i < n; ++i)
        for (int j = 0; j < r; ++j) V[i * r + j] = Up[i + (size_t)j * M];
    free(A);
    free(Up);
    free(VT);
    free(iwork);
    free(work);
    return info == 0 ? ZO_OK : ZO_INVALID_INPUT;
}

/* Tall (m >= n) core by Householder QR + one-sided Jacobi on R. */
static int svd_core_tall(const double* a, size_t m, size_t n, double* U, double* s, double* V) {
    double* A = dalloc(m * n);
    double* tau = dalloc(n);
    double* R = dalloc(n * n);
    double* Vr = dalloc(n * n);
    size_t* ord = (size_t*)malloc(sizeof(size_t) * n);
    double* B = dalloc(m * n);
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j) A[j * m + i] = a[i * n + j];
    house_qr(A, m, n, tau);
    for (size_t j = 0; j < n; ++j)
        for (size_t i = 0; i <= j; ++i) R[j * n + i] = A[j * m + i];
    jacobi(R, n, n, Vr);
    for (size_t j = 0; j < n; ++j) {
        s[j] = sqrt(dot(R + j * n, R + j * n, n));
        ord[j] = j;
    }
    /* stable sort by sigma descending */
    for (size_t i = 1; i < n; ++i) {
        size_t x = ord[i];
        size_t j = i;
        while (j > 0 && s[ord[j - 1]] < s[x]) {
            ord[j] = ord[j - 1];
            --j;
        }
        ord[j] = x;
    }
    double* sv = dalloc(n);
    for (size_t j = 0; j < n; ++j) sv[j] = s[ord[j]];
    /* B = [U_R ; 0] (m x n col-major), U_R(:,j) = w_j / sigma_j */
    for (size_t j = 0; j < n; ++j) {
        size_t src = ord[j];
        double sg = sv[j];
        for (size_t i = 0; i < n; ++i) B[j * m + i] = sg > 0.0 ? R[src * n + i] / sg : 0.0;
        for (size_t r = 0; r < n; ++r) V[r * n + j] = Vr[src * n + r];
    }
    house_apply_q(A, m, n, tau, B, n);
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j) U[i * n + j] = B[j * m + i];
    memcpy(s, sv, n * sizeof(double));
    free(sv);
    free(A);
    free(tau);
    free(R);
    free(Vr);
    free(ord);
    free(B);
    return ZO_OK;
}

/* thin_svd, svd.hpp:90-131: full decomposition, then keep sigma_i while
 * sigma_i > 0 and sigma_i >= 1e-12 * sigma_max. */
int zo_thin_svd(const double* a, size_t m, size_t n, zo_factors* out) {
    memset(out, 0, sizeof(*out));
    if (m < 1 || n < 1) return ZO_INVALID_INPUT;           /* svd.hpp:91-93 */
    if (!all_finite(a, m * n)) return ZO_INVALID_INPUT;    /* svd.hpp:94-96 */
    size_t r = m < n ? m : n;
    double* U = dalloc(m * r);
    double* V = dalloc(n * r);
    double* s = dalloc(r);
    int st;
    if (g_backend == 1 && g_dgesdd) {
        st = svd_core_lapack(a, m, n, U, s, V);
    } else if (m >= n) {
        st = svd_core_tall(a, m, n, U, s, V);
    } else {
        double* at = dalloc(m * n);
        for (size_t i = 0; i < m; ++i)
            for (size_t j = 0; j < n; ++j) at[j * m + i] = a[i * n + j];
        /* a^T = U' S V'^T  =>  a = V' S U'^T */
        st = svd_core_tall(at, n, m, V, s, U);
        free(at);
    }
    if (st) {
        free(U);
        free(V);
        free(s);
        return st;
    }
    double cutoff = CUTOFF * (r > 0 ? s[0] : 0.0);
    size_t k = 0;
    while (k < r && s[k] > 0.0 && s[k] >= cutoff) ++k;     /* svd.hpp:118-124 */
    st = factors_alloc(out, m, n, k);
    if (!st) {
        for (size_t i = 0; i < m; ++i)
            for (size_t j = 0; j < k; ++j) out->u[i * k + j] = U[i * r + j];
        for (size_t i = 0; i < n; ++i)
            for (size_t j = 0; j < k; ++j) out->v[i * k + j] = V[i * r + j];
        memcpy(out->s, s, k * sizeof(double));
        if (!all_finite(out->u, m * k) || !all_finite(out->v, n * k)) st = ZO_INVALID_INPUT;
    }
    free(U);
    free(V);
    free(s);
    return st;
}

/* leading-column copy (DenseMatrix::left_cols, matrix.hpp:109-117) */
static int keep_leading(const zo_factors* in, size_t keep, zo_factors* out) {
    int st = factors_alloc(out, in->m, in->n, keep);
    if (st) return st;
    for (size_t i = 0; i < in->m; ++i)
        for (size_t j = 0; j < keep; ++j) out->u[i * keep + j] = in->u[i * in->k + j];
    for (size_t i = 0; i < in->n; ++i)
        for (size_t j = 0; j < keep; ++j) out->v[i * keep + j] = in->v[i * in->k + j];
    memcpy(out->s, in->s, keep * sizeof(double));
    return ZO_OK;
}

static int policy_ok(int policy, double xi, size_t k) {
    if (policy == ZO_ENERGY) return (xi > 0.0) && xi <= 1.0;
    if (policy == ZO_FIXED_RANK) return k >= 1;
    return 0;
}

/* truncate_rank, svd.hpp:135-164 (ENERGY); FIXED_RANK keeps min(k, r). */
int zo_truncate(const zo_factors* in, int policy, double xi, size_t k, zo_factors* out) {
    memset(out, 0, sizeof(*out));
    if (!policy_ok(policy, xi, k)) return ZO_INVALID_PARAMETER;   /* svd.hpp:136-138 */
    size_t r = in->k;
    if (policy == ZO_FIXED_RANK) return keep_leading(in, k < r ? k : r, out);
    double total = 0.0;
    for (size_t i = 0; i < r; ++i) total += in->s[i] * in->s[i];
    if (total == 0.0) return factors_empty(out, in->m, in->n);     /* svd.hpp:144-146 */
    size_t keep = r;
    double cum = 0.0;
    for (size_t i = 0; i < r; ++i) {
        cum += in->s[i] * in->s[i];
        if (cum / total >= xi) {
            keep = i + 1;
            break;
        }
    }
    return keep_leading(in, keep, out);
}

/* canonical_sign, svd.hpp:179-203 */
void zo_canonical_sign(zo_factors* f) {
    for (size_t j = 0; j < f->k; ++j) {
        size_t pivot = 0;
        double best = -1.0;
        for (size_t i = 0; i < f->n; ++i) {
            double mag = fabs(f->v[i * f->k + j]);
            if (mag > best) {
                best = mag;
                pivot = i;
            }
        }
        if (f->n > 0 && f->v[pivot * f->k + j] < 0.0) {
            for (size_t i = 0; i < f->n; ++i) f->v[i * f->k + j] = -f->v[i * f->k + j];
            for (size_t i = 0; i < f->m; ++i) f->u[i * f->k + j] = -f->u[i * f->k + j];
        }
    }
}

/* reconstruct, svd.hpp:167-174 */
int zo_reconstruct(const zo_factors* f, double* out) {
    for (size_t i = 0; i < f->m; ++i)
        for (size_t j = 0; j < f->n; ++j) {
            double acc = 0.0;
            for (size_t t = 0; t < f->k; ++t) acc += f->u[i * f->k + t] * f->s[t] * f->v[j * f->k + t];
            out[i * f->n + j] = acc;
        }
    return ZO_OK;
}

/* orthonormality_defect, svd.hpp:48-58 */
double zo_orthonormality_defect(const double* m, size_t rows, size_t cols) {
    if (rows < cols) return -1.0;
    double worst = 0.0;
    for (size_t a = 0; a < cols; ++a)
        for (size_t b = 0; b < cols; ++b) {
            double g = 0.0;
            for (size_t i = 0; i < rows; ++i) g += m[i * cols + a] * m[i * cols + b];
            if (a == b) g -= 1.0;
            if (fabs(g) > worst) worst = fabs(g);
        }
    return worst;
}

/* ---------------------------------------------------------- storage phase */

/* open_block_from_row, store.hpp:55-57 */
int zo_open_block_from_row(const double* row, size_t c, zo_factors* out) {
    return zo_thin_svd(row, 1, c, out);
}

/* incremental_update, store.hpp:63-97 */
int zo_incremental_update(const zo_factors* blk, size_t rows_seen, const double* row,
                          size_t capacity, zo_factors* out) {
    memset(out, 0, sizeof(*out));
    if (rows_seen >= capacity) return ZO_LOGIC_ERROR;             /* store.hpp:65-67 */
    size_t c = blk->n, k = blk->k;
    if (!all_finite(row, c)) return ZO_INVALID_INPUT;
    double* stacked = dalloc((k + 1) * c);
    for (size_t i = 0; i < k; ++i)
        for (size_t j = 0; j < c; ++j) stacked[i * c + j] = blk->s[i] * blk->v[j * k + i];
    memcpy(stacked + k * c, row, c * sizeof(double));
    zo_factors inner;
    int st = zo_thin_svd(stacked, k + 1, c, &inner);
    free(stacked);
    if (st) return st;
    size_t kn = inner.k;
    st = factors_alloc(out, rows_seen + 1, c, kn);
    if (st) {
        zo_factors_free(&inner);
        return st;
    }
    if (kn > 0) {
        /* top rows: U * U_inner[0:k, :] ; last row: U_inner[k, :] (store.hpp:87-93) */
        for (size_t r = 0; r < rows_seen; ++r)
            for (size_t j = 0; j < kn; ++j) {
                double acc = 0.0;
                for (size_t t = 0; t < k; ++t) acc += blk->u[r * k + t] * inner.u[t * kn + j];
                out->u[r * kn + j] = acc;
            }
        for (size_t j = 0; j < kn; ++j) out->u[rows_seen * kn + j] = inner.u[k * kn + j];
    }
    memcpy(out->s, inner.s, kn * sizeof(double));
    memcpy(out->v, inner.v, c * kn * sizeof(double));
    zo_factors_free(&inner);
    return ZO_OK;
}

/* reorthonormalize, store.hpp:102-127 */
int zo_reorthonormalize(const zo_factors* blk, zo_factors* out) {
    size_t k = blk->k, m = blk->m, c = blk->n;
    if (k == 0 || zo_orthonormality_defect(blk->u, m, k) <= ORTHO_TOL) return zo_factors_copy(blk, out);
    double* A = dalloc(m * k);
    double* tau = dalloc(k);
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < k; ++j) A[j * m + i] = blk->u[i * k + j];
    house_qr(A, m, k, tau);
    /* absorbed = R * diag(sigma) * V^T  (k x c) */
    double* absorbed = dalloc(k * c);
    for (size_t i = 0; i < k; ++i)
        for (size_t j = 0; j < c; ++j) {
            double acc = 0.0;
            for (size_t t = i; t < k; ++t) acc += A[t * m + i] * blk->s[t] * blk->v[j * k + t];
            absorbed[i * c + j] = acc;
        }
    zo_factors inner;
    int st = zo_thin_svd(absorbed, k, c, &inner);
    free(absorbed);
    if (st) {
        free(A);
        free(tau);
        return st;
    }
    size_t kn = inner.k;
    /* U = Q * U_inner: Q (m x k thin) applied to [U_inner ; 0] */
    double* B = dalloc(m * kn);
    for (size_t j = 0; j < kn; ++j)
        for (size_t i = 0; i < k; ++i) B[j * m + i] = inner.u[i * kn + j];
    house_apply_q(A, m, k, tau, B, kn);
    st = factors_alloc(out, m, c, kn);
    if (!st) {
        for (size_t i = 0; i < m; ++i)
            for (size_t j = 0; j < kn; ++j) out->u[i * kn + j] = B[j * m + i];
        memcpy(out->s, inner.s, kn * sizeof(double));
        memcpy(out->v, inner.v, c * kn * sizeof(double));
    }
    zo_factors_free(&inner);
    free(B);
    free(A);
    free(tau);
    return st;
}

struct zo_store {
    size_t b, c, kf;
    double xi;
    int policy, mode;
    size_t total_rows;
    size_t nsealed, cap;
    zo_factors* sealed;
    /* open block */
    int has_open;
    size_t rows_seen;
    size_t updates_since_reorth;
    zo_factors open;     /* incremental mode: running factors */
    double* open_raw;    /* direct mode: raw rows (b x c) */
    int open_cached;     /* direct mode: open factors valid */
};

/* BlockStore ctor, store.hpp:163-171 */
zo_store* zo_store_create(size_t b, size_t c, int policy, double xi, size_t k, int mode,
                          int* status) {
    *status = ZO_OK;
    if (b < 1 || c < 1 || !policy_ok(policy, xi, k)) {
        *status = ZO_INVALID_PARAMETER;
        return NULL;
    }
    zo_store* s = (zo_store*)calloc(1, sizeof(zo_store));
    s->b = b;
    s->c = c;
    s->kf = k;
    s->xi = xi;
    s->policy = policy;
    s->mode = mode;
    if (mode == ZO_DIRECT) s->open_raw = dalloc(b * c);
    return s;
}

void zo_store_destroy(zo_store* s) {
    if (!s) return;
    for (size_t i = 0; i < s->nsealed; ++i) zo_factors_free(&s->sealed[i]);
    free(s->sealed);
    zo_factors_free(&s->open);
    free(s->open_raw);
    free(s);
}

static int push_sealed(zo_store* s, zo_factors* f) {
    if (s->nsealed == s->cap) {
        size_t nc = s->cap ? 2 * s->cap : 16;
        zo_factors* p = (zo_factors*)realloc(s->sealed, nc * sizeof(zo_factors));
        if (!p) return ZO_NO_MEMORY;
        s->sealed = p;
        s->cap = nc;
    }
    s->sealed[s->nsealed++] = *f;
    return ZO_OK;
}

/* seal_open_block, store.hpp:234-240: reorth -> truncate -> canonical_sign */
static int seal(zo_store* s) {
    zo_factors base, kept;
    int st;
    if (s->mode == ZO_INCREMENTAL) {
        st = zo_reorthonormalize(&s->open, &base);
    } else {
        st = zo_thin_svd(s->open_raw, s->b, s->c, &base);
    }
    if (st) return st;
    st = zo_truncate(&base, s->policy, s->xi, s->kf, &kept);
    zo_factors_free(&base);
    if (st) return st;
    zo_canonical_sign(&kept);
    st = push_sealed(s, &kept);
    zo_factors_free(&s->open);
    s->has_open = 0;
    s->rows_seen = 0;
    s->updates_since_reorth = 0;
    s->open_cached = 0;
    return st;
}

/* BlockStore::append, store.hpp:182-198 (one row) */
static int append_row(zo_store* s, const double* row) {
    if (!all_finite(row, s->c)) return ZO_INVALID_INPUT;       /* check_row, store.hpp:41-50 */
    int st = ZO_OK;
    if (s->mode == ZO_DIRECT) {
        memcpy(s->open_raw + s->rows_seen * s->c, row, s->c * sizeof(double));
        s->has_open = 1;
        s->rows_seen += 1;
        s->open_cached = 0;
        zo_factors_free(&s->open);
    } else if (!s->has_open) {
        st = zo_open_block_from_row(row, s->c, &s->open);
        if (st) return st;
        s->has_open = 1;
        s->rows_seen = 1;
        s->updates_since_reorth = 0;
    } else {
        zo_factors next;
        st = zo_incremental_update(&s->open, s->rows_seen, row, s->b, &next);
        if (st) return st;
        zo_factors_free(&s->open);
        s->open = next;
        s->rows_seen += 1;
        if (++s->updates_since_reorth >= REORTH_CADENCE) {
            zo_factors fixed;
            st = zo_reorthonormalize(&s->open, &fixed);
            if (st) return st;
            zo_factors_free(&s->open);
            s->open = fixed;
            s->updates_since_reorth = 0;
        }
    }
    if (s->rows_seen == s->b) st = seal(s);
    if (st) return st;
    s->total_rows += 1;
    return ZO_OK;
}

int zo_store_append(zo_store* s, const double* rows, size_t nrows) {
    for (size_t i = 0; i < nrows; ++i) {
        int st = append_row(s, rows + i * s->c);
        if (st) return st;
    }
    return ZO_OK;
}

size_t zo_store_total_rows(const zo_store* s) { return s->total_rows; }
size_t zo_store_sealed_count(const zo_store* s) { return s->nsealed; }
size_t zo_store_open_rows(const zo_store* s) { return s->has_open ? s->rows_seen : 0; }

/* block factors: StoreSnapshot::block_factors, store.hpp:150-155.  In direct
 * mode the open factors are the untruncated thin_svd of the raw rows (App.A #3). */
static const zo_factors* block_ref(zo_store* s, size_t i, int* st) {
    *st = ZO_OK;
    if (i < s->nsealed) return &s->sealed[i];
    if (i == s->nsealed && s->has_open) {
        if (s->mode == ZO_DIRECT && !s->open_cached) {
            zo_factors_free(&s->open);
            *st = zo_thin_svd(s->open_raw, s->rows_seen, s->c, &s->open);
            if (*st) return NULL;
            s->open_cached = 1;
        }
        return &s->open;
    }
    *st = ZO_RANGE_ERROR;
    return NULL;
}

int zo_store_block(zo_store* s, size_t i, zo_factors* out) {
    int st;
    const zo_factors* f = block_ref(s, i, &st);
    if (!f) return st;
    return zo_factors_copy(f, out);
}

/* ------------------------------------------------------------ query phase */

/* TimeRange::resolve, query.hpp:34-51 */
int zo_resolve(const zo_store* s, size_t first, size_t last, zo_range* r) {
    if (s->total_rows == 0) return ZO_RANGE_ERROR;
    if (last < first || last >= s->total_rows) return ZO_RANGE_ERROR;
    r->first_row = first;
    r->last_row = last;
    r->start_block = first / s->b;
    r->end_block = last / s->b;
    r->skip_front = first - r->start_block * s->b;
    r->keep_front = s->b - r->skip_front;
    r->keep_back = last - r->end_block * s->b + 1;
    size_t rows_e = r->end_block < s->nsealed ? s->b : s->rows_seen;
    r->skip_back = rows_e - r->keep_back;
    return ZO_OK;
}

/* trim_block, query.hpp:64-89 */
int zo_trim_block(const zo_factors* block, size_t keep_from, size_t keep_to, int policy, double xi,
                  size_t k, zo_factors* out) {
    memset(out, 0, sizeof(*out));
    if (!policy_ok(policy, xi, k)) return ZO_INVALID_PARAMETER;
    if (keep_from > keep_to || keep_to >= block->m) return ZO_INVALID_PARAMETER;
    size_t rows = keep_to - keep_from + 1, kb = block->k, n = block->n;
    if (kb == 0) return factors_empty(out, rows, n);
    double* sliced = dalloc(rows * kb);
    for (size_t i = 0; i < rows; ++i)
        for (size_t j = 0; j < kb; ++j) sliced[i * kb + j] = block->u[(keep_from + i) * kb + j] * block->s[j];
    zo_factors full, inner;
    int st = zo_thin_svd(sliced, rows, kb, &full);
    free(sliced);
    if (st) return st;
    st = zo_truncate(&full, policy, xi, k, &inner);
    zo_factors_free(&full);
    if (st) return st;
    size_t kt = inner.k;
    st = factors_alloc(out, rows, n, kt);
    if (!st) {
        memcpy(out->u, inner.u, rows * kt * sizeof(double));
        memcpy(out->s, inner.s, kt * sizeof(double));
        /* V' = V * V_inner  (n x kb)(kb x kt) */
        for (size_t i = 0; i < n; ++i)
            for (size_t j = 0; j < kt; ++j) {
                double acc = 0.0;
                for (size_t t = 0; t < kb; ++t) acc += block->v[i * kb + t] * inner.v[t * kt + j];
                out->v[i * kt + j] = acc;
            }
    }
    zo_factors_free(&inner);
    return st;
}

/* stitch_parts, query.hpp:95-144 */
static int stitch_refs(const zo_factors* const* parts, size_t np, int policy, double xi, size_t k,
                       zo_factors* out) {
    memset(out, 0, sizeof(*out));
    if (np == 0) return ZO_INVALID_PARAMETER;
    if (!policy_ok(policy, xi, k)) return ZO_INVALID_PARAMETER;
    size_t n = parts[0]->n, total_rank = 0, total_rows = 0;
    for (size_t p = 0; p < np; ++p) {
        if (parts[p]->n != n) return ZO_INVALID_INPUT;
        total_rank += parts[p]->k;
        total_rows += parts[p]->m;
    }
    if (total_rank == 0) return factors_empty(out, total_rows, n);
    double* stacked = dalloc(total_rank * n);
    size_t band = 0;
    for (size_t p = 0; p < np; ++p)
        for (size_t i = 0; i < parts[p]->k; ++i, ++band)
            for (size_t j = 0; j < n; ++j)
                stacked[band * n + j] = parts[p]->s[i] * parts[p]->v[j * parts[p]->k + i];
    zo_factors full, inner;
    int st = zo_thin_svd(stacked, total_rank, n, &full);
    free(stacked);
    if (st) return st;
    st = zo_truncate(&full, policy, xi, k, &inner);
    zo_factors_free(&full);
    if (st) return st;
    size_t ko = inner.k;
    st = factors_alloc(out, total_rows, n, ko);
    if (!st) {
        size_t row_off = 0, rank_off = 0;
        for (size_t p = 0; p < np; ++p) {
            const zo_factors* f = parts[p];
            if (f->k > 0 && ko > 0) {
                for (size_t r = 0; r < f->m; ++r)
                    for (size_t j = 0; j < ko; ++j) {
                        double acc = 0.0;
                        for (size_t t = 0; t < f->k; ++t) acc += f->u[r * f->k + t] * inner.u[(rank_off + t) * ko + j];
                        out->u[(row_off + r) * ko + j] = acc;
                    }
            }
            row_off += f->m;
            rank_off += f->k;
        }
        memcpy(out->s, inner.s, ko * sizeof(double));
        memcpy(out->v, inner.v, n * ko * sizeof(double));
    }
    zo_factors_free(&inner);
    return st;
}

/* stitch, query.hpp:150-157 */
int zo_stitch(const zo_factors* parts, size_t nparts, int policy, double xi, size_t k,
              zo_factors* out) {
    const zo_factors** refs = (const zo_factors**)malloc(sizeof(void*) * (nparts ? nparts : 1));
    for (size_t i = 0; i < nparts; ++i) refs[i] = &parts[i];
    int st = stitch_refs(refs, nparts, policy, xi, k, out);
    free(refs);
    return st;
}

/* range_query, query.hpp:163-191 (+ canonical_sign at :190) */
int zo_range_query(zo_store* s, size_t first, size_t last, int policy, double xi, size_t k,
                   zo_factors* out) {
    memset(out, 0, sizeof(*out));
    if (!policy_ok(policy, xi, k)) return ZO_INVALID_PARAMETER;   /* query.hpp:165-167 */
    zo_range r;
    int st = zo_resolve(s, first, last, &r);
    if (st) return st;
    if (r.start_block == r.end_block) {
        const zo_factors* blk = block_ref(s, r.start_block, &st);
        if (!blk) return st;
        size_t base = r.start_block * s->b;
        st = zo_trim_block(blk, first - base, last - base, policy, xi, k, out);
    } else {
        zo_factors head, tail;
        const zo_factors* bs = block_ref(s, r.start_block, &st);
        if (!bs) return st;
        st = zo_trim_block(bs, r.skip_front, s->b - 1, policy, xi, k, &head);
        if (st) return st;
        const zo_factors* be = block_ref(s, r.end_block, &st);
        if (!be) {
            zo_factors_free(&head);
            return st;
        }
        st = zo_trim_block(be, 0, r.keep_back - 1, policy, xi, k, &tail);
        if (st) {
            zo_factors_free(&head);
            return st;
        }
        size_t np = r.end_block - r.start_block + 1;
        const zo_factors** parts = (const zo_factors**)malloc(sizeof(void*) * np);
        parts[0] = &head;
        for (size_t i = r.start_block + 1; i < r.end_block; ++i) parts[i - r.start_block] = &s->sealed[i];
        parts[np - 1] = &tail;
        st = stitch_refs(parts, np, policy, xi, k, out);
        free(parts);
        zo_factors_free(&head);
        zo_factors_free(&tail);
    }
    if (st) return st;
    zo_canonical_sign(out);
    return ZO_OK;
}
