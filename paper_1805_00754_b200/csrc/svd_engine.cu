// svd_engine.cu — batched fp64 thin SVD for sm_100a (one CTA per matrix).
//
// Replaces the Eigen call sites of the reference hot path:
// thin_svd (svd.hpp:90-131: JacobiSVD / BDCSVD + 1e-12 rank cutoff),
// truncate_rank (svd.hpp:135-164), canonical_sign (svd.hpp:179-203), and the
// small products fused around them in trim_block (query.hpp:79-87).
//
// Work matrix W (p x q, p >= q): W = A when m >= n, W = A^T otherwise, q <= 64.
// Fast path: CholeskyQR2 + one-sided Jacobi on R^T, as phase kernels (see the
// v3 section below).  Robust path: one-sided Jacobi on W in global scratch
// (rank-deficient or ill-conditioned inputs, exact zero blocks), re-doing the
// tasks the fast path flags.  All reductions use a fixed order, so results are
// bitwise reproducible.
#include <cfloat>
#include <cstdint>
#include <type_traits>

#include "eigh_warp.cuh"
#include "zsvd_internal.h"

namespace zsvd {

// Tasks re-done by the fallback kernel (diagnostics: zsvd_fallback_count()).
__device__ unsigned long long g_fallback_tasks = 0;
// Factorisations finished by a direct route (eigen phase + k-column Jacobi here,
// wide_eig.cuh on the wide path; diagnostics: zsvd_direct_count()).
__device__ unsigned long long g_direct_tasks = 0;

// One-pass CholeskyQR threshold on the pivots of R1 (min / max).  After one
// pass R1^T R1 equals the Gram up to its rounding (eps ||G||), so the kept
// sigma_j and U are accurate to c eps (sigma_1 / sigma_j)^2 (c <= 0.06 on the
// cfg2 blocks): what matters is the retained spread, which mid-2 checks
// (sigma_1 <= 3000 sigma_k, else the robust path), and the check phase still
// enforces the 1e-10 orthonormality contract.  The pivot spread is the early
// proxy: every cfg1/cfg2/cfg4 block (ratios 6e-3 .. 0.14) takes one pass,
// graded inputs below 3e-3 keep the second pass (P2 + Cholesky of Q1^T Q1).
// Host-settable (ZSVD_TWO_PASS=1 sets 2.0: always two passes).
__device__ double g_onepass_pivot = 3e-3;
// No-solve U formation (mid2_body step 5) when sigma_1 <= ratio * sigma_k;
// host-settable (ZSVD_NOSOLVE_RATIO, 0 disables).
__device__ double g_nosolve_ratio = 1000.0;

namespace {

constexpr int T = kEngineThreads;
constexpr int NWARPS = T / 32;
constexpr int kMaxChunk = 128;

struct Small {
    double sig[kQMax];
    double sgn[kQMax];
    int ord[kQMax];
    int m, n, p, q, tall, k, knum;
    int status;
    int flag;
    int sweeps;
    int reason;
    long long clk[8];
    double pivmin, pivmax;
    // scratch of the bodies, kept here rather than as function-scope
    // __shared__ arrays: under relocatable device code every template
    // instantiation's statics are charged to each kernel, which cost
    // occupancy
    double raw[kQMax];      // sort_and_truncate: column norms
    double inv_sig[kQMax];  // 1 / sigma
    double rinv[kQMax];     // chol3: 1 / R_jj
    double scale;           // mid2: power-of-two scaling of R
    int flags[2];           // jacobi_bisect64: sweep flags
    int bigf[2];            // Jacobi: a rotation of cosine >= kCheckCos this sweep
    int conv;               // gram_converged result
    int onepass;            // mid-1 decision (SvdTask::onepass)
    int roff[kQMax];        // mid2: row starts of the packed R
};

// 1 / sqrt(x) for a normal positive x: the MUFU seed (2^-20, measured) and one
// third-order correction y (1 + e/2 + 3e^2/8), e = 1 - x y^2: four dependent
// operations, <= 1 ulp over 6.7e7 samples (scripts/dev/rsqrt_check.cu; two
// Newton steps: six operations, 1.4 ulp).  Inline: the library rsqrt calls a
// slow-path subroutine on the Jacobi and Cholesky critical paths.
__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x * y, y, 1.0);
    return fma(y * e, fma(0.375, e, 0.5), y);
}

__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double a_at(const SvdTask& t, int i, int j) {
    double x = t.a[(int64_t)i * t.lda + j];
    return t.colscale ? x * t.colscale[j] : x;
}

// W(i, j) for the work matrix.
__device__ __forceinline__ double w_at(const SvdTask& t, bool tall, int i, int j) {
    return tall ? a_at(t, i, j) : a_at(t, j, i);
}

// ---------------------------------------------------------------- Jacobi
// One-sided Jacobi on W (p x q, column-major, ld p), V (q x q, col-major, ld q).
// Round-robin (circle method) ordering: q' - 1 rounds of q'/2 disjoint pairs per
// sweep; one warp per pair; convergence when a whole sweep rotates nothing.
__device__ void jacobi(double* W, int ldw, int p, int q, double* V, Small& sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < q * q; i += T) V[i] = (i % (q + 1) == 0) ? 1.0 : 0.0;
    const int qe = q + (q & 1);
    const int npairs = qe / 2;
    const double tol = (double)(p > 1 ? p : 1) * DBL_EPSILON;
    __syncthreads();
    for (int sweep = 0; sweep < 60; ++sweep) {
        if (threadIdx.x == 0) sm.flag = 0;
        __syncthreads();
        for (int round = 0; round < qe - 1; ++round) {
            for (int pr = warp; pr < npairs; pr += NWARPS) {
                int pa = pr, pb = qe - 1 - pr;
                int i = pa == 0 ? 0 : ((pa - 1 + round) % (qe - 1)) + 1;
                int j = pb == 0 ? 0 : ((pb - 1 + round) % (qe - 1)) + 1;
                if (i >= q || j >= q) continue;
                if (i > j) { int tmp = i; i = j; j = tmp; }
                double* wi = W + (int64_t)i * ldw;
                double* wj = W + (int64_t)j * ldw;
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int r = lane; r < p; r += 32) {
                    double x = wi[r], y = wj[r];
                    al = fma(x, x, al);
                    be = fma(y, y, be);
                    ga = fma(x, y, ga);
                }
                al = warp_sum(al);
                be = warp_sum(be);
                ga = warp_sum(ga);
                if (al == 0.0 || be == 0.0) continue;
                if (fabs(ga) <= tol * sqrt(al) * sqrt(be)) continue;
                double zeta = (be - al) / (2.0 * ga);
                double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                double c = 1.0 / sqrt(1.0 + tt * tt);
                double s = c * tt;
                for (int r = lane; r < p; r += 32) {
                    double x = wi[r], y = wj[r];
                    wi[r] = c * x - s * y;
                    wj[r] = s * x + c * y;
                }
                double* vi = V + i * q;
                double* vj = V + j * q;
                for (int r = lane; r < q; r += 32) {
                    double x = vi[r], y = vj[r];
                    vi[r] = c * x - s * y;
                    vj[r] = s * x + c * y;
                }
                if (lane == 0) sm.flag = 1;
            }
            __syncthreads();
        }
        if (sm.flag == 0) {
            if (threadIdx.x == 0) sm.sweeps = sweep + 1;
            break;
        }
        __syncthreads();
        if (threadIdx.x == 0) sm.sweeps = sweep + 1;
    }
    __syncthreads();
}

// Column norms of W -> sm.sig (unsorted), then ranks -> sm.ord (sorted desc,
// ties by index), then the rank cutoff and the truncation policy -> sm.k.
__device__ void sort_and_truncate(const double* W, int ldw, int p, int q, const SvdTask& t,
                                  Small& sm, bool norms_in_raw = false) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* raw = sm.raw;
    if (norms_in_raw) {  // squared column norms left exact by the Jacobi (jacobi_bisect64)
        if (threadIdx.x < q) raw[threadIdx.x] = sqrt(raw[threadIdx.x]);
    } else {
        for (int j = warp; j < q; j += NWARPS) {
            const double* w = W + (int64_t)j * ldw;
            double a = 0.0;
            for (int r = lane; r < p; r += 32) a = fma(w[r], w[r], a);
            a = warp_sum(a);
            if (lane == 0) raw[j] = sqrt(a);
        }
    }
    __syncthreads();
    if (threadIdx.x < q) {
        int me = threadIdx.x;
        double s = raw[me];
        int rank = 0;
        for (int j = 0; j < q; ++j) {
            double o = raw[j];
            rank += (o > s) || (o == s && j < me);
        }
        sm.ord[rank] = me;
        sm.sig[rank] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // svd.hpp:118-124
        double cutoff = kNumericalRankCutoff * (q > 0 ? sm.sig[0] : 0.0);
        int k = 0;
        while (k < q && sm.sig[k] > 0.0 && sm.sig[k] >= cutoff) ++k;
        sm.knum = k;
        int keep = k;
        if (t.trunc.kind == TRUNC_FIXED) {
            keep = t.trunc.k < k ? t.trunc.k : k;
        } else if (t.trunc.kind == TRUNC_ENERGY) {
            // svd.hpp:141-160: sequential cumulative energy, early break
            double total = 0.0;
            for (int i = 0; i < k; ++i) total += sm.sig[i] * sm.sig[i];
            if (total == 0.0) {
                keep = 0;
            } else {
                double cum = 0.0;
                for (int i = 0; i < k; ++i) {
                    cum += sm.sig[i] * sm.sig[i];
                    if (cum / total >= t.trunc.xi) {
                        keep = i + 1;
                        break;
                    }
                }
            }
        }
        if (keep > t.kcap) sm.status = TASK_CAPACITY;
        sm.k = keep;
    }
    __syncthreads();
}

// canonical_sign (svd.hpp:179-203) on the output V (nv x k, ld) in global
// memory: pivot = first index of the strict max |v|; flip when negative.
// Leaves the multipliers in sm.sgn and flips V in place.
__device__ void canonical_sign_global(double* v, int64_t ldv, int nv, int k, Small& sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int c = warp; c < k; c += NWARPS) {
        double best = -1.0;
        int idx = 0x7fffffff;
        for (int r = lane; r < nv; r += 32) {
            double mag = fabs(v[(int64_t)r * ldv + c]);
            if (mag > best) { best = mag; idx = r; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            double ob = __shfl_xor_sync(0xffffffffu, best, o);
            int oi = __shfl_xor_sync(0xffffffffu, idx, o);
            if (ob > best || (ob == best && oi < idx)) { best = ob; idx = oi; }
        }
        double sg = (nv > 0 && v[(int64_t)idx * ldv + c] < 0.0) ? -1.0 : 1.0;
        if (lane == 0) sm.sgn[c] = sg;
        if (sg < 0.0)
            for (int r = lane; r < nv; r += 32) v[(int64_t)r * ldv + c] = -v[(int64_t)r * ldv + c];
    }
    __syncthreads();
}

// Writes V_final (nv x k) = [vpre *] Vsrc(:, ord) where Vsrc(j, r) = src[ord[r]*ld + j] * scale[r].
__device__ void write_v(const SvdTask& t, const double* src, int ld, int nsrc, const double* colscale,
                        Small& sm) {
    const int k = sm.k;
    if (t.vpre) {
        const int nv = t.nvpre;
        for (int idx = threadIdx.x; idx < nv * k; idx += T) {
            int a = idx / k, r = idx % k;
            const double* col = src + (int64_t)sm.ord[r] * ld;
            const double* pre = t.vpre + (int64_t)a * t.ldvpre;
            double acc = 0.0;
            for (int j = 0; j < nsrc; ++j) acc = fma(pre[j], col[j], acc);
            t.v[(int64_t)a * t.ldv + r] = colscale ? acc * colscale[r] : acc;
        }
    } else {
        for (int idx = threadIdx.x; idx < nsrc * k; idx += T) {
            int a = idx / k, r = idx % k;
            double x = src[(int64_t)sm.ord[r] * ld + a];
            t.v[(int64_t)a * t.ldv + r] = colscale ? x * colscale[r] : x;
        }
    }
    __syncthreads();
}

// Epilogue shared by the direct path and the fallback: W (p x q, col-major,
// ld p) holds the rotated columns, V (q x q) the accumulated rotations.
__device__ void finish_from_jacobi(SvdTask& t, double* W, int ldw, double* V, Small& sm) {
    const int p = sm.p, q = sm.q;
    sort_and_truncate(W, ldw, p, q, t, sm);
    if (sm.status != TASK_OK) return;
    const int k = sm.k;
    double* inv_sig = sm.inv_sig;
    if (threadIdx.x < k) inv_sig[threadIdx.x] = 1.0 / sm.sig[threadIdx.x];
    __syncthreads();
    const int nv = t.vpre ? t.nvpre : (sm.tall ? q : p);
    // A's V: tall -> V(:, ord); wide -> W(:, ord) / sigma.
    if (sm.tall) write_v(t, V, q, q, nullptr, sm);
    else write_v(t, W, ldw, p, inv_sig, sm);
    if (t.sign) {
        canonical_sign_global(t.v, t.ldv, nv, k, sm);
    } else {
        if (threadIdx.x < k) sm.sgn[threadIdx.x] = 1.0;
        __syncthreads();
    }
    // A's U (m x k): tall -> W(:, ord) / sigma; wide -> V(:, ord).
    const int m = sm.m;
    for (int idx = threadIdx.x; idx < m * k; idx += T) {
        int i = idx / k, r = idx % k;
        double x = sm.tall ? W[(int64_t)sm.ord[r] * ldw + i] * inv_sig[r] : V[sm.ord[r] * q + i];
        t.u[(int64_t)i * t.ldu + r] = x * sm.sgn[r];
    }
    if (threadIdx.x < k) t.s[threadIdx.x] = sm.sig[threadIdx.x];
    if (threadIdx.x == 0) *t.k_out = (double)k;
    __syncthreads();
}

__device__ bool setup(SvdTask& t, Small& sm) {
    if (threadIdx.x == 0) {
        int m = t.m_from ? t.m_from[0] : t.m;
        int n = t.n_from ? (int)t.n_from[0] : t.n;
        sm.m = m;
        sm.n = n;
        sm.tall = m >= n;
        sm.p = sm.tall ? m : n;
        sm.q = sm.tall ? n : m;
        sm.status = TASK_OK;
        sm.k = 0;
        sm.sweeps = 0;
        sm.reason = 0;
        for (int i = 0; i < 8; ++i) sm.clk[i] = 0;
        sm.clk[0] = clock64();
        if (m == 0 || n == 0) {
            *t.k_out = 0.0;
        } else if (sm.q > kQMax) {
            sm.status = TASK_UNSUPPORTED;
        }
    }
    __syncthreads();
    return sm.m > 0 && sm.n > 0 && sm.status == TASK_OK;
}

// ===================================================================== v4
// Phase kernels.  A task's rows are split into `nsplit` ranges of
// `rows_per_split` rows; pass kernels run one CTA per (split, task) and leave
// Q x Q partial Grams in the task workspace, mid kernels run one CTA per task
// and combine them in a fixed order (bitwise reproducible).
//
//   P1  G  = sum_s W_s^T W_s                              (DMMA Gram)
//   M1  G  = R1^T R1 (blocked Cholesky); inverses of R1's 8x8 diagonal blocks
//   P2  G2 = sum_s (W_s R1^-1)^T (W_s R1^-1)               (DMMA block TRSM + Gram)
//   M2  G2 = R2^T R2, R = R2 R1  (CholeskyQR2: W = Q2 R, Q2 orthonormal)
//       one-sided Jacobi on R^T:  R^T J = Y,  Y = V S  (sigma_j = |y_j|, V_W = Y S^-1)
//       J = R^-T Y_k (the left singular vectors of R), M = R^-1 J S-signs
//   P3  U_W = W M  streamed out (DMMA GEMM), U_W^T U_W partials
//   C   orthonormality check (else the robust fallback), wide-case sign, rank
//
// Why J = R^-T Y and not R V S^-1: an angle error d of v_c towards v_1 turns
// into kappa_c^2 d in R V S^-1 but into d / kappa_c in R^-T Y, so U_W = Q2 J
// stays orthonormal to ~eps * kappa(R) (checked in C against 1e-10).
// W = A (m >= n) or A^T; q = min(m, n) <= Q in {16, 32, 64}.

constexpr int WS_Q2 = kWsQ2;  // layout constants: zsvd_internal.h

template <int Q>
struct G3 {
    static constexpr int JLD = Q + 2;         // Jacobi column stride (16-byte aligned columns)
    static constexpr int LPP = Q >= 32 ? 8 : 4;                      // lanes per Jacobi pair
    static constexpr int EPL2 = Q / (2 * LPP);                       // double2 per lane per column
    static constexpr int SLOTS = T / LPP;
};

struct Geo {
    int m, n, p, q, tall;
};

__device__ __forceinline__ Geo geometry(const SvdTask& t) {
    Geo g;
    g.m = t.m_from ? t.m_from[0] : t.m;
    g.n = t.n_from ? (int)t.n_from[0] : t.n;
    g.tall = g.m >= g.n;
    g.p = g.tall ? g.m : g.n;
    g.q = g.tall ? g.n : g.m;
    return g;
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// Blocked upper Cholesky of the leading q x q block of G (row-major ld Q), in
// place; identity beyond q, zero strict lower part.  8-column blocks: warp 0
// factors the diagonal block in registers (lane L holds entries L and L + 32
// of the 8 x 8 block; pivots and row j travel by shuffles, no shared-memory
// round trips), the panel is solved column-parallel in eager order (each x_i
// is folded into the later accumulators as soon as it exists: the critical
// path is 8 multiply-adds, not 36), the trailing matrix is updated in
// parallel with two accumulator chains (3 barriers per block).
template <int Q>
__device__ bool chol3(double* G, int q, Small& sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* rinv = sm.rinv;  // 1 / R_jj
    if (threadIdx.x == 0) {
        sm.flag = 1;
        sm.pivmin = DBL_MAX;
        sm.pivmax = 0.0;
    }
    __syncthreads();
    for (int o = 0; o < q; o += 8) {
        const int w = min(8, q - o);
        if (warp == 0) {
            // entry e of the block: (l, c) = (e >> 3, e & 7); lane holds e = lane, lane + 32
            const int l0 = lane >> 3, c0 = lane & 7, l1 = l0 + 4;
            double v0 = (l0 < w && c0 < w) ? G[(o + l0) * Q + o + c0] : 0.0;
            double v1 = (l1 < w && c0 < w) ? G[(o + l1) * Q + o + c0] : 0.0;
            bool ok = true;
            double pmin = DBL_MAX, pmax = 0.0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (j < w) {
                    const int ej = 9 * j;  // (j, j)
                    const double d = __shfl_sync(0xffffffffu, ej < 32 ? v0 : v1, ej & 31);
                    const bool okj = d >= DBL_MIN && isfinite(d);
                    const double inv = okj ? rsqrt_nr(d) : 1.0;
                    const double r = okj ? d * inv : 1.0;
                    ok = ok && okj;
                    pmin = fmin(pmin, okj ? r : 0.0);
                    pmax = fmax(pmax, r);
                    if (lane == 0) rinv[o + j] = inv;
                    // row j: (j, j) = r, (j, c > j) scaled
                    if (j < 4) {
                        if (l0 == j) v0 = c0 == j ? r : (c0 > j ? v0 * inv : v0);
                    } else {
                        if (l1 == j) v1 = c0 == j ? r : (c0 > j ? v1 * inv : v1);
                    }
                    // R_j,c0, R_j,l0, R_j,l1 (row j lives in one slot)
                    const double src = j < 4 ? v0 : v1;
                    const int base = (8 * j) & 31;
                    const double rjc = __shfl_sync(0xffffffffu, src, base + c0);
                    const double rjl0 = __shfl_sync(0xffffffffu, src, base + l0);
                    const double rjl1 = __shfl_sync(0xffffffffu, src, base + l1);
                    if (l0 > j && c0 >= l0) v0 = fma(-rjl0, rjc, v0);
                    if (l1 > j && c0 >= l1) v1 = fma(-rjl1, rjc, v1);
                }
            }
            if (l0 < w && c0 < w && c0 >= l0) G[(o + l0) * Q + o + c0] = v0;
            if (l1 < w && c0 < w && c0 >= l1) G[(o + l1) * Q + o + c0] = v1;
            if (lane == 0) {
                if (!ok) sm.flag = 0;
                sm.pivmin = fmin(sm.pivmin, pmin);
                sm.pivmax = fmax(sm.pivmax, pmax);
            }
        }
        __syncthreads();
        if (!sm.flag) return false;
        // panel: R[o:o+w, c] = R_oo^-T G[o:o+w, c] for c >= o + w (column-parallel, eager)
        for (int c = o + w + threadIdx.x; c < q; c += T) {
            double acc[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = j < w ? G[(o + j) * Q + c] : 0.0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (i < w) {
                    acc[i] *= rinv[o + i];
#pragma unroll
                    for (int j = i + 1; j < 8; ++j)
                        if (j < w) acc[j] = fma(-G[(o + i) * Q + o + j], acc[i], acc[j]);
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (j < w) G[(o + j) * Q + c] = acc[j];
        }
        __syncthreads();
        // trailing update (upper triangle): G[l][c] -= sum_j R[o+j][l] R[o+j][c]
        const int base = o + w;
        for (int l = base + warp; l < q; l += NWARPS) {
            double rl[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) rl[j] = j < w ? G[(o + j) * Q + l] : 0.0;
            for (int c = l + lane; c < q; c += 32) {
                double a0 = G[l * Q + c], a1 = 0.0;
#pragma unroll
                for (int j = 0; j < 8; j += 2) {
                    a0 = fma(-rl[j], j < w ? G[(o + j) * Q + c] : 0.0, a0);
                    a1 = fma(-rl[j + 1], j + 1 < w ? G[(o + j + 1) * Q + c] : 0.0, a1);
                }
                G[l * Q + c] = a0 + a1;
            }
        }
        __syncthreads();
    }
    for (int idx = threadIdx.x; idx < Q * Q; idx += T) {
        const int i = idx / Q, c = idx % Q;
        if (i >= q || c >= q) G[idx] = (i == c) ? 1.0 : 0.0;
        else if (c < i) G[idx] = 0.0;
    }
    __syncthreads();
    return true;
}

// A sweep whose rotations all had |cos| < kCheckCos is in the quadratic
// regime: instead of a confirming rotation-free sweep (q - 1 dependent rounds),
// the whole Gram Y^T Y is formed once (~2 us) and every pair is tested
// against the sweep's own criterion g^2 <= tol^2 a b with exact norms.  If one
// fails, sweeping continues as before.
constexpr double kCheckCos = 1e-6;

// Y (Q x Q col-major, ld JLD, columns >= q ignored): true iff every live pair
// satisfies g^2 <= tol2 a b.  Thread t owns a (Q/16) x (Q/16) tile of the Gram.
template <int Q, int JLD>
__device__ bool gram_converged(const double* Y, int q, double tol2, Small& sm) {
    constexpr int TL = Q / 16;
    const int ti = threadIdx.x >> 4, tj = threadIdx.x & 15;
    double acc[TL][TL];
#pragma unroll
    for (int r = 0; r < TL; ++r)
#pragma unroll
        for (int c = 0; c < TL; ++c) acc[r][c] = 0.0;
    const double* yi = Y + ti * TL * JLD;
    const double* yj = Y + tj * TL * JLD;
#pragma unroll 4
    for (int e = 0; e < Q; ++e) {
        double a[TL], b[TL];
#pragma unroll
        for (int r = 0; r < TL; ++r) {
            a[r] = yi[r * JLD + e];
            b[r] = yj[r * JLD + e];
        }
#pragma unroll
        for (int r = 0; r < TL; ++r)
#pragma unroll
            for (int c = 0; c < TL; ++c) acc[r][c] = fma(a[r], b[c], acc[r][c]);
    }
    double* nrm = sm.raw;
    if (threadIdx.x == 0) sm.conv = 1;
    if (ti == tj) {
#pragma unroll
        for (int r = 0; r < TL; ++r) nrm[ti * TL + r] = acc[r][r];
    }
    __syncthreads();
    bool ok = true;
#pragma unroll
    for (int r = 0; r < TL; ++r)
#pragma unroll
        for (int c = 0; c < TL; ++c) {
            const int i = ti * TL + r, j = tj * TL + c;
            if (i < j && j < q) {
                const double a = nrm[i], b = nrm[j], g = acc[r][c];
                if (a > 0.0 && b > 0.0 && g * g > tol2 * a * b) ok = false;
            }
        }
    if (!ok) sm.conv = 0;
    __syncthreads();
    const bool conv = sm.conv != 0;
    __syncthreads();
    return conv;
}

// One-sided Jacobi on the q live columns of Y (Q x Q col-major, ld JLD), no
// accumulation.  LPP lanes per pair (double2 accesses), all pairs of a round
// at once (circle ordering).  The rotation angle uses approximate reciprocals
// (it only steers convergence); cos/sin come from a full-precision rsqrt, so
// every applied rotation is orthogonal to working precision.
template <int Q>
__device__ void jacobi4(double* Y, int q, Small& sm) {
    using C3 = G3<Q>;
    const int slot = threadIdx.x / C3::LPP, li = threadIdx.x % C3::LPP;
    const int qe = q + (q & 1);
    const int npairs = qe / 2;
    const double tol = (double)(q > 1 ? q : 1) * DBL_EPSILON;
    const double tol2 = tol * tol;
    const double chk2 = kCheckCos * kCheckCos;
    int sweep = 0;
    for (; sweep < 40; ++sweep) {
        if (threadIdx.x == 0) {
            sm.flag = 0;
            sm.bigf[0] = 0;
        }
        __syncthreads();
        int ia = slot, ib = qe - 1 - slot;
        for (int round = 0; round < qe - 1; ++round) {
            for (int base = 0; base < npairs; base += C3::SLOTS) {
                const int pr = base + slot;
                int i = 0, j = 0;
                bool act = pr < npairs;
                if (act) {
                    int pi = pr == 0 ? 0 : ia, pj = ib;
                    if (base > 0) {
                        const int pa = pr, pb = qe - 1 - pr;
                        pi = pa == 0 ? 0 : ((pa - 1 + round) % (qe - 1)) + 1;
                        pj = pb == 0 ? 0 : ((pb - 1 + round) % (qe - 1)) + 1;
                    }
                    i = min(pi, pj);
                    j = max(pi, pj);
                    act = j < q;
                }
                double2* yi = reinterpret_cast<double2*>(Y + i * C3::JLD);
                double2* yj = reinterpret_cast<double2*>(Y + j * C3::JLD);
                double2 xi[C3::EPL2], xj[C3::EPL2];
                double a = 0.0, b = 0.0, g = 0.0, a1 = 0.0, b1 = 0.0, g1 = 0.0;
#pragma unroll
                for (int e = 0; e < C3::EPL2; ++e) {
                    xi[e] = act ? yi[li + e * C3::LPP] : make_double2(0.0, 0.0);
                    xj[e] = act ? yj[li + e * C3::LPP] : make_double2(0.0, 0.0);
                }
#pragma unroll
                for (int e = 0; e < C3::EPL2; ++e) {
                    a = fma(xi[e].x, xi[e].x, a);
                    b = fma(xj[e].x, xj[e].x, b);
                    g = fma(xi[e].x, xj[e].x, g);
                    a1 = fma(xi[e].y, xi[e].y, a1);
                    b1 = fma(xj[e].y, xj[e].y, b1);
                    g1 = fma(xi[e].y, xj[e].y, g1);
                }
                a += a1;
                b += b1;
                g += g1;
#pragma unroll
                for (int o = 1; o < C3::LPP; o <<= 1) {
                    a += __shfl_xor_sync(0xffffffffu, a, o);
                    b += __shfl_xor_sync(0xffffffffu, b, o);
                    g += __shfl_xor_sync(0xffffffffu, g, o);
                }
                if (act && a > 0.0 && b > 0.0 && g * g > tol2 * a * b) {
                    const double d = b - a;
                    const double h2 = fma(d, d, 4.0 * g * g);
                    double rh, rd;
                    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rh) : "d"(h2));
                    const double den = fma(h2, rh, fabs(d));  // |d| + sqrt(d^2 + 4 g^2)
                    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rd) : "d"(den));
                    rd = rd * fma(-den, rd, 2.0);
                    double tt = 2.0 * g * rd;
                    if (d < 0.0) tt = -tt;
                    const double cth = rsqrt_nr(fma(tt, tt, 1.0));
                    const double sth = cth * tt;
#pragma unroll
                    for (int e = 0; e < C3::EPL2; ++e) {
                        yi[li + e * C3::LPP] = make_double2(cth * xi[e].x - sth * xj[e].x, cth * xi[e].y - sth * xj[e].y);
                        yj[li + e * C3::LPP] = make_double2(sth * xi[e].x + cth * xj[e].x, sth * xi[e].y + cth * xj[e].y);
                    }
                    sm.flag = 1;
                    if (g * g > chk2 * a * b) sm.bigf[0] = 1;
                }
            }
            if (slot != 0) ia = ia == qe - 1 ? 1 : ia + 1;
            ib = ib == qe - 1 ? 1 : ib + 1;
            __syncthreads();
        }
        if (sm.flag == 0) break;
        const bool check = sm.bigf[0] == 0;
        __syncthreads();
        if (check && gram_converged<Q, C3::JLD>(Y, q, tol2, sm)) break;
    }
    if (threadIdx.x == 0) sm.sweeps = sweep + 1;
    __syncthreads();
}

// One-sided Jacobi for Q = 64 in the recursive-bisection tournament ordering:
// phase G = 32, 16, ..., 1 pairs the two halves of every 2G-group, G rounds per
// phase (63 rounds per sweep, every pair once).  Within a phase each slot keeps
// its "x" column in registers and only its partner "y" moves (to the neighbour
// slot, through its home column in Y), so a round moves one column per pair
// instead of two.  Columns >= q are dummies.  Same rotation as jacobi4.
__device__ void jacobi_bisect64(double* Y, int q, Small& sm) {
    using C3 = G3<64>;
    constexpr int LPP = C3::LPP, EPL2 = C3::EPL2;  // 8 lanes, 4 double2 per lane per column
    int* flags = sm.flags;
    double* nrm = sm.raw;  // squared column norms, tracked through the rotations
    const int slot = threadIdx.x / LPP, li = threadIdx.x % LPP;  // 32 slots
    const double tol = (double)(q > 1 ? q : 1) * DBL_EPSILON;
    const double tol2 = tol * tol;
    const double chk2 = kCheckCos * kCheckCos;
    if (threadIdx.x == 0) flags[0] = flags[1] = sm.bigf[0] = sm.bigf[1] = 0;
    __syncthreads();
    int sweep = 0;
    for (; sweep < 40; ++sweep) {
        const int fcur = sweep & 1;
        if (threadIdx.x == 0) flags[fcur ^ 1] = sm.bigf[fcur ^ 1] = 0;
        // fresh norms at every sweep start: the tracked values steer the rotations
        // within a sweep; the last (rotation-free) sweep decides on exact norms
        for (int cc = slot; cc < 64; cc += 32) {
            const double2* col = reinterpret_cast<const double2*>(Y + cc * C3::JLD);
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int e = 0; e < EPL2; ++e) {
                const double2 v = col[li + e * LPP];
                a0 = fma(v.x, v.x, a0);
                a1 = fma(v.y, v.y, a1);
            }
            double a = a0 + a1;
#pragma unroll
            for (int o = 1; o < LPP; o <<= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (li == 0) nrm[cc] = cc < q ? a : 0.0;
        }
        __syncthreads();
        for (int G = 32; G >= 1; G >>= 1) {
            const int grp = slot / G, ls = slot % G;
            const int xi = grp * 2 * G + ls;
            const bool xlive = xi < q;
            double2 X[EPL2], Yc[EPL2];
            const double2* xcol = reinterpret_cast<const double2*>(Y + xi * C3::JLD);
#pragma unroll
            for (int e = 0; e < EPL2; ++e) X[e] = xlive ? xcol[li + e * LPP] : make_double2(0.0, 0.0);
            double a = nrm[xi];
            for (int r = 0; r < G; ++r) {
                const int yi = grp * 2 * G + G + ((ls + r) & (G - 1));
                const bool act = xlive && yi < q;
                double2* ycol = reinterpret_cast<double2*>(Y + yi * C3::JLD);
#pragma unroll
                for (int e = 0; e < EPL2; ++e) Yc[e] = act ? ycol[li + e * LPP] : make_double2(0.0, 0.0);
                double g = 0.0, g1 = 0.0;
#pragma unroll
                for (int e = 0; e < EPL2; ++e) {
                    g = fma(X[e].x, Yc[e].x, g);
                    g1 = fma(X[e].y, Yc[e].y, g1);
                }
                g += g1;
#pragma unroll
                for (int o = 1; o < LPP; o <<= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
                const double b = nrm[yi];
                if (act && a > 0.0 && b > 0.0 && g * g > tol2 * a * b) {
                    // pair (i, j) = (x, y) since x < y always
                    const double d = b - a;
                    const double h2 = fma(d, d, 4.0 * g * g);
                    double rh, rd;
                    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rh) : "d"(h2));
                    const double den = fma(h2, rh, fabs(d));
                    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rd) : "d"(den));
                    rd = rd * fma(-den, rd, 2.0);
                    double tt = 2.0 * g * rd;
                    if (d < 0.0) tt = -tt;
                    const double cth = rsqrt_nr(fma(tt, tt, 1.0));
                    const double sth = cth * tt;
#pragma unroll
                    for (int e = 0; e < EPL2; ++e) {
                        const double2 x = X[e], y = Yc[e];
                        X[e] = make_double2(cth * x.x - sth * y.x, cth * x.y - sth * y.y);
                        ycol[li + e * LPP] = make_double2(sth * x.x + cth * y.x, sth * x.y + cth * y.y);
                    }
                    // |x'|^2 = a - t g, |y'|^2 = b + t g for the exact rotation
                    a = fma(-tt, g, a);
                    if (li == 0) nrm[yi] = fma(tt, g, b);
                    flags[fcur] = 1;
                    if (g * g > chk2 * a * b) sm.bigf[fcur] = 1;
                }
                __syncthreads();  // y columns (and norms) home before the neighbour reads them
            }
            if (xlive) {
                double2* xw = reinterpret_cast<double2*>(Y + xi * C3::JLD);
#pragma unroll
                for (int e = 0; e < EPL2; ++e) xw[li + e * LPP] = X[e];
                if (li == 0) nrm[xi] = a;
            }
            __syncthreads();
        }
        const bool done = flags[fcur] == 0;
        const bool check = sm.bigf[fcur] == 0;
        __syncthreads();  // everyone has read the flag before it is reset
        if (done) break;
        if (check && gram_converged<64, C3::JLD>(Y, q, tol2, sm)) break;
    }
    if (threadIdx.x == 0) sm.sweeps = sweep + 1;
    __syncthreads();
}

// ---------------------------------------------------------------- bodies
// ---------------------------------------------------------------- slab passes
// Passes 1-3 by warp pairs over 16-row double slabs.  Pair p (warps 2p, 2p+1)
// streams rows r0 + 16 d, d = p, p + 4, ..., through a two-deep cp.async
// staging ring of its own and synchronises only with named barriers, so a
// pass needs no CTA barrier per chunk.  Member m loads / solves / forms the
// 8-row half m; both members then fold both halves into their half of the
// upper Gram tiles (tile index parity = member), held in registers.
// Register layouts (mma.m8n8k4 f64 fragments, lane L):
//   C (accumulator)  X[L>>2][8i + 2(L&3) + {0,1}]    one double2 per 8x8 tile i
//   A (row operand)  X[L>>2][4s + (L&3)]              k-slice s of a row block
//   F (Gram operand) X[4h + (L&3)][8i + (L>>2)]       tile i, k-step h (= A and
//                                                     B operand of X^T X tiles)
// The pairs' partial Grams are summed in a fixed order (deterministic).
template <int Q>
struct SlabG {
    static constexpr int LDX = Q + 4;                   // staging row stride
    static constexpr int HALF = 8 * LDX;                // one 8-row half
    static constexpr int SLAB = 2 * HALF;               // one staged double slab
    static constexpr int T8 = Q / 8;
    static constexpr int NUP = T8 * (T8 + 1) / 2;
    static constexpr int NOWN = (NUP + 1) / 2;          // tiles per member
    static constexpr int NPAIR = NWARPS / 2;
    static constexpr int STAGE = NPAIR * 2 * SLAB;      // all pairs' rings
    static constexpr int MLD = Q + 4;                   // R1 / M row stride in smem
    static constexpr int DLD = 20;                      // Dinv block row stride
    // (strides = 4 mod 16 doubles: the 4 k-rows of a B fragment hit distinct banks)
};

__device__ __forceinline__ void pair_sync() {
    asm volatile("bar.sync %0, 64;" ::"r"(1 + (int)(threadIdx.x >> 6)) : "memory");
}

// C-layout tile -> A fragment of k-slice s (4 columns) of the same rows.
__device__ __forceinline__ double c_to_a(double2 c, int s) {
    const int lane = threadIdx.x & 31;
    const int src = (lane & ~3) | (2 * (s & 1) + ((lane & 3) >> 1));
    const double x = __shfl_sync(0xffffffffu, c.x, src);
    const double y = __shfl_sync(0xffffffffu, c.y, src);
    return (lane & 1) ? y : x;
}

template <int Q>
struct SlabGram {
    using S = SlabG<Q>;
    double c[S::NOWN][2];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int i = 0; i < S::NOWN; ++i) c[i][0] = c[i][1] = 0.0;
    }
    // F fragments of one 8-row half into this member's tiles among the first
    // LT column tiles (compile-time member and extent: a predicated-off mma
    // still occupies the tensor pipe)
    template <int M, int LT>
    __device__ __forceinline__ void add(const double (&F)[S::T8][2]) {
        int idx = 0;
#pragma unroll
        for (int ti = 0; ti < S::T8; ++ti)
#pragma unroll
            for (int tj = ti; tj < S::T8; ++tj, ++idx)
                if ((idx & 1) == M && tj < LT) {
                    dmma(c[idx / 2][0], c[idx / 2][1], F[ti][0], F[tj][0]);
                    dmma(c[idx / 2][0], c[idx / 2][1], F[ti][1], F[tj][1]);
                }
    }
    // Sum of all warps' partials -> dst (Q x Q, ld ldd, both triangles).  G is
    // Q x Q shared scratch; ends with a barrier.
    __device__ void reduce_store(double* G, double* dst, int ldd) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, member = warp & 1;
        for (int w = 0; w < NWARPS; ++w) {
            if (warp == w) {
                int idx = 0;
#pragma unroll
                for (int ti = 0; ti < S::T8; ++ti)
#pragma unroll
                    for (int tj = ti; tj < S::T8; ++tj, ++idx)
                        if ((idx & 1) == member) {
                            double* g = G + (8 * ti + (lane >> 2)) * Q + 8 * tj + 2 * (lane & 3);
                            if (w < 2) {
                                g[0] = c[idx / 2][0];
                                g[1] = c[idx / 2][1];
                            } else {
                                g[0] += c[idx / 2][0];
                                g[1] += c[idx / 2][1];
                            }
                        }
            }
            __syncthreads();
        }
        for (int idx = threadIdx.x; idx < Q * Q; idx += T) {
            const int i = idx / Q, j = idx % Q;
            dst[i * ldd + j] = (i / 8 <= j / 8) ? G[idx] : G[j * Q + i];
        }
        __syncthreads();
    }
};

// Issues the staged load of rows [row0, row0 + 8) into half (this warp only).
// Fast path: 16-byte cp.async of the q live columns; rows >= rend are zero.
// Otherwise scalar loads through w_at (wide or scaled operands).
template <int Q>
__device__ __forceinline__ void slab_issue(const SvdTask& t, const Geo& g, bool fast, double* half, int row0,
                                           int rend) {
    using S = SlabG<Q>;
    const int lane = threadIdx.x & 31;
    if (fast) {
        const int segs = g.q / 2;
        for (int idx = lane; idx < 8 * segs; idx += 32) {
            const int r = idx / segs, sg = idx % segs;
            const int gr = row0 + r;
            double* d = half + r * S::LDX + 2 * sg;
            if (gr < rend) {
                cp_async16(d, t.a + (int64_t)gr * t.lda + 2 * sg);
            } else {
                d[0] = 0.0;
                d[1] = 0.0;
            }
        }
    } else {
        for (int idx = lane; idx < 8 * g.q; idx += 32) {
            const int r = idx / g.q, j = idx % g.q;
            const int gr = row0 + r;
            half[r * S::LDX + j] = gr < rend ? w_at(t, g.tall, gr, j) : 0.0;
        }
    }
    cp_async_commit();
}

template <int Q>
__device__ __forceinline__ void slab_load_f(const double* half, double (&F)[SlabG<Q>::T8][2]) {
    using S = SlabG<Q>;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < S::T8; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h) F[i][h] = half[(4 * h + (lane & 3)) * S::LDX + 8 * i + (lane >> 2)];
}

// X (8 rows, C layout) <- X R^-1 (R upper triangular row-major ld Q, Dinv the
// inverses of its 16x16 diagonal blocks), block column by block column:
// Y_b = X_b Dinv_b, then X_t -= Y_b R[b, t] for the tiles t beyond the block.
template <int Q>
__device__ __forceinline__ void slab_trsm(double2 (&X)[SlabG<Q>::T8], const double* R, const double* Dinv, int q) {
    using S = SlabG<Q>;
    const int lane = threadIdx.x & 31;
    const int kr = lane & 3, nc = lane >> 2;
#pragma unroll
    for (int b = 0; b < Q / 16; ++b) {
        if (16 * b >= q) break;
        double a[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) a[s] = c_to_a(X[2 * b + s / 2], s);
        const double* D = Dinv + b * 16 * S::DLD;
        double2 y[2];
#pragma unroll
        for (int n = 0; n < 2; ++n) {
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int s = 0; s < 4; ++s) dmma(c0, c1, a[s], D[(4 * s + kr) * S::DLD + 8 * n + nc]);
            y[n] = make_double2(c0, c1);
        }
        X[2 * b] = y[0];
        X[2 * b + 1] = y[1];
#pragma unroll
        for (int s = 0; s < 4; ++s) a[s] = c_to_a(y[s / 2], s);
#pragma unroll
        for (int tt = 2 * b + 2; tt < S::T8; ++tt) {
            if (8 * tt >= q) break;
            double c0 = X[tt].x, c1 = X[tt].y;
#pragma unroll
            for (int s = 0; s < 4; ++s) dmma(c0, c1, a[s], -R[(16 * b + 4 * s + kr) * S::MLD + 8 * tt + nc]);
            X[tt] = make_double2(c0, c1);
        }
    }
}

template <int Q, int PHASE, int M, int LT>
__device__ void slab_loop(SvdTask& t, const Geo& g, int split, double* dyn, bool fast, double* out, int64_t ldo) {
    using S = SlabG<Q>;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pair = warp >> 1;
    double* ring = dyn + pair * 2 * S::SLAB;
    const double* Mt = dyn + S::STAGE;  // P2: R1 (Q x MLD) | P3: M (Q x MLD)
    const double* Dv = Mt + Q * S::MLD; // P2: 16x16 diagonal inverses (ld DLD)
    const int r0 = split * t.rows_per_split;
    const int rend = min(g.p, r0 + t.rows_per_split);
    const int nds = rend > r0 ? (rend - r0 + 15) / 16 : 0;
    const int k = t.krank;
    SlabGram<Q> gr;
    gr.init();
    if (pair < nds) slab_issue<Q>(t, g, fast, ring + M * S::HALF, r0 + 16 * pair + 8 * M, rend);
    int it = 0;
    for (int d = pair; d < nds; d += S::NPAIR, ++it) {
        double* buf = ring + (it & 1) * S::SLAB;
        if (d + S::NPAIR < nds) {
            slab_issue<Q>(t, g, fast, ring + ((it + 1) & 1) * S::SLAB + M * S::HALF,
                          r0 + 16 * (d + S::NPAIR) + 8 * M, rend);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        double* mine = buf + M * S::HALF;
        if constexpr (PHASE == 2) {
            __syncwarp();
            double2 X[S::T8];
#pragma unroll
            for (int i = 0; i < S::T8; ++i)
                X[i] = *reinterpret_cast<const double2*>(mine + (lane >> 2) * S::LDX + 8 * i + 2 * (lane & 3));
            slab_trsm<Q>(X, Mt, Dv, g.q);
            __syncwarp();
#pragma unroll
            for (int i = 0; i < S::T8; ++i)
                *reinterpret_cast<double2*>(mine + (lane >> 2) * S::LDX + 8 * i + 2 * (lane & 3)) = X[i];
        } else if constexpr (PHASE == 3) {
            // U rows = X M (M = R^-1 J, Q x Q row-major, zero beyond k <= 8 LT)
            __syncwarp();
            double2 U[LT];
#pragma unroll
            for (int n = 0; n < LT; ++n) U[n] = make_double2(0.0, 0.0);
#pragma unroll
            for (int s = 0; s < Q / 4; ++s) {
                if (4 * s >= g.q) break;
                const double a = mine[(lane >> 2) * S::LDX + 4 * s + (lane & 3)];
#pragma unroll
                for (int n = 0; n < LT; ++n)
                    dmma(U[n].x, U[n].y, a, Mt[(4 * s + (lane & 3)) * S::MLD + 8 * n + (lane >> 2)]);
            }
            __syncwarp();
            const int row = r0 + 16 * d + 8 * M + (lane >> 2);
            const bool rl = row < rend;
#pragma unroll
            for (int n = 0; n < LT; ++n) {
                const int col = 8 * n + 2 * (lane & 3);
                if (rl) {
                    if (col < k) out[(int64_t)row * ldo + col] = U[n].x;
                    if (col + 1 < k) out[(int64_t)row * ldo + col + 1] = U[n].y;
                }
                // rows beyond rend and columns beyond k do not enter U^T U
                U[n].x = (rl && col < k) ? U[n].x : 0.0;
                U[n].y = (rl && col + 1 < k) ? U[n].y : 0.0;
                *reinterpret_cast<double2*>(mine + (lane >> 2) * S::LDX + col) = U[n];
            }
        }
        pair_sync();  // both halves staged (and solved / formed)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            double F[S::T8][2];
            slab_load_f<Q>(buf + hh * S::HALF, F);
            gr.template add<M, LT>(F);
        }
        pair_sync();  // both members are done with buf before it is refilled
    }
    // all warps' partial Grams -> this split's slot (the staging ring is free now)
    __syncthreads();
    gr.reduce_store(dyn, t.ws + (int64_t)split * WS_Q2, kQMax);
}

// Pass 3 over k columns: the smallest k-tile extent LT >= lt (lt >= 1).
template <int Q, int M, int LT>
__device__ void p3_dispatch(int lt, SvdTask& t, const Geo& g, int split, double* dyn, bool fast, double* out,
                            int64_t ldo) {
    if constexpr (LT < SlabG<Q>::T8) {
        if (lt > LT) {
            p3_dispatch<Q, M, LT + 1>(lt, t, g, split, dyn, fast, out, ldo);
            return;
        }
    }
    slab_loop<Q, 3, M, LT>(t, g, split, dyn, fast, out, ldo);
}

template <int Q, int PHASE>
__device__ void slab_pass(SvdTask& t, const Geo& g, int split, double* dyn) {
    using S = SlabG<Q>;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int member = warp & 1;
    double* ring = dyn + (warp >> 1) * 2 * S::SLAB;
    double* Mt = dyn + S::STAGE;
    double* Dv = Mt + Q * S::MLD;
    const bool fast = g.tall && t.colscale == nullptr && (t.lda % 2 == 0) && (g.q % 2 == 0) &&
                      ((reinterpret_cast<uintptr_t>(t.a) & 15) == 0);
    const int nsp = t.nsplit;
    // dead columns of this member's staging halves read as zero
    if (g.q < Q)
        for (int idx = lane; idx < 2 * 8 * (Q - g.q); idx += 32) {
            const int r = idx / (Q - g.q), j = g.q + idx % (Q - g.q);
            ring[(r / 8) * S::SLAB + member * S::HALF + (r % 8) * S::LDX + j] = 0.0;
        }
    if (PHASE == 2 || PHASE == 3) {
        const double* src = t.ws + (PHASE == 2 ? ws_off_r1(nsp) : ws_off_m(nsp));
        for (int idx = threadIdx.x; idx < Q * Q; idx += T) Mt[(idx / Q) * S::MLD + idx % Q] = src[(idx / Q) * kQMax + idx % Q];
    }
    if (PHASE == 2) {
        const double* dsrc = t.ws + ws_off_dinv(nsp);  // (Q/16) blocks of 16 x 16, row-major
        for (int idx = threadIdx.x; idx < Q * 16; idx += T) Dv[(idx / 16) * S::DLD + idx % 16] = dsrc[idx];
    }
    __syncthreads();
    double* out = nullptr;  // P3 output
    int64_t ldo = 0;
    if (PHASE == 3) {
        if (g.tall) {
            out = t.u;
            ldo = t.ldu;
        } else if (t.vpre) {
            out = t.ws + ws_off_stage(nsp);
            ldo = kQMax;
        } else {
            out = t.v;
            ldo = t.ldv;
        }
        // k = 0 still writes the (zero) partial Gram
        const int lt = max(1, (t.krank + 7) / 8);
        if (member) p3_dispatch<Q, 1, 1>(lt, t, g, split, dyn, fast, out, ldo);
        else p3_dispatch<Q, 0, 1>(lt, t, g, split, dyn, fast, out, ldo);
    } else {
        if (member) slab_loop<Q, PHASE, 1, S::T8>(t, g, split, dyn, fast, out, ldo);
        else slab_loop<Q, PHASE, 0, S::T8>(t, g, split, dyn, fast, out, ldo);
    }
}

// G (Q x Q) = sum of the nsplit partial Grams, added in split order (so the
// result is bitwise that of a sequential sum).  The partials were just written
// by other SMs and sit in L2: each thread keeps 8 entries x 3 splits = 24
// loads in flight per step instead of one dependent load-add chain per entry.
template <int Q>
__device__ void sum_partials(const SvdTask& t, int q, double* G) {
    constexpr int EPT = (Q * Q + T - 1) / T;  // entries per thread: 16 / 4 / 1
    constexpr int EC = EPT < 8 ? EPT : 8;     // entries per chunk
    constexpr int SC = 3;                     // splits per step
    const int ns = t.nsplit;
    const double* ws = t.ws;
#pragma unroll
    for (int e0 = 0; e0 < EPT; e0 += EC) {
        int off[EC];
        double acc[EC];
#pragma unroll
        for (int e = 0; e < EC; ++e) {
            const int idx = threadIdx.x + (e0 + e) * T;
            const int i = idx / Q, c = idx % Q;
            off[e] = (idx < Q * Q && i < q && c < q) ? i * kQMax + c : -1;
            acc[e] = 0.0;
        }
        for (int s0 = 0; s0 < ns; s0 += SC) {
            double v[SC][EC];
#pragma unroll
            for (int d = 0; d < SC; ++d)
#pragma unroll
                for (int e = 0; e < EC; ++e)
                    v[d][e] = (s0 + d < ns && off[e] >= 0) ? ws[(int64_t)(s0 + d) * WS_Q2 + off[e]] : 0.0;
#pragma unroll
            for (int d = 0; d < SC; ++d)
#pragma unroll
                for (int e = 0; e < EC; ++e)
                    if (s0 + d < ns) acc[e] += v[d][e];
        }
#pragma unroll
        for (int e = 0; e < EC; ++e) {
            const int idx = threadIdx.x + (e0 + e) * T;
            if (idx < Q * Q) G[idx] = acc[e];
            // every entry of W reaches one diagonal entry of G = W^T W as a square:
            // a NaN / Inf entry (or one squaring past DBL_MAX) leaves it non-finite
            if (t.nonfinite && off[e] >= 0 && idx / Q == idx % Q && !isfinite(acc[e])) atomicExch(t.nonfinite, 1);
        }
    }
    __syncthreads();
}

template <int Q>
__device__ void mid1_body(SvdTask& t, const Geo& g, double* dyn, Small& sm) {
    double* G = dyn;
    sum_partials<Q>(t, g.q, G);
    // the eigen phase (eig_body) reads the summed Gram from partial 0
    if (Q == 64 && t.nsplit > 1 && t.trunc.kind == TRUNC_FIXED && !t.gram_only)
        for (int idx = threadIdx.x; idx < Q * Q; idx += T) t.ws[(idx / Q) * kQMax + idx % Q] = G[idx];
    const bool ok = chol3<Q>(G, g.q, sm) && sm.pivmin >= 1e-6 * sm.pivmax;  // kappa beyond ~1e6: CholeskyQR2 error ~eps kappa exceeds the bar
    if (!ok) {
        if (threadIdx.x == 0) {
            sm.status = TASK_NEEDS_FALLBACK;
            sm.reason = 2;
        }
        __syncthreads();
        return;
    }
    double* dst = t.ws + ws_off_r1(t.nsplit);
    for (int idx = threadIdx.x; idx < Q * Q; idx += T) dst[(idx / Q) * kQMax + idx % Q] = G[idx];
    const bool one = sm.pivmin >= g_onepass_pivot * sm.pivmax;
    __syncthreads();
    if (threadIdx.x == 0) sm.onepass = one;
    if (one) return;  // P2 (which needs the diagonal-block inverses) is skipped
    if (t.gram_only) {  // no rows for a second pass (gram_stitch.cu): the caller redoes the task
        if (threadIdx.x == 0) {
            sm.status = TASK_NEEDS_FALLBACK;
            sm.reason = 6;
        }
        __syncthreads();
        return;
    }
    // inverses of the 16x16 diagonal blocks (back substitution per column, in
    // shared scratch: keeps this kernel's register count low for occupancy)
    double* dloc = dyn + Q * Q;  // Q x 16
    // eager order: x_l = acc_l / R_ll (the Cholesky's reciprocal), then folded
    // into every acc_i, i < l, at once (critical path 16 multiply-adds)
    if (threadIdx.x < Q) {
        const int blk = threadIdx.x / 16, c = threadIdx.x % 16, o = blk * 16;
        double* D = dloc + blk * 256;
        double acc[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = (i == c) ? 1.0 : 0.0;
#pragma unroll
        for (int l = 15; l >= 0; --l) {
            const double x = l <= c ? acc[l] * (o + l < g.q ? sm.rinv[o + l] : 1.0) : 0.0;
            D[l * 16 + c] = x;
#pragma unroll
            for (int i = 0; i < l; ++i) acc[i] = fma(-G[(o + i) * Q + o + l], x, acc[i]);
        }
    }
    __syncthreads();
    double* dv = t.ws + ws_off_dinv(t.nsplit);
    for (int idx = threadIdx.x; idx < Q * 16; idx += T) dv[idx] = dloc[idx];
}

// Leading eigenvectors of the Gram for mid-2 (storage_eig_kernel, q in (32, 64]).
// A FIXED_RANK(k) block keeps k of its q singular triplets, yet the one-sided
// Jacobi of mid-2 diagonalises all of R (q x q: ~8 sweeps of q - 1 dependent
// rounds, 65% of a cfg2 flush).  Here the kk = min(k, q) leading eigenvectors X
// of G = W^T W come from eigh_warp_top (one warp per block: tridiagonalisation
// + bisection + inverse iteration, every block of a flush resident at once) and
// mid-2 (DIRECT) only has to orthogonalise the kk columns of R X, which start
// orthogonal to the Gram's rounding: sigma, V and U keep the one-sided
// accuracy (errors ~eps sigma_1 / sigma_j relative to R), the subspace that of
// the one-pass CholeskyQR (the Gram's).  Any failed check leaves the task to
// the full mid-2.
constexpr int kDirectK = eighw::KMAX;  // most kept triplets
constexpr int kDirectLd = 24;          // row stride of X in the stage area
__device__ int g_storage_direct = 1;

template <int Q, bool DIRECT = false>
__device__ void mid2_body(SvdTask& t, const Geo& g, double* dyn, Small& sm) {
    using C3 = G3<Q>;
    double* Y = dyn;                 // G2 -> R2 (Q x Q row-major), then R^T for Jacobi (Q x JLD col-major)
    double* P = dyn + Q * C3::JLD;   // R, packed upper triangle by rows (Q (Q + 1) / 2)
    int* roff = sm.roff;             // start of packed row r
    const int q = g.q;
    const int nsp = t.nsplit;
    if (threadIdx.x < Q) roff[threadIdx.x] = threadIdx.x * Q - threadIdx.x * (threadIdx.x - 1) / 2;
    if (threadIdx.x == 0) sm.clk[0] = clock64();
    const bool one = sm.onepass;
    if (!one) sum_partials<Q>(t, q, Y);
    if (threadIdx.x == 0) sm.clk[1] = clock64();
    if (!one && (!chol3<Q>(Y, q, sm) || sm.pivmin < 0.5 || sm.pivmax > 2.0)) {
        if (threadIdx.x == 0) {
            sm.status = TASK_NEEDS_FALLBACK;
            sm.reason = 3;
        }
        __syncthreads();
        return;
    }
    double& scale = sm.scale;
    if (threadIdx.x == 0) sm.clk[2] = clock64();
    const double* R1 = t.ws + ws_off_r1(nsp);
    if (threadIdx.x == 0) {
        int e;
        frexp(R1[0], &e);
        scale = ldexp(1.0, e);  // power of two: exact scaling
    }
    __syncthreads();
    const double inv_scale = 1.0 / scale;
    // R = R2 R1 (scaled) -> P (packed; R2 is read from the Y region); after one
    // pass R = R1, written to P and (as R^T) to Y in the same sweep
    if (one) {
        for (int idx = threadIdx.x; idx < Q * Q; idx += T) {
            const int i = idx / Q, c = idx % Q;
            const double v = (c >= i && i < q && c < q) ? R1[i * kQMax + c] * inv_scale : 0.0;
            if (c >= i) P[i * Q - i * (i - 1) / 2 + c - i] = v;
            Y[i * C3::JLD + c] = v;
        }
        __syncthreads();
        if (threadIdx.x == 0) sm.clk[3] = sm.clk[4] = clock64();
    }
    for (int idx = threadIdx.x; idx < Q * Q && !one; idx += T) {
        const int i = idx / Q, c = idx % Q;
        if (c < i) continue;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        if (c < q) {
            int l = i;
            for (; l + 3 <= c; l += 4) {
                a0 = fma(Y[i * Q + l], R1[l * kQMax + c], a0);
                a1 = fma(Y[i * Q + l + 1], R1[(l + 1) * kQMax + c], a1);
                a2 = fma(Y[i * Q + l + 2], R1[(l + 2) * kQMax + c], a2);
                a3 = fma(Y[i * Q + l + 3], R1[(l + 3) * kQMax + c], a3);
            }
            for (; l <= c; ++l) a0 = fma(Y[i * Q + l], R1[l * kQMax + c], a0);
        }
        P[roff[i] + c - i] = (i < q && c < q) ? ((a0 + a1) + (a2 + a3)) * inv_scale : 0.0;
    }
    if (!one) {
        __syncthreads();
        if (threadIdx.x == 0) sm.clk[3] = clock64();
        for (int idx = threadIdx.x; idx < Q * Q; idx += T) {  // Y <- R^T (column i = row i of R)
            const int i = idx / Q, c = idx % Q;
            Y[i * C3::JLD + c] = c >= i ? P[roff[i] + c - i] : 0.0;
        }
        __syncthreads();
        if (threadIdx.x == 0) sm.clk[4] = clock64();
    }
    if (t.qr_only) {
        // W = Q R only (a trim whose truncation keeps every column, query.hpp:79-87
        // with FIXED_RANK k >= rank): Y = R^T is used as is with sigma = 1, so the
        // epilogue below yields V = vpre R^T and M = R^-1, i.e. U = W R^-1 = Q.
        // The stitch sees the part's rows R V^T, which equal the trim's
        // sigma' V'^T up to a k x k rotation that the stitch absorbs.
        if (threadIdx.x < Q) {
            sm.ord[threadIdx.x] = threadIdx.x;
            sm.sig[threadIdx.x] = inv_scale;  // x scale = 1 exactly (power of two)
        }
        if (threadIdx.x == 0) sm.k = sm.knum = q;
        __syncthreads();
    } else {
        if constexpr (DIRECT) {
            // One-sided Jacobi on the kk columns of [R X; X] (rotation angles from the top
            // half, the bottom half carried along): on exit column j is [sigma_j u_j; v_j].
            // Pairs by the circle method, 8 lanes per pair.
            constexpr int DLD = 2 * Q + 2;
            double* D = dyn + Q * C3::JLD + Q * (Q + 1) / 2;
            if (threadIdx.x == 0) sm.conv = 0;
            const int kk = t.trunc.k < q ? t.trunc.k : q;
            const int ke = kk + (kk & 1);
            const double* Xg = t.ws + ws_off_stage(nsp);
            {   // (a thread's loads of X issued together, before its stores)
                constexpr int XPT = (kDirectK * Q + T - 1) / T;
                double xv[XPT];
#pragma unroll
                for (int u = 0; u < XPT; ++u) {
                    const int idx = threadIdx.x + u * T;
                    const int j = idx / Q, r = idx % Q;
                    xv[u] = (idx < ke * Q && j < kk && r < q) ? Xg[r * kDirectLd + j] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < XPT; ++u) {
                    const int idx = threadIdx.x + u * T;
                    if (idx < ke * Q) D[(idx / Q) * DLD + Q + idx % Q] = xv[u];
                }
            }
            __syncthreads();
            for (int idx = threadIdx.x; idx < ke * Q; idx += T) {
                const int j = idx / Q, i = idx % Q;
                double a0 = 0.0, a1 = 0.0;
                if (j < kk && i < q) {
                    const double* pr = P + roff[i] - i;
                    const double* x = D + j * DLD + Q;
                    int c = i;
                    for (; c + 1 < q; c += 2) {
                        a0 = fma(pr[c], x[c], a0);
                        a1 = fma(pr[c + 1], x[c + 1], a1);
                    }
                    if (c < q) a0 = fma(pr[c], x[c], a0);
                }
                D[j * DLD + i] = a0 + a1;
            }
            __syncthreads();
            const int l8 = threadIdx.x & 7, slot = threadIdx.x >> 3;
            const double tol = (double)Q * DBL_EPSILON;
            bool conv = false;
            int sweep = 0;
            for (; sweep < 10 && !conv; ++sweep) {
                if (threadIdx.x == 0) sm.flag = 0;
                __syncthreads();
                for (int round = 0; round < ke - 1; ++round) {
                    int i = 0, j = 0;
                    bool act = slot < ke / 2;
                    if (act) {
                        const int pa = slot, pb = ke - 1 - slot;
                        i = pa == 0 ? 0 : ((pa - 1 + round) % (ke - 1)) + 1;
                        j = pb == 0 ? 0 : ((pb - 1 + round) % (ke - 1)) + 1;
                        act = i < kk && j < kk;
                    }
                    double* di = D + i * DLD;
                    double* dj = D + j * DLD;
                    double al = 0.0, be = 0.0, ga = 0.0;
                    if (act) {
#pragma unroll
                        for (int u = 0; u < Q / 8; ++u) {
                            const double x = di[l8 + 8 * u], y = dj[l8 + 8 * u];
                            al = fma(x, x, al);
                            be = fma(y, y, be);
                            ga = fma(x, y, ga);
                        }
                    }
#pragma unroll
                    for (int o = 1; o < 8; o <<= 1) {
                        al += __shfl_xor_sync(0xffffffffu, al, o);
                        be += __shfl_xor_sync(0xffffffffu, be, o);
                        ga += __shfl_xor_sync(0xffffffffu, ga, o);
                    }
                    if (act && al > 0.0 && be > 0.0 && ga * ga > tol * tol * al * be) {
                        // the angle only steers convergence (reciprocals / root from the MUFU seeds with
                        // one correction); c, s from a full-precision rsqrt keep the rotation orthogonal
                        const double zeta = 0.5 * (be - al) * eighw::rcp_nr(ga);
                        const double hz = fma(zeta, zeta, 1.0);
                        const double tt = (zeta >= 0.0 ? 1.0 : -1.0) * eighw::rcp_nr(fabs(zeta) + hz * rsqrt_nr(hz));
                        const double c = rsqrt_nr(fma(tt, tt, 1.0));
                        const double sn = c * tt;
                        // (loads first: shared-memory loads are not hoisted over earlier stores)
                        double xs[2 * Q / 8], ys[2 * Q / 8];
#pragma unroll
                        for (int u = 0; u < 2 * Q / 8; ++u) {
                            xs[u] = di[l8 + 8 * u];
                            ys[u] = dj[l8 + 8 * u];
                        }
#pragma unroll
                        for (int u = 0; u < 2 * Q / 8; ++u) {
                            di[l8 + 8 * u] = c * xs[u] - sn * ys[u];
                            dj[l8 + 8 * u] = sn * xs[u] + c * ys[u];
                        }
                        if (l8 == 0) sm.flag = 1;
                    }
                    __syncthreads();
                }
                conv = sm.flag == 0;
                __syncthreads();
                if (!conv) {
                    // a rotating sweep leaves the columns orthogonal to the square of what it met
                    // (they start at the Gram's rounding, ~1e-10): instead of a confirming sweep of
                    // ke - 1 dependent rounds every pair is tested at once, one thread per pair
                    if (threadIdx.x == 0) sm.flag = 0;
                    __syncthreads();
                    for (int pi = threadIdx.x; pi < kk * (kk - 1) / 2; pi += T) {
                        int i = 0, rem = pi;
                        while (rem >= kk - 1 - i) {
                            rem -= kk - 1 - i;
                            ++i;
                        }
                        const int j = i + 1 + rem;
                        const double* di = D + i * DLD;
                        const double* dj = D + j * DLD;
                        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll 8
                        for (int r = 0; r < Q; ++r) {
                            const double x = di[r], y = dj[r];
                            al = fma(x, x, al);
                            be = fma(y, y, be);
                            ga = fma(x, y, ga);
                        }
                        if (al > 0.0 && be > 0.0 && ga * ga > tol * tol * al * be) sm.flag = 1;
                    }
                    __syncthreads();
                    conv = sm.flag == 0;
                    __syncthreads();
                }
            }
            if (threadIdx.x == 0) sm.sweeps = sweep;
            if (!conv) {  // not expected (the columns start orthogonal to ~1e-10): the full Jacobi takes over
                if (threadIdx.x == 0) sm.conv = -1;
                __syncthreads();
                return;
            }
            // Y in mid-2's convention: column j = sigma_j v_j (the rest zero, below the rank cutoff)
            if (threadIdx.x < kk) {
                const double* dc = D + threadIdx.x * DLD;
                double n0 = 0.0, n1 = 0.0;
#pragma unroll 8
                for (int r = 0; r < Q; r += 2) {
                    n0 = fma(dc[r], dc[r], n0);
                    n1 = fma(dc[r + 1], dc[r + 1], n1);
                }
                sm.raw[threadIdx.x] = sqrt(n0 + n1);
            }
            __syncthreads();
            for (int idx = threadIdx.x; idx < Q * Q; idx += T) {
                const int j = idx / Q, c = idx % Q;
                Y[j * C3::JLD + c] = (j < kk && c < q) ? sm.raw[j] * D[j * DLD + Q + c] : 0.0;
            }
            __syncthreads();
        } else if constexpr (Q == 64) {
            jacobi_bisect64(Y, q, sm);
        } else {
            jacobi4<Q>(Y, q, sm);
        }
        if (threadIdx.x == 0) sm.clk[5] = clock64();
        sort_and_truncate(Y, C3::JLD, Q, q, t, sm, Q == 64 && !DIRECT);
        if (sm.status != TASK_OK) return;
        // After one QR pass R^T R carries the Gram's rounding (eps ||G||): the
        // kept sigma_j are accurate to c eps (sigma_1 / sigma_j)^2 (c <= 0.06
        // measured on 100 cfg2 blocks with sigma_1 / sigma_20 up to 880), inside
        // the 1e-9 bar with 10x margin while sigma_1 <= 3000 sigma_k; spread
        // retained spectra take the robust path instead.
        if (one && sm.k > 0 && sm.sig[0] > 3000.0 * sm.sig[sm.k - 1]) {
            __syncthreads();
            if (threadIdx.x == 0) {
                sm.status = TASK_NEEDS_FALLBACK;
                sm.reason = 5;
            }
            __syncthreads();
            return;
        }
    }
    const int k = sm.k;
    double* inv_sig = sm.inv_sig;
    if (threadIdx.x < k) inv_sig[threadIdx.x] = 1.0 / sm.sig[threadIdx.x];
    __syncthreads();
    // ---- A's V (tall) or A's U (wide): V_W = Y S^-1
    if (g.tall && !t.vpre) {
        // canonical_sign (svd.hpp:179-203) decided on Y in shared memory (V_W =
        // Y S^-1 scales columns by positive numbers: same pivot), then V written once
        if (t.sign) {
            for (int c = warp_id(); c < k; c += NWARPS) {
                const double* y = Y + sm.ord[c] * C3::JLD;
                double best = -1.0;
                int idx = 0x7fffffff;
                for (int r = threadIdx.x & 31; r < q; r += 32) {
                    const double mag = fabs(y[r]);
                    if (mag > best) {
                        best = mag;
                        idx = r;
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
                    if (ob > best || (ob == best && oi < idx)) {
                        best = ob;
                        idx = oi;
                    }
                }
                if ((threadIdx.x & 31) == 0) sm.sgn[c] = (q > 0 && y[idx] < 0.0) ? -1.0 : 1.0;
            }
        } else if (threadIdx.x < k) {
            sm.sgn[threadIdx.x] = 1.0;
        }
        __syncthreads();
        for (int idx = threadIdx.x; idx < q * k; idx += T) {
            const int a = idx / k, r = idx % k;
            t.v[(int64_t)a * t.ldv + r] = Y[sm.ord[r] * C3::JLD + a] * (inv_sig[r] * sm.sgn[r]);
        }
        __syncthreads();
    } else if (g.tall) {
        const int nv = t.vpre ? t.nvpre : q;
        for (int idx = threadIdx.x; idx < nv * k; idx += T) {
            const int a = idx / k, r = idx % k;
            const double* y = Y + sm.ord[r] * C3::JLD;
            double acc;
            if (t.vpre) {
                acc = 0.0;
                const double* pre = t.vpre + (int64_t)a * t.ldvpre;
                if (t.vscale)
                    for (int j = 0; j < q; ++j) acc = fma(pre[j] * t.vscale[j], y[j], acc);
                else
                    for (int j = 0; j < q; ++j) acc = fma(pre[j], y[j], acc);
                acc *= inv_sig[r];
            } else {
                acc = y[a] * inv_sig[r];
            }
            t.v[(int64_t)a * t.ldv + r] = acc;
        }
        __syncthreads();
        if (t.sign) {
            canonical_sign_global(t.v, t.ldv, nv, k, sm);
        } else {
            if (threadIdx.x < k) sm.sgn[threadIdx.x] = 1.0;
            __syncthreads();
        }
    } else {
        for (int idx = threadIdx.x; idx < q * k; idx += T) {
            const int a = idx / k, r = idx % k;
            t.u[(int64_t)a * t.ldu + r] = Y[sm.ord[r] * C3::JLD + a] * inv_sig[r];
        }
        if (threadIdx.x < k) sm.sgn[threadIdx.x] = 1.0;
        __syncthreads();
    }
    if (threadIdx.x == 0) sm.clk[6] = clock64();
    // ---- M_k with U_W = W M_k.  Well-separated spectra (sigma_1 <= 1000
    // sigma_k, not a QR-only trim): M_k = V_k Sigma_k^-1 = Y_k Sigma_k^-2, no
    // solves (U's orthogonality loss is ~eps sigma_1 / sigma_k, measured
    // <= 2e-14 on the BASELINE blocks; the check phase still enforces 1e-10).
    if (!t.qr_only && k > 0 && sm.sig[0] <= g_nosolve_ratio * sm.sig[k - 1]) {
        double* mg = t.ws + ws_off_m(nsp);
        for (int idx = threadIdx.x; idx < Q * Q; idx += T) {
            const int l = idx / Q, r = idx % Q;
            mg[l * kQMax + r] = (r < k && l < q)
                                    ? Y[sm.ord[r] * C3::JLD + l] * (inv_sig[r] * inv_sig[r]) * inv_scale * sm.sgn[r]
                                    : 0.0;
        }
    } else {
        // Otherwise J_k = R^-T Y_k (forward substitution), then M_k = R^-1 J_k (back
        // substitution), all k columns at once, in place in Y's columns ord[0..k).
        // 8-row blocks: one thread per column solves the diagonal block in
        // registers in eager order with the reciprocals of R's diagonal (no
        // divisions on the chain), then a (column, row-group) grid updates the rows
        // beyond it with two accumulator chains.
        double* rr = sm.rinv;  // 1 / R_jj (chol3's values are dead by now)
        if (threadIdx.x < q) rr[threadIdx.x] = 1.0 / P[roff[threadIdx.x]];
        __syncthreads();
        for (int o = 0; o < q; o += 8) {
            const int w = min(8, q - o);
            for (int r = threadIdx.x; r < k; r += T) {
                double* y = Y + sm.ord[r] * C3::JLD;
                double x[8];
    #pragma unroll
                for (int j = 0; j < 8; ++j) x[j] = j < w ? y[o + j] : 0.0;
    #pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (i < w) {
                        x[i] *= rr[o + i];
    #pragma unroll
                        for (int j = i + 1; j < 8; ++j)
                            if (j < w) x[j] = fma(-P[roff[o + i] + j - i], x[i], x[j]);
                    }
                }
    #pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < w) y[o + j] = x[j];
            }
            __syncthreads();
            for (int c = threadIdx.x & 31; c < k; c += 32) {
                double* y = Y + sm.ord[c] * C3::JLD;
                for (int l = o + w + (threadIdx.x >> 5); l < q; l += NWARPS) {
                    double a0 = y[l], a1 = 0.0;
    #pragma unroll
                    for (int i = 0; i < 8; i += 2) {
                        if (i < w) a0 = fma(-P[roff[o + i] + l - o - i], y[o + i], a0);
                        if (i + 1 < w) a1 = fma(-P[roff[o + i + 1] + l - o - i - 1], y[o + i + 1], a1);
                    }
                    y[l] = a0 + a1;
                }
            }
            __syncthreads();
        }
        for (int o = ((q - 1) / 8) * 8; o >= 0; o -= 8) {
            const int w = min(8, q - o);
            for (int r = threadIdx.x; r < k; r += T) {
                double* y = Y + sm.ord[r] * C3::JLD;
                double x[8];
    #pragma unroll
                for (int j = 0; j < 8; ++j) x[j] = j < w ? y[o + j] : 0.0;
    #pragma unroll
                for (int i = 7; i >= 0; --i) {
                    if (i < w) {
                        x[i] *= rr[o + i];
    #pragma unroll
                        for (int j = 0; j < i; ++j) x[j] = fma(-P[roff[o + j] + i - j], x[i], x[j]);
                    }
                }
    #pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < w) y[o + j] = x[j];
            }
            __syncthreads();
            for (int c = threadIdx.x & 31; c < k; c += 32) {
                double* y = Y + sm.ord[c] * C3::JLD;
                for (int l = threadIdx.x >> 5; l < o; l += NWARPS) {
                    double a0 = y[l], a1 = 0.0;
    #pragma unroll
                    for (int i = 0; i < 8; i += 2) {
                        if (i < w) a0 = fma(-P[roff[l] + o + i - l], y[o + i], a0);
                        if (i + 1 < w) a1 = fma(-P[roff[l] + o + i + 1 - l], y[o + i + 1], a1);
                    }
                    y[l] = a0 + a1;
                }
            }
            __syncthreads();
        }
        // M (Q x Q row-major at ld kQMax, zero beyond q x k); undo the R scaling
        double* mg = t.ws + ws_off_m(nsp);
        for (int idx = threadIdx.x; idx < Q * Q; idx += T) {
            const int l = idx / Q, r = idx % Q;
            mg[l * kQMax + r] = (r < k && l < q) ? Y[sm.ord[r] * C3::JLD + l] * inv_scale * sm.sgn[r] : 0.0;
        }
    }
    double* sg = t.ws + ws_off_sig(nsp);
    if (threadIdx.x < k) sg[threadIdx.x] = sm.sig[threadIdx.x] * scale;
    __syncthreads();
    if (threadIdx.x == 0) sm.clk[7] = clock64();
}

template <int Q>
__device__ void check_body(SvdTask& t, const Geo& g, double* dyn, Small& sm) {
    double* G = dyn;
    const int q = g.q, k = t.krank;
    sum_partials<Q>(t, k, G);
    if (threadIdx.x == 0) sm.flag = 0;
    __syncthreads();
    // U_W orthonormality (the svd.hpp:25 contract, 1e-10); else the robust path
    for (int idx = threadIdx.x; idx < k * k; idx += T) {
        const int i = idx / k, c = idx % k;
        if (fabs(G[i * Q + c] - (i == c ? 1.0 : 0.0)) > kOrthonormalityTol) sm.flag = 1;
    }
    __syncthreads();
    if (sm.flag) {
        if (threadIdx.x == 0) {
            sm.status = TASK_NEEDS_FALLBACK;
            sm.reason = 4;
        }
        __syncthreads();
        return;
    }
    if (!g.tall && k > 0) {
        const int p = g.p;
        const int nv = t.vpre ? t.nvpre : p;
        if (t.vpre) {
            const double* st = t.ws + ws_off_stage(t.nsplit);
            for (int idx = threadIdx.x; idx < nv * k; idx += T) {
                const int a = idx / k, r = idx % k;
                const double* pre = t.vpre + (int64_t)a * t.ldvpre;
                double acc = 0.0;
                for (int j = 0; j < p; ++j) acc = fma(pre[j], st[j * kQMax + r], acc);
                t.v[(int64_t)a * t.ldv + r] = acc;
            }
            __syncthreads();
        }
        if (t.sign) {
            canonical_sign_global(t.v, t.ldv, nv, k, sm);
            for (int idx = threadIdx.x; idx < q * k; idx += T) {
                const int a = idx / k, r = idx % k;
                if (sm.sgn[r] < 0.0) t.u[(int64_t)a * t.ldu + r] = -t.u[(int64_t)a * t.ldu + r];
            }
        }
    }
    const double* sg = t.ws + ws_off_sig(t.nsplit);
    if (threadIdx.x < k) t.s[threadIdx.x] = sg[threadIdx.x];
    if (threadIdx.x == 0) *t.k_out = (double)k;
    __syncthreads();
}

template <int QF, int KIND>  // KIND: 1, 2, 3 pass; 11 mid1; 12 mid2; 13 check; 14 eigen; 15 mid2 direct
__device__ __forceinline__ void run_phase(SvdTask* tasks, int ti, int split, double* dyn, Small& sm) {
    SvdTask t = tasks[ti];
    const Geo g = geometry(t);
    if (KIND == 12 && t.direct == 2) return;  // finished by the direct mid-2
    if (KIND == 15 && t.direct != 1) return;
    if (KIND <= 3) {
        if (t.status != TASK_OK || g.m == 0 || g.n == 0 || g.q > kQMax) return;
        if (KIND == 2 && t.onepass) return;
    } else {
        if (threadIdx.x == 0) {
            sm.onepass = KIND == 11 ? 0 : t.onepass;
            sm.status = t.status;
            sm.reason = t.reason;
            sm.sweeps = t.sweeps;
            for (int i = 0; i < 8; ++i) sm.clk[i] = t.clk[i];
            sm.m = g.m;
            sm.n = g.n;
            sm.p = g.p;
            sm.q = g.q;
            sm.tall = g.tall;
            sm.k = 0;
        }
        __syncthreads();
        if (KIND == 11) {
            if (g.m == 0 || g.n == 0) {
                if (threadIdx.x == 0) *t.k_out = 0.0;
                return;
            }
            if (g.q > kQMax) {
                if (threadIdx.x == 0) tasks[ti].status = TASK_UNSUPPORTED;
                return;
            }
        }
        if (sm.status != TASK_OK || g.m == 0 || g.n == 0) return;
    }
#define ZSVD_DISPATCH(BODY)      \
    if constexpr (QF == 16) {    \
        BODY(16);                \
    } else if constexpr (QF == 32) { \
        BODY(32);                \
    } else if constexpr (QF == 64) { \
        BODY(64);                \
    } else {                     \
        if (g.q <= 16) BODY(16); \
        else if (g.q <= 32) BODY(32); \
        else BODY(64);           \
    }
    if constexpr (KIND <= 3) {
#define ZSVD_PASS(QQ) slab_pass<QQ, KIND>(t, g, split, dyn)
        ZSVD_DISPATCH(ZSVD_PASS)
#undef ZSVD_PASS
    } else {
        if constexpr (KIND == 11) {
#define ZSVD_M1(QQ) mid1_body<QQ>(t, g, dyn, sm)
            ZSVD_DISPATCH(ZSVD_M1)
#undef ZSVD_M1
        } else if constexpr (KIND == 15) {
            mid2_body<64, true>(t, g, dyn, sm);
            if (threadIdx.x == 0 && sm.conv == -1) tasks[ti].direct = 0;  // declined: the full mid-2 runs
            if (sm.conv == -1) return;
            if (threadIdx.x == 0) {
                tasks[ti].direct = 2;
                if (sm.status == TASK_OK) atomicAdd(&g_direct_tasks, 1ull);
            }
        } else if constexpr (KIND == 12) {
#define ZSVD_M2(QQ) mid2_body<QQ>(t, g, dyn, sm)
            ZSVD_DISPATCH(ZSVD_M2)
#undef ZSVD_M2
        } else {
#define ZSVD_C(QQ) check_body<QQ>(t, g, dyn, sm)
            ZSVD_DISPATCH(ZSVD_C)
#undef ZSVD_C
        }
        if (threadIdx.x == 0) {
            tasks[ti].status = sm.status;
            tasks[ti].reason = sm.reason;
            tasks[ti].sweeps = sm.sweeps;
            if (KIND == 11) tasks[ti].onepass = sm.onepass;
            if (KIND == 12 || KIND == 15) tasks[ti].krank = sm.status == TASK_OK ? sm.k : 0;
            for (int i = 0; i < 8; ++i) tasks[ti].clk[i] = sm.clk[i];
        }
    }
#undef ZSVD_DISPATCH
}

template <int Q>
constexpr int smem_pass(int phase) {
    using S = SlabG<Q>;
    return 8 * (S::STAGE + (phase == 2 ? Q * S::MLD + Q * S::DLD : phase == 3 ? Q * S::MLD : 0));
}
template <int Q>
constexpr int smem_mid() {  // R^T (Q x JLD) + packed R; three CTAs per SM at Q = 64
    return 8 * (Q * G3<Q>::JLD + Q * (Q + 1) / 2);
}

}  // namespace

// ---------------------------------------------------------------- kernels
// Resident CTAs per SM each phase is compiled for (register cap 65536 /
// (256 x this)); P2 and P3 are held to 2 by their shared memory anyway.
#ifndef ZSVD_M2_CTAS
#define ZSVD_M2_CTAS 3
#endif
template <int KIND>
constexpr int phase_min_blocks() {
    return (KIND == 1 || KIND == 2 || KIND == 3 || KIND == 15) ? 2 : (KIND == 12 ? ZSVD_M2_CTAS : 3);
}

template <int QF, int KIND>
__global__ void __launch_bounds__(kEngineThreads, phase_min_blocks<KIND>()) svd_phase_kernel(SvdTask* tasks, int ntasks) {
    ZSVD_PDL_WAIT();
    extern __shared__ __align__(16) double dyn[];
    __shared__ Small sm;
    const int ti = blockIdx.y;
    if (ti >= ntasks) return;
    if (KIND <= 3 && (int)blockIdx.x >= tasks[ti].nsplit) return;
    run_phase<QF, KIND>(tasks, ti, blockIdx.x, dyn, sm);
}

#define ZSVD_INST(QF)                                              \
    template __global__ void svd_phase_kernel<QF, 1>(SvdTask*, int);  \
    template __global__ void svd_phase_kernel<QF, 2>(SvdTask*, int);  \
    template __global__ void svd_phase_kernel<QF, 3>(SvdTask*, int);  \
    template __global__ void svd_phase_kernel<QF, 11>(SvdTask*, int); \
    template __global__ void svd_phase_kernel<QF, 12>(SvdTask*, int); \
    template __global__ void svd_phase_kernel<QF, 13>(SvdTask*, int);
ZSVD_INST(0)
ZSVD_INST(16)
ZSVD_INST(32)
ZSVD_INST(64)
#undef ZSVD_INST
template __global__ void svd_phase_kernel<64, 15>(SvdTask*, int);

// Eigen phase of the storage flush (between mid-1 and mid-2; grid: tasks, one
// warp each): X = the leading eigenvectors of the block's Gram into the stage
// area, task.direct = 1; any ineligible task or failed check leaves direct = 0.
__device__ long long g_eig_clk[8];  // task 0's phase stamps (diagnostics)
__global__ void __launch_bounds__(32) storage_eig_kernel(SvdTask* tasks, int ntasks) {
    ZSVD_PDL_WAIT();
    extern __shared__ __align__(16) double dyn[];
    const int ti = blockIdx.x;
    if (ti >= ntasks) return;
    const SvdTask t = tasks[ti];
    const int lane = threadIdx.x;
    if (lane == 0) tasks[ti].direct = 0;
    if (t.status != TASK_OK) return;
    const Geo g = geometry(t);
    const int q = g.q;
    if (g.m == 0 || g.n == 0 || q > kQMax) return;
    const int kk = t.trunc.k < q ? t.trunc.k : q;
    if (!(g_storage_direct && t.onepass && t.trunc.kind == TRUNC_FIXED && kk >= 1 && kk <= kDirectK && q > 32 &&
          2 * kk <= q && g.tall && !t.qr_only && !t.gram_only && !t.vpre))
        return;
    const double* G = t.ws;  // summed by mid-1 (ld kQMax)
    double mx = 0.0;
    for (int i = lane; i < q; i += 32) mx = fmax(mx, G[i * kQMax + i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (!(mx > 0.0 && mx < 1e300)) return;
    int e2 = 0;
    frexp(mx, &e2);
    const double scale = ldexp(1.0, -e2);
    if (eighw::eigh_warp_top(G, kQMax, q, kk, scale, dyn, t.ws + ws_off_stage(t.nsplit), kDirectLd,
                             ti == 0 ? g_eig_clk : nullptr))
        return;
    __syncwarp();
    if (lane == 0) tasks[ti].direct = 1;
}
int storage_eig_smem_bytes() { return eighw::bytes(); }

// Dynamic shared memory of a phase kernel (QF = 0 sizes for Q = 64).
int phase_smem_bytes(int qf, int kind) {
    const int q = qf == 0 ? 64 : qf;
    auto pick = [&](auto tag) {
        constexpr int QQ = decltype(tag)::value;
        if (kind <= 3) return smem_pass<QQ>(kind);
        if (kind == 15) return smem_mid<QQ>() + 8 * (kDirectK * (2 * QQ + 2));
        if (kind == 13) return 8 * QQ * QQ;
        if (kind == 11) return 8 * (QQ * QQ + QQ * 16);
        return smem_mid<QQ>();
    };
    if (q == 16) return pick(std::integral_constant<int, 16>());
    if (q == 32) return pick(std::integral_constant<int, 32>());
    return pick(std::integral_constant<int, 64>());
}

int64_t workspace_doubles(int nsplit) { return ws_total(nsplit); }

// ---------------------------------------------------------------- fused QR trims
// Both boundary trims of a range query (query.hpp:64-89) in one launch, one CTA
// per trim, when the trim's truncation keeps every column (FIXED_RANK k >= the
// block's rank capacity, capacity <= 32; SvdTask::qr_only form).  The slice
// rows U_s of the block's U (m x n) are orthonormal columns cut short, so one
// CholeskyQR pass is exact to ~eps kappa(U_s)^2:
//   G = U_s^T U_s (DMMA, eight warps over row strips, partials summed in warp
//   order), R = chol(G), X = R^-1 (per-column eager back substitution),
//   U = U_s X (the part's Q), V = vpre diag(sigma) R^T, sigma = 1, k = n,
// so the stack rows of the part are R Sigma V^T.  A slice whose pivots spread
// beyond 100x (short or rank-deficient slices), or with fewer rows than the
// rank, takes the full trim SVD in the same CTA (one-sided Jacobi in global
// scratch, the fallback kernel's path), i.e. the reference semantics.
constexpr int kTrimQ = 32;
constexpr double kTrimPivot = 1e-2;
constexpr int kTrimCluster = 8;              // CTAs per trim (one thread-block cluster)
constexpr int kTrimRowBytes = 131072;        // slice rows per CTA, staged whole

int trim_qr_smem_bytes() { return 8 * (3 * kTrimQ * kTrimQ) + kTrimRowBytes; }
int trim_qr_cluster() { return kTrimCluster; }
int trim_qr_row_bytes() { return kTrimRowBytes; }

namespace {
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// Generic address of the same shared-memory object in cluster CTA `rank` (DSMEM).
template <class P>
__device__ __forceinline__ P* cluster_peer(P* p, unsigned rank) {
    unsigned long long out;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(reinterpret_cast<unsigned long long>(p)), "r"(rank));
    return reinterpret_cast<P*>(out);
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// Robust trim (the fallback kernel's path): one-sided Jacobi on W = U_s Sigma
// in global scratch, truncation and the 1e-12 cutoff as the reference.
__device__ void trim_robust(SvdTask t, double* W, int64_t slot_doubles, Small& sm) {  // (t by value)
    if (t.qr_only) {
        t.qr_only = 0;
        t.colscale = t.vscale;
        t.vscale = nullptr;
    }
    if (!setup(t, sm)) return;
    if (threadIdx.x == 0) atomicAdd(&g_fallback_tasks, 1ull);
    const int p = sm.p, q = sm.q;
    if ((int64_t)p * q + q * q > slot_doubles) return;  // sized by the host: cannot happen
    double* V = W + (int64_t)p * q;
    for (int64_t idx = threadIdx.x; idx < (int64_t)p * q; idx += T) {
        const int i = (int)(idx % p), j = (int)(idx / p);
        W[(int64_t)j * p + i] = w_at(t, sm.tall, i, j);
    }
    __syncthreads();
    jacobi(W, p, p, q, V, sm);
    finish_from_jacobi(t, W, p, V, sm);
}
}  // namespace

// Fused QR-form trims: cluster y = trim y, CTA r of the cluster owns rows
// [r m / 8, (r + 1) m / 8) of the slice.  Each CTA stages its rows in shared
// memory with one bulk copy (TMA), forms its partial Gram on DMMA; CTA 0 sums
// the eight partials through distributed shared memory, factors R, forms
// X = R^-1 and V; every CTA then reads X from CTA 0 and writes its rows of
// Q = U_s X.  A pivot spread beyond 100x, or fewer rows than the rank, makes
// CTA 0 take the full trim SVD alone (reference semantics).  CTA 0 leaves
// clock64 deltas of its stages in tasks[].clk (ZSVD_DEBUG prints them).
__global__ void __cluster_dims__(kTrimCluster, 1, 1) __launch_bounds__(kEngineThreads)
    trim_qr_kernel(SvdTask* tasks, int ntasks, double* scratch, int64_t slot_doubles) {
    ZSVD_PDL_WAIT();
    constexpr int Q = kTrimQ;
    extern __shared__ __align__(16) double dyn[];
    __shared__ Small sm;
    __shared__ __align__(8) uint64_t bar;
    __shared__ int fast_ok;
    const int ti = blockIdx.y;
    const unsigned rank = cluster_rank();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* Gw = dyn;                 // this CTA's partial Gram, then (CTA 0) G / R
    double* X = dyn + Q * Q;          // R^-1
    double* Wt = dyn + 2 * Q * Q;     // per-warp scratch (sum of the warps' tiles)
    double* rowsbuf = dyn + 3 * Q * Q;
    SvdTask t = tasks[ti];
    const int m = t.m_from ? t.m_from[0] : t.m;
    const int n = t.n_from ? (int)t.n_from[0] : t.n;
    const bool aligned = (t.lda % 2 == 0) && ((reinterpret_cast<uintptr_t>(t.a) & 15) == 0);
    // uniform over the cluster (all CTAs read the same task)
    const bool try_fast = t.qr_only && aligned && m >= n && n >= 1 && n <= Q &&
                          (int64_t)((m + kTrimCluster - 1) / kTrimCluster) * t.lda * 8 <= kTrimRowBytes;
    if (!try_fast) {
        if (rank == 0) {
            if (m == 0 || n == 0) {  // a rank-0 block trims to empty factors (query.hpp:74-76)
                if (threadIdx.x == 0) *t.k_out = 0.0;
            } else {
                trim_robust(t, scratch + (int64_t)ti * slot_doubles, slot_doubles, sm);
            }
        }
        return;  // no DSMEM traffic on this path
    }
    // ---- stage this CTA's rows (one bulk copy)
    const int per = (m + kTrimCluster - 1) / kTrimCluster;
    const int r0 = min(m, (int)rank * per), r1 = min(m, r0 + per);
    const int rows = r1 - r0;
    const int64_t lda = t.lda;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    long long ck0 = clock64();
    if (threadIdx.x == 0 && rows > 0) {
        const unsigned bytes = (unsigned)(rows * lda * 8);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(rowsbuf)),
            "l"(t.a + (int64_t)r0 * lda), "r"(bytes), "r"(smem_u32(&bar))
            : "memory");
    }
    if (rows > 0)
        asm volatile(
            "{\n .reg .pred p;\n TQW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra TQW_%=;\n}" ::"r"(
                smem_u32(&bar))
            : "memory");
    long long ck1 = clock64();
    // ---- partial Gram of the staged rows (DMMA, upper 8x8 tiles); columns >= n
    // read neighbouring data and only feed entries that are never used
    {
        double c[10][2];
#pragma unroll
        for (int i = 0; i < 10; ++i) c[i][0] = c[i][1] = 0.0;
        const int col = lane >> 2, kk = lane & 3;
        const int full = rows & ~3;
        for (int k0 = 4 * warp; k0 < rows; k0 += 4 * NWARPS) {
            const int row = k0 + kk;
            double x[4];
            if (k0 < full) {
#pragma unroll
                for (int T4 = 0; T4 < 4; ++T4) x[T4] = rowsbuf[row * lda + 8 * T4 + col];
            } else {
#pragma unroll
                for (int T4 = 0; T4 < 4; ++T4) x[T4] = row < rows ? rowsbuf[row * lda + 8 * T4 + col] : 0.0;
            }
            int tt = 0;
#pragma unroll
            for (int I = 0; I < 4; ++I)
#pragma unroll
                for (int J = I; J < 4; ++J, ++tt) dmma(c[tt][0], c[tt][1], x[I], x[J]);
        }
        // sum the warps' tiles in warp order (deterministic): warp w adds into Wt in turn
        for (int w = 0; w < NWARPS; ++w) {
            if (warp == w) {
                int tt = 0;
#pragma unroll
                for (int I = 0; I < 4; ++I)
#pragma unroll
                    for (int J = I; J < 4; ++J, ++tt) {
                        const int r = 8 * I + (lane >> 2), cc = 8 * J + 2 * (lane & 3);
                        Wt[r * Q + cc] = (w == 0 ? 0.0 : Wt[r * Q + cc]) + c[tt][0];
                        Wt[r * Q + cc + 1] = (w == 0 ? 0.0 : Wt[r * Q + cc + 1]) + c[tt][1];
                    }
            }
            __syncthreads();
        }
        for (int idx = threadIdx.x; idx < Q * Q; idx += T) Gw[idx] = Wt[idx];
    }
    long long ck2 = clock64();
    cluster_sync_all();  // every CTA's partial Gram is visible
    long long ck3 = clock64(), ck4 = 0, ck5 = 0, ck6 = 0;
    if (rank == 0) {
        // G = sum of the cluster's partials in rank order (upper, live part); all
        // eight remote loads of an entry are in flight together
        const double* peer[kTrimCluster];
#pragma unroll
        for (unsigned q = 0; q < kTrimCluster; ++q) peer[q] = cluster_peer(Gw, q);
        for (int idx = threadIdx.x; idx < Q * Q; idx += T) {
            const int r = idx / Q, cc = idx % Q;
            double acc = 0.0;
            if (cc >= r && r < n && cc < n) {
                double v[kTrimCluster];
#pragma unroll
                for (unsigned q = 0; q < kTrimCluster; ++q) v[q] = peer[q][idx];
#pragma unroll
                for (unsigned q = 0; q < kTrimCluster; ++q) acc += v[q];
            }
            Wt[idx] = acc;
        }
        __syncthreads();
        double* G = Wt;
        ck4 = clock64();
        const bool ok = chol3<Q>(G, n, sm) && sm.pivmin >= kTrimPivot * sm.pivmax;
        ck5 = clock64();
        if (threadIdx.x == 0) fast_ok = ok;
        if (ok) {
            // Z = diag(sigma) R^T in Gw (this CTA's partial is consumed)
            for (int idx = threadIdx.x; idx < Q * Q; idx += T) {
                const int r = idx / Q, c2 = idx % Q;
                Gw[c2 * Q + r] = (r < n && c2 < n) ? t.vscale[c2] * G[idx] : 0.0;  // Z[j = c2][r]
            }
            __syncthreads();
            // X = R^-1 by columns, 8 lanes per column j: lane g owns rows i = g (mod 8);
            // x_l = acc_l / R_ll comes from its owner by a shuffle, then every lane
            // folds it into its rows (eager back substitution, 32 short steps)
            {
                const int j = threadIdx.x >> 3, g8 = threadIdx.x & 7;
                const int base = (threadIdx.x & 31) & ~7;
                double acc[Q / 8];
#pragma unroll
                for (int s2 = 0; s2 < Q / 8; ++s2) acc[s2] = (g8 + 8 * s2 == j) ? 1.0 : 0.0;
#pragma unroll
                for (int l = Q - 1; l >= 0; --l) {
                    double xl = (g8 == (l & 7) && l <= j && j < n) ? acc[l >> 3] * sm.rinv[l] : 0.0;
                    xl = __shfl_sync(0xffffffffu, xl, base + (l & 7));
                    if (g8 == (l & 7)) X[l * Q + j] = xl;
#pragma unroll
                    for (int s2 = 0; s2 < Q / 8; ++s2) {
                        const int i = g8 + 8 * s2;
                        if (i < l) acc[s2] = fma(-G[i * Q + l], xl, acc[s2]);
                    }
                }
            }
            // V = vpre Z: thread (row a, quarter of the outputs), the row of vpre
            // loaded once into registers (one memory latency per row)
            const int nv = t.nvpre;
            for (int it = threadIdx.x; it < nv * 4; it += T) {
                const int aa = it >> 2, qq = it & 3;
                const double* pre = t.vpre + (int64_t)aa * t.ldvpre;
                double pr[Q];
#pragma unroll
                for (int j = 0; j < Q; ++j) pr[j] = j < n ? pre[j] : 0.0;
                for (int r = qq; r < n; r += 4) {
                    double a0 = 0.0, a1 = 0.0;
#pragma unroll
                    for (int j = 0; j < Q; j += 2) {
                        a0 = fma(pr[j], Gw[j * Q + r], a0);
                        a1 = fma(pr[j + 1], Gw[(j + 1) * Q + r], a1);
                    }
                    t.v[(int64_t)aa * t.ldv + r] = a0 + a1;
                }
            }
            if (threadIdx.x < n) t.s[threadIdx.x] = 1.0;
            if (threadIdx.x == 0) *t.k_out = (double)n;
        }
        __syncthreads();
        ck6 = clock64();
    }
    cluster_sync_all();  // X and the decision are visible
    long long ck7 = clock64();
    const int* okp = cluster_peer(&fast_ok, 0);
    const bool ok = *okp != 0;
    if (ok) {
        const double* X0 = cluster_peer(X, 0);
        const double* Xs = X;
        if (rank != 0) {
            for (int idx = threadIdx.x; idx < Q * Q; idx += T) Wt[idx] = X0[idx];
            Xs = Wt;
        }
        __syncthreads();
        // rows of U = U_s X on DMMA: warp w takes 8-row tiles w, w + 8, ...
        const int nks = (n + 3) / 4;
        for (int r8 = 8 * warp; r8 < rows; r8 += 8 * NWARPS) {
            double cc[4][2];
#pragma unroll
            for (int J = 0; J < 4; ++J) cc[J][0] = cc[J][1] = 0.0;
            const int arow = r8 + (lane >> 2);
            for (int ks = 0; ks < nks; ++ks) {
                const int kc = 4 * ks + (lane & 3);
                const double av = (arow < rows && kc < n) ? rowsbuf[arow * lda + kc] : 0.0;
#pragma unroll
                for (int J = 0; J < 4; ++J) dmma(cc[J][0], cc[J][1], av, Xs[kc * Q + 8 * J + (lane >> 2)]);
            }
            if (arow < rows) {
                double* out = t.u + (int64_t)(r0 + arow) * t.ldu;
#pragma unroll
                for (int J = 0; J < 4; ++J) {
                    const int col0 = 8 * J + 2 * (lane & 3);
                    if (col0 < n) out[col0] = cc[J][0];
                    if (col0 + 1 < n) out[col0 + 1] = cc[J][1];
                }
            }
        }
    }
    cluster_sync_all();  // CTA 0's shared memory stays alive until every peer is done
    if (rank == 0 && threadIdx.x == 0) {
        int64_t* ck = tasks[ti].clk;
        ck[0] = ck1 - ck0; ck[1] = ck2 - ck1; ck[2] = ck3 - ck2; ck[3] = ck4 - ck3;
        ck[4] = ck5 - ck4; ck[5] = ck6 - ck5; ck[6] = ck7 - ck6; ck[7] = clock64() - ck7;
    }
    if (!ok && rank == 0) trim_robust(t, scratch + (int64_t)ti * slot_doubles, slot_doubles, sm);
}

// Re-does flagged tasks by one-sided Jacobi on W in global scratch.  Grid-stride
// over tasks; CTA b owns scratch slot b (slot_doubles each).
__global__ void __launch_bounds__(kEngineThreads) svd_fallback_kernel(SvdTask* tasks, int ntasks,
                                                                      double* scratch,
                                                                      int64_t slot_doubles) {
    ZSVD_PDL_WAIT();
    __shared__ Small sm;
    // the usual launch has nothing flagged: the CTA's tasks are probed in parallel (one
    // per thread) instead of one dependent global load per task, and the CTA leaves
    {
        int any = 0;
        for (int ti = blockIdx.x + (int)gridDim.x * (int)threadIdx.x; ti < ntasks; ti += (int)gridDim.x * T)
            any |= tasks[ti].status == TASK_NEEDS_FALLBACK;
        if (!__syncthreads_or(any)) return;
    }
    for (int ti = blockIdx.x; ti < ntasks; ti += gridDim.x) {
        if (tasks[ti].status != TASK_NEEDS_FALLBACK) continue;
        if (threadIdx.x == 0) atomicAdd(&g_fallback_tasks, 1ull);
        __syncthreads();
        SvdTask t = tasks[ti];
        if (t.qr_only) {  // the fast QR of a trim failed: the full trim SVD instead
            t.qr_only = 0;
            t.colscale = t.vscale;
            t.vscale = nullptr;
        }
        if (!setup(t, sm)) continue;
        const int p = sm.p, q = sm.q;
        if ((int64_t)p * q + q * q > slot_doubles) {
            if (threadIdx.x == 0) tasks[ti].status = TASK_CAPACITY;
            continue;
        }
        double* W = scratch + (int64_t)blockIdx.x * slot_doubles;
        double* V = W + (int64_t)p * q;
        for (int64_t idx = threadIdx.x; idx < (int64_t)p * q; idx += T) {
            int i = (int)(idx % p), j = (int)(idx / p);
            W[(int64_t)j * p + i] = w_at(t, sm.tall, i, j);
        }
        __syncthreads();
        jacobi(W, p, p, q, V, sm);
        finish_from_jacobi(t, W, p, V, sm);
        if (threadIdx.x == 0) tasks[ti].status = sm.status == TASK_OK ? TASK_DONE_FALLBACK : sm.status;
        __syncthreads();
    }
}

}  // namespace zsvd
