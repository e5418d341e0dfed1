// svd_engine.cu — batched fp64 thin SVD for sm_100a (one CTA per matrix).
//
// Replaces the Eigen call sites of the reference hot path:
// thin_svd (svd.hpp:90-131: JacobiSVD / BDCSVD + 1e-12 rank cutoff),
// truncate_rank (svd.hpp:135-164), canonical_sign (svd.hpp:179-203), and the
// small products fused around them in trim_block (query.hpp:79-87).
//
// Work matrix W (p x q, p >= q): W = A when m >= n, W = A^T otherwise, q <= 64.
//   direct path  (W fits shared memory, p small): one-sided Hestenes Jacobi on W
//                with V accumulated; U = normalised columns.
//   tall path    (p large, W = A): never holds W on chip.  Streams row chunks
//                through shared memory three times:
//                  pass 1  G  = W^T W                       (register-tiled Gram)
//                  chol    G  = R1^T R1
//                  pass 2  G2 = (W R1^-1)^T (W R1^-1)        (blocked TRSM + Gram)
//                  chol    G2 = R2^T R2,  R = R2 R1          (CholeskyQR2)
//                  jacobi  R V = U_R S                       (one-sided, in smem)
//                  pass 3  U = (W R^-1) U_R                  (TRSM + GEMM, streamed out)
//                CholeskyQR2 is backward stable for kappa(A) << eps^-1/2; blocks
//                whose Cholesky pivots say otherwise, or whose final U is not
//                orthonormal to 1e-10, are re-done by the fallback kernel.
//   fallback     one-sided Jacobi on W copied to global scratch (rank-deficient
//                or ill-conditioned blocks, exact zero blocks).
// All reductions use a fixed order, so results are bitwise reproducible.
#include <cfloat>
#include <cstdint>

#include "zsvd_internal.h"

namespace zsvd {

// Tasks re-done by the fallback kernel (diagnostics: zsvd_fallback_count()).
__device__ unsigned long long g_fallback_tasks = 0;

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
    double pivmin, pivmax;
};

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
        if (sm.flag == 0) break;
        __syncthreads();
    }
    __syncthreads();
}

// Column norms of W -> sm.sig (unsorted), then ranks -> sm.ord (sorted desc,
// ties by index), then the rank cutoff and the truncation policy -> sm.k.
__device__ void sort_and_truncate(const double* W, int ldw, int p, int q, const SvdTask& t,
                                  Small& sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ double raw[kQMax];
    for (int j = warp; j < q; j += NWARPS) {
        const double* w = W + (int64_t)j * ldw;
        double a = 0.0;
        for (int r = lane; r < p; r += 32) a = fma(w[r], w[r], a);
        a = warp_sum(a);
        if (lane == 0) raw[j] = sqrt(a);
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
    __shared__ double inv_sig[kQMax];
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

// ------------------------------------------------------- tall-path pieces
// Per-thread 4x4 register tile of a w x w Gram matrix, with row groups when
// the tile grid is smaller than the CTA.
struct GramAcc {
    double acc[4][4];
    int ti, tj, group, groups, active;
    __device__ void init(int w) {
        int tn = (w + 3) / 4, nt = tn * tn;
        groups = T / nt;
        if (groups < 1) groups = 1;
        int tile = threadIdx.x % nt;
        group = threadIdx.x / nt;
        active = group < groups;
        ti = tile / tn;
        tj = tile % tn;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    }
    // Y: rows x w in smem, row-major with ld.
    __device__ void add(const double* Y, int rows, int ld, int w) {
        if (!active) return;
        const int i0 = ti * 4, j0 = tj * 4;
        for (int r = group; r < rows; r += groups) {
            const double* y = Y + r * ld;
            double a[4], b[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                a[e] = (i0 + e < w) ? y[i0 + e] : 0.0;
                b[e] = (j0 + e < w) ? y[j0 + e] : 0.0;
            }
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
                for (int z = 0; z < 4; ++z) acc[x][z] = fma(a[x], b[z], acc[x][z]);
        }
    }
    // G (w x w row-major, ld w) = sum over groups, fixed group order.
    __device__ void store(double* G, int w) {
        const int i0 = ti * 4, j0 = tj * 4;
        for (int g = 0; g < groups; ++g) {
            if (active && group == g) {
#pragma unroll
                for (int x = 0; x < 4; ++x)
#pragma unroll
                    for (int z = 0; z < 4; ++z)
                        if (i0 + x < w && j0 + z < w) {
                            double* d = G + (i0 + x) * w + (j0 + z);
                            *d = (g == 0) ? acc[x][z] : *d + acc[x][z];
                        }
            }
            __syncthreads();
        }
    }
};

// In-place upper Cholesky G = R^T R (G row-major q x q).  Records pivot range.
__device__ bool cholesky(double* G, int q, Small& sm) {
    if (threadIdx.x == 0) {
        sm.flag = 1;
        sm.pivmin = DBL_MAX;
        sm.pivmax = 0.0;
    }
    __syncthreads();
    for (int j = 0; j < q; ++j) {
        if (threadIdx.x == 0) {
            double d = G[j * q + j];
            if (!(d > 0.0) || !isfinite(d)) {
                sm.flag = 0;
            } else {
                double r = sqrt(d);
                G[j * q + j] = r;
                sm.pivmin = fmin(sm.pivmin, r);
                sm.pivmax = fmax(sm.pivmax, r);
            }
        }
        __syncthreads();
        if (!sm.flag) return false;
        const double rjj = G[j * q + j];
        for (int l = j + 1 + threadIdx.x; l < q; l += T) G[j * q + l] /= rjj;
        __syncthreads();
        const int rem = q - j - 1;
        for (int idx = threadIdx.x; idx < rem * rem; idx += T) {
            int l = j + 1 + idx / rem, c = j + 1 + idx % rem;
            if (c >= l) G[l * q + c] -= G[j * q + l] * G[j * q + c];
        }
        __syncthreads();
    }
    return true;
}

// X (rows x q, ld) <- X R^-1 for upper triangular R (row-major, ld q).
// Blocked by 8 columns: thread-per-row diagonal solve + parallel trailing update.
__device__ void trsm_right_upper(double* X, int rows, int ld, const double* R, int q) {
    for (int J0 = 0; J0 < q; J0 += 8) {
        const int J1 = min(J0 + 8, q);
        for (int r = threadIdx.x; r < rows; r += T) {
            double* x = X + r * ld;
            for (int j = J0; j < J1; ++j) {
                double acc = x[j];
                for (int i = J0; i < j; ++i) acc = fma(-x[i], R[i * q + j], acc);
                x[j] = acc / R[j * q + j];
            }
        }
        __syncthreads();
        const int rest = q - J1;
        if (rest > 0) {
            for (int idx = threadIdx.x; idx < rows * rest; idx += T) {
                int r = idx / rest, l = J1 + idx % rest;
                double* x = X + r * ld;
                double acc = x[l];
                for (int i = J0; i < J1; ++i) acc = fma(-x[i], R[i * q + l], acc);
                x[l] = acc;
            }
            __syncthreads();
        }
    }
}

__device__ void load_chunk(const SvdTask& t, double* X, int ld, int r0, int rows, int q) {
    for (int idx = threadIdx.x; idx < rows * q; idx += T) {
        int r = idx / q, j = idx % q;
        X[r * ld + j] = a_at(t, r0 + r, j);
    }
    __syncthreads();
}

// Tall path (W = A, m >= n).  Returns with sm.status set.
__device__ void tall_path(SvdTask& t, double* dyn, int budget, Small& sm) {
    const int p = sm.p, q = sm.q;
    const int q2 = q * q;
    double* C = dyn;            // G / R1 / R (row-major q x q)
    double* B = dyn + q2;       // G2 / R2, then V (col-major), then U_R (row-major q x k)
    double* tail = dyn + 2 * q2;
    const int tail_sz = budget - 2 * q2;
    const int ldx = q + 1;
    int ch12 = tail_sz / ldx;
    if (ch12 > kMaxChunk) ch12 = kMaxChunk;

    // pass 1: G = A^T A
    GramAcc g;
    g.init(q);
    for (int r0 = 0; r0 < p; r0 += ch12) {
        int rows = min(ch12, p - r0);
        load_chunk(t, tail, ldx, r0, rows, q);
        g.add(tail, rows, ldx, q);
        __syncthreads();
    }
    g.store(C, q);
    if (!cholesky(C, q, sm) || sm.pivmin < 1e-6 * sm.pivmax) {
        if (threadIdx.x == 0) sm.status = TASK_NEEDS_FALLBACK;
        __syncthreads();
        return;
    }
    // pass 2: G2 = Q1^T Q1, Q1 = A R1^-1
    g.init(q);
    for (int r0 = 0; r0 < p; r0 += ch12) {
        int rows = min(ch12, p - r0);
        load_chunk(t, tail, ldx, r0, rows, q);
        trsm_right_upper(tail, rows, ldx, C, q);
        g.add(tail, rows, ldx, q);
        __syncthreads();
    }
    g.store(B, q);
    if (!cholesky(B, q, sm) || sm.pivmin < 0.5 || sm.pivmax > 2.0) {
        if (threadIdx.x == 0) sm.status = TASK_NEEDS_FALLBACK;
        __syncthreads();
        return;
    }
    // R = R2 R1 -> W_R (tail, col-major) and back into C (row-major)
    double* WR = tail;
    for (int idx = threadIdx.x; idx < q2; idx += T) {
        int i = idx / q, j = idx % q;
        double acc = 0.0;
        if (j >= i)
            for (int l = i; l <= j; ++l) acc = fma(B[i * q + l], C[l * q + j], acc);
        WR[j * q + i] = acc;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < q2; idx += T) {
        int i = idx / q, j = idx % q;
        C[i * q + j] = WR[j * q + i];
    }
    __syncthreads();
    // SVD of R by one-sided Jacobi (V in B)
    jacobi(WR, q, q, q, B, sm);
    sort_and_truncate(WR, q, q, q, t, sm);
    if (sm.status != TASK_OK) return;
    const int k = sm.k;
    write_v(t, B, q, q, nullptr, sm);
    if (t.sign) {
        canonical_sign_global(t.v, t.ldv, t.vpre ? t.nvpre : q, k, sm);
    } else {
        if (threadIdx.x < k) sm.sgn[threadIdx.x] = 1.0;
        __syncthreads();
    }
    // U_R (row-major q x k) = W_R(:, ord) / sigma * sign  -> B
    double* UR = B;
    for (int idx = threadIdx.x; idx < q * k; idx += T) {
        int i = idx / k, r = idx % k;
        UR[i * k + r] = WR[sm.ord[r] * q + i] / sm.sig[r] * sm.sgn[r];
    }
    __syncthreads();
    // pass 3: U = (A R^-1) U_R, streamed out; U^T U accumulated for the check
    double* X = tail;
    int ch3 = k > 0 ? tail_sz / (ldx + k) : ch12;
    if (ch3 > kMaxChunk) ch3 = kMaxChunk;
    double* Uc = tail + ch3 * ldx;
    GramAcc gu;
    gu.init(k > 0 ? k : 1);
    if (k > 0) {
        for (int r0 = 0; r0 < p; r0 += ch3) {
            int rows = min(ch3, p - r0);
            load_chunk(t, X, ldx, r0, rows, q);
            trsm_right_upper(X, rows, ldx, C, q);
            for (int idx = threadIdx.x; idx < rows * k; idx += T) {
                int r = idx / k, c = idx % k;
                const double* x = X + r * ldx;
                double acc = 0.0;
                for (int l = 0; l < q; ++l) acc = fma(x[l], UR[l * k + c], acc);
                Uc[r * k + c] = acc;
                t.u[(int64_t)(r0 + r) * t.ldu + c] = acc;
            }
            __syncthreads();
            gu.add(Uc, rows, k, k);
            __syncthreads();
        }
        // orthonormality check of U (svd.hpp:48-58 contract, 1e-10)
        double* GU = tail;
        gu.store(GU, k);
        if (threadIdx.x == 0) sm.flag = 0;
        __syncthreads();
        for (int idx = threadIdx.x; idx < k * k; idx += T) {
            int i = idx / k, j = idx % k;
            double d = GU[idx] - (i == j ? 1.0 : 0.0);
            if (fabs(d) > kOrthonormalityTol) sm.flag = 1;
        }
        __syncthreads();
        if (sm.flag) {
            if (threadIdx.x == 0) sm.status = TASK_NEEDS_FALLBACK;
            __syncthreads();
            return;
        }
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
        if (m == 0 || n == 0) {
            *t.k_out = 0.0;
        } else if (sm.q > kQMax) {
            sm.status = TASK_UNSUPPORTED;
        }
    }
    __syncthreads();
    return sm.m > 0 && sm.n > 0 && sm.status == TASK_OK;
}

}  // namespace

__global__ void __launch_bounds__(kEngineThreads) svd_engine_kernel(SvdTask* tasks, int ntasks) {
    extern __shared__ double dyn[];
    __shared__ Small sm;
    if ((int)blockIdx.x >= ntasks) return;
    SvdTask t = tasks[blockIdx.x];
    if (!setup(t, sm)) {
        if (threadIdx.x == 0) tasks[blockIdx.x].status = sm.status;
        return;
    }
    const int budget = kEngineSmemBytes / 8;
    const int p = sm.p, q = sm.q;
    const bool direct = (int64_t)p * q + q * q <= budget && (p <= 2 * q || p <= 96 || !sm.tall);
    if (direct) {
        double* W = dyn;
        double* V = dyn + p * q;
        for (int idx = threadIdx.x; idx < p * q; idx += T) {
            int i, j;
            if (sm.tall) { i = idx / q; j = idx % q; }   // coalesced over A's rows
            else { j = idx / p; i = idx % p; }
            W[j * p + i] = w_at(t, sm.tall, i, j);
        }
        __syncthreads();
        jacobi(W, p, p, q, V, sm);
        finish_from_jacobi(t, W, p, V, sm);
    } else if (sm.tall) {
        tall_path(t, dyn, budget, sm);
    } else {
        if (threadIdx.x == 0) sm.status = TASK_UNSUPPORTED;
        __syncthreads();
    }
    if (threadIdx.x == 0) tasks[blockIdx.x].status = sm.status;
}

// Re-does flagged tasks by one-sided Jacobi on W in global scratch.  Grid-stride
// over tasks; CTA b owns scratch slot b (slot_doubles each).
__global__ void __launch_bounds__(kEngineThreads) svd_fallback_kernel(SvdTask* tasks, int ntasks,
                                                                      double* scratch,
                                                                      int64_t slot_doubles) {
    __shared__ Small sm;
    for (int ti = blockIdx.x; ti < ntasks; ti += gridDim.x) {
        if (tasks[ti].status != TASK_NEEDS_FALLBACK) continue;
        if (threadIdx.x == 0) atomicAdd(&g_fallback_tasks, 1ull);
        __syncthreads();
        SvdTask t = tasks[ti];
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
