// eigh.cuh — symmetric eigensolver for one n x n matrix (n <= 64) on one CTA
// of 256 threads, built for latency: the stitch of a range query has exactly
// one such problem (the Gram G = S^T S of the stacked sigma_p V_p^T,
// query.hpp:113-124), and sigma = sqrt(lambda), V = the eigenvectors.
//
// The one-sided Jacobi it replaces (svd_engine.cu mid-2) needs ~8 sweeps of
// n - 1 dependent rounds (~500 rounds of ~1,000 cycles at n = 64).  Here the
// sequential depth is ~n steps:
//
//  1. Householder tridiagonalisation T = Q^T G Q (LAPACK dsytd2, lower) with
//     G in the registers of four warps (no shared-memory traffic for the
//     matrix) and Q accumulated explicitly by the other four in the shadow of
//     the step.  Warp 4 forms reflector j + 1 from a stashed copy of row j + 1
//     (look-ahead) while the matrix warps run the rank-2 update of step j, and
//     the two 32-lane sums of a step go through the tensor pipe (warp_sum_mma);
//  2. the kv largest eigenvalues of T by Sturm-count multisection, warp-local:
//     ceil(kv / 8) eigenvalues per warp, one point per lane per iteration with a
//     division-free three-term recurrence (exact power-of-two rescale every
//     eight terms), brackets updated from a ballot, to ~4 eps ||T||;
//  3. inverse iteration (two solves, LU with partial pivoting as dgttrf, the
//     first solve's forward half fused into the factorisation) for each
//     eigenvalue on its own thread;
//  4. the eigenvectors of T made orthonormal (normalisation only, one symmetric
//     orthogonalisation step, or Cholesky QR, by how far from orthogonal they
//     are; a vector nearly parallel to earlier ones fails the task), then
//     taken back to G's basis as Q Z;
//  5. a residual check ||G x - lambda x||_max <= 1e-12 ||G||: the caller falls
//     back to its robust path on failure (status != 0).
//
// Accuracy is that of a backward-stable eigensolver of the Gram: eigenvalues
// to ~eps ||G||, eigenvectors to ~eps ||G|| / gap — the Gram-level accuracy the
// one-pass CholeskyQR path already accepts.  Reciprocals and
// square roots use the MUFU seeds with one third-order correction (<= 1 ulp),
// not the library's subroutines.
#pragma once

#include <cstdint>
#include <type_traits>

#ifndef EIGH_CLK
#define EIGH_CLK(i)
#endif
#ifndef EIGH_NOQ
#define EIGH_NOQ 0
#endif
#ifndef EIGH_NOUPD
#define EIGH_NOUPD 0
#endif
#ifndef EIGH_WSUM
#define EIGH_WSUM warp_sum_mma
#endif
#ifndef EIGH_SUB
#define EIGH_SUB(i)
#define EIGH_SUB_INIT
#define EIGH_SUB_DONE
#endif

namespace zsvd {
namespace eigh {

constexpr int kThreads = 256;
constexpr int kLd = 68;  // row stride of A (doubles): the 4-threads-per-row matvec / update are conflict-free
// Shared-memory plan (doubles) for n <= 64 and kk <= KMAX wanted eigenpairs.
// Z's row stride keeps the back-transform's (column, row-part) lanes
// conflict-free: 2 (part) + column spans 16 distinct banks.
template <int KMAX>
struct Plan {
    static constexpr int LDZ = KMAX <= 24 ? 26 : 66;
    static constexpr int A = 0;                  // n x n (ld kLd): G, then the reflectors below the diagonal
    static constexpr int Z = A + 64 * kLd;       // n x kk (ld LDZ): eigenvectors
    static constexpr int LU = Z + 64 * LDZ;      // 4 x n x kk: U diag^-1, U super-1, U super-2, L
    static constexpr int D = LU + 4 * 64 * KMAX; // d, e, e^2, tau, lam (64 each)
    static constexpr int V = D + 5 * 64;         // tridiagonalisation vectors: 2 x 72 v, 2 x 64 p, 2 x 72 rows
    static constexpr int RED = V + 416;          // 32 scratch
    static constexpr int BR = RED + 32;          // 128 scratch: B's diagonal, R_aa^-1
    static constexpr int TOTAL = BR + 128;
    static constexpr int bytes() { return TOTAL * 8; }
    static_assert(4 * 64 * KMAX >= KMAX * kLd, "the Cholesky QR's B reuses the LU area");
};

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// Sum over the warp on the tensor pipe (latency: three DMMAs and one shuffle
// against five shuffle + add levels): x as the 8 x 4 operand times ones gives
// every lane the sum of its group of four, the eight group sums as two 4 x 8
// operands under a ones matrix give the total.  Every lane gets the same bits.
// All 32 lanes must call it.
__device__ __forceinline__ double warp_sum_mma(double x) {
    const int lane = threadIdx.x & 31;
    double g0 = 0.0, g1 = 0.0;
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(g0), "+d"(g1)
        : "d"(x), "d"(1.0));
    const double b1 = __shfl_sync(0xffffffffu, g0, 4 * (lane & 3));
    const double b2 = __shfl_sync(0xffffffffu, g0, 16 + 4 * (lane & 3));
    double t0 = 0.0, t1 = 0.0;
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(t0), "+d"(t1)
        : "d"(1.0), "d"(b1));
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(t0), "+d"(t1)
        : "d"(1.0), "d"(b2));
    return t0;
}

// 1 / x and 1 / sqrt(x) from the MUFU seeds (~2^-20) with one third-order
// correction: <= 1 ulp, four dependent operations, no subroutine call.
__device__ __forceinline__ double rcp_nr(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x, y, 1.0);
    return fma(y * e, 1.0 + e, y);  // y (1 + e + e^2)
}
__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x * y, y, 1.0);
    return fma(y * e, fma(0.375, e, 0.5), y);
}

// 2^-(exponent of max(|a|, |b|)): an exact power of two bringing the larger of
// a, b to [1, 2) (1 when both are zero).
__device__ __forceinline__ double renorm_factor(double a, double b) {
    const int ea = (__double2hiint(a) >> 20) & 0x7ff, eb = (__double2hiint(b) >> 20) & 0x7ff;
    const int e = ea > eb ? ea : eb;
    return e == 0 ? 1.0 : __hiloint2double((2046 - e) << 20, 0);
}

// Deterministic start vector entries in [0.5, 1.5) with pseudo-random signs.
__device__ __forceinline__ double start_entry(int i, int t) {
    unsigned h = (unsigned)(i * 0x9E3779B1u) ^ (unsigned)((t + 1) * 0x85EBCA77u);
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    const double u = 0.5 + (double)(h & 0xFFFFFu) * (1.0 / 1048576.0);
    return (h & 0x100000u) ? -u : u;
}

// Householder reflector (dlarfg) of [alpha; x_tail] with s = ||x_tail||^2:
// beta, tau and the tail scale 1 / (alpha - beta); tau = 0 means H = I.
__device__ __forceinline__ void reflector(double alpha, double s, double& beta, double& tau, double& sc) {
    beta = alpha;
    tau = 0.0;
    sc = 0.0;
    if (s > 0.0) {
        const double h = fma(alpha, alpha, s);
        const double nrm = h * rsqrt_nr(h);
        beta = alpha >= 0.0 ? -nrm : nrm;
        tau = fma(-alpha, rcp_nr(beta), 1.0);  // (beta - alpha) / beta
        sc = rcp_nr(alpha - beta);
    }
}

// Eigen-decomposition of the symmetric n x n matrix G (global, row-major, ld ldg;
// only the upper triangle i <= j is read) times `scale` (a power of two making
// max |G| ~ 1).  Computes the kv >= kk largest eigenvalues (descending) and
// the eigenvectors of the first kk:
//   sm[Plan<KMAX>::D + 256 + t]          = lambda_t (of the scaled matrix), t < kv
//   sm[Plan<KMAX>::Z + i * Plan::LDZ + t] = component i of eigenvector t
// Returns 0 on success, nonzero when the result failed its orthogonality (2)
// or residual (3) check (the caller's robust path takes over).  All 256
// threads call it; sm holds Plan<KMAX>::bytes().  n >= 1, 1 <= kk <= min(n, KMAX),
// kk <= kv <= min(n, 64).
template <int KMAX>
__device__ int eigh_top(const double* __restrict__ G, int64_t ldg, int n, int kk, int kv, double scale, double* sm) {
    using P = Plan<KMAX>;
    constexpr int kLdZ = P::LDZ;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* A = sm + P::A;
    double* Z = sm + P::Z;
    double* LUb = sm + P::LU;
    double* d = sm + P::D;
    double* e = d + 64;
    double* ee = d + 128;
    double* tau = d + 192;
    double* lam = d + 256;
    double* red = sm + P::RED;
    double* br = sm + P::BR;
    __shared__ int status;
#define RED_A(w) red[16 + (w)]

    // ---- load the upper triangle, mirror, scale (zero-padded to 64 x 64) ---------
    // (a thread's loads are issued together, before its stores: a load is not hoisted
    // over a store through a generic pointer — one L2 round trip per entry otherwise)
    {
        constexpr int kPer = 64 * 64 / kThreads;
        static_assert(kPer * kThreads == 64 * 64, "whole entries per thread");
        double gv[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int x = tid + u * kThreads;
            const int i = x >> 6, j = x & 63;
            const int a = i <= j ? i : j, b = i <= j ? j : i;
            gv[u] = (i < n && j < n) ? G[(int64_t)a * ldg + b] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int x = tid + u * kThreads;
            A[(x >> 6) * kLd + (x & 63)] = scale * gv[u];
        }
    }
    if (tid == 0) status = 0;
    __syncthreads();
    EIGH_CLK(0);

    // ---- 1. tridiagonalisation ---------------------------------------------------
    // Step j: H_j = I - tau_j v v^T (v_c = 0 for c <= j, v_{j+1} = 1) zeroes
    // A[j+2.., j].  A lives in the registers of warps 0-3: warp w holds rows
    // 32 (w & 1) .. + 31 (one per lane), columns 32 (w >> 1) .. + 31, so the
    // matvec p = tau A v and the rank-2 update A -= v w^T + w v^T never touch
    // shared memory but for the vectors.  Warps 4-7 hold Q = H_0 H_1 ... (two
    // lanes per row, 32 columns each) and apply each reflector while A's warps
    // run the next step, so the back-transform is one n x n x kk product at the
    // end.  A step costs two barriers: p's halves (A's warps only), then v_{j+1},
    // which the two warps holding row j + 1 form from it once updated.
    const bool isA = warp < 4;
    const int hA = warp >> 1, rA = ((warp & 1) << 5) | lane;  // A: column half, row
    const int rQ = (tid - 128) >> 1, hQ = tid & 1;            // Q: row, column half
    double* vs = sm + P::V;          // 2 x 72: v (half 1 at +34: the Q lanes' halves differ in bank)
    double* pp = vs + 144;           // 2 x 64: the matvec's column-half partials
    double* rowbuf = pp + 128;       // 2 x 72: row j + 1 before update j (same layout as v), by step parity
    auto vo = [](int c) { return c + (c >= 32 ? 2 : 0); };
    double a[32];
    if (isA) {
#pragma unroll
        for (int u = 0; u < 32; ++u) a[u] = A[rA * kLd + 32 * hA + u];
    } else {
#pragma unroll
        for (int u = 0; u < 32; ++u) a[u] = (32 * hQ + u == rQ) ? 1.0 : 0.0;
    }
    // the two A threads holding row r put it (as it stands) in row buffer `buf`
    auto stash_row = [&](int r, int buf) {
        if (isA && (warp & 1) == (r >> 5) && lane == (r & 31)) {
            double* rw = rowbuf + 72 * buf + 34 * hA;
#pragma unroll
            for (int u = 0; u < 32; u += 2) *reinterpret_cast<double2*>(rw + u) = make_double2(a[u], a[u + 1]);
        }
    };
    // reflector r from row r of the current matrix, x[h] = entry lane + 32 h (one
    // warp): v_r into v buffer `buf`, tau[r], e[r], d[r]
    auto finish_reflector = [&](int r, int buf, const double (&x)[2]) {
        double ssq = 0.0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = lane + 32 * h;
            if (c >= r + 2 && c < n) ssq = fma(x[h], x[h], ssq);
        }
        ssq = EIGH_WSUM(ssq);
        const double xa = __shfl_sync(0xffffffffu, (r + 1) >= 32 ? x[1] : x[0], (r + 1) & 31);
        const double xd = __shfl_sync(0xffffffffu, r >= 32 ? x[1] : x[0], r & 31);
        const double alpha = r + 1 < n ? xa : 0.0;
        double beta, tr, sc;
        reflector(alpha, ssq, beta, tr, sc);
        double* vn = vs + 72 * buf;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = lane + 32 * h;
            vn[vo(c)] = c <= r || c >= n ? 0.0 : (c == r + 1 ? 1.0 : x[h] * sc);
        }
        if (lane == 0) {
            tau[r] = r + 1 < n ? tr : 0.0;
            e[r] = r + 1 < n ? beta : 0.0;
            d[r] = xd;
        }
    };
    __syncthreads();  // A's registers loaded: the A area is free (Q lands there at the end)
    stash_row(0, 1);
    stash_row(1, 0);
    __syncthreads();
    if (warp == 4) {
        double x[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) x[h] = lane + 32 * h < n ? rowbuf[72 + vo(lane + 32 * h)] : 0.0;
        finish_reflector(0, 0, x);
    }
    __syncthreads();
    EIGH_SUB_INIT
    for (int j = 0; j + 2 < n; ++j) {
        EIGH_SUB(0);
        const int cb = j & 1;
        const double* v = vs + 72 * cb;
        const double tj = tau[j];
        if (isA) {
            const bool rows_live = 32 * (warp & 1) + 31 > j;  // warp-uniform
            double vc[32];
#pragma unroll
            for (int u = 0; u < 32; u += 2) {
                const double2 t2 = *reinterpret_cast<const double2*>(v + 34 * hA + u);
                vc[u] = t2.x;
                vc[u + 1] = t2.y;
            }
            double pr = 0.0;
            if (tj != 0.0 && rows_live) {
                double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int g = 0; g < 4; ++g)
                    if (32 * hA + 8 * g + 7 > j) {
#pragma unroll
                        for (int u = 8 * g; u < 8 * g + 8; ++u) acc[u & 7] = fma(a[u], vc[u], acc[u & 7]);
                    }
                pr = rA > j ? tj * (((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]))) : 0.0;
            }
            pp[64 * hA + rA] = pr;
            const double vi = v[vo(rA)];
            double pv = EIGH_WSUM(pr * vi);
            if (lane == 0) RED_A(warp) = pv;
            EIGH_SUB(1);
            asm volatile("bar.sync 1, 160;" ::: "memory");
            EIGH_SUB(2);
            if (tj != 0.0 && rows_live && !EIGH_NOUPD) {
                const double K = -0.5 * tj * ((RED_A(0) + RED_A(1)) + (RED_A(2) + RED_A(3)));
                // a_ic -= v_i w_c + w_i v_c with w = p + K v, as v_i p_c + (w_i + K v_i) v_c
                const double wi = fma(K, vi, fma(K, vi, pp[rA] + pp[64 + rA]));
#pragma unroll
                for (int g = 0; g < 4; ++g)
                    if (32 * hA + 8 * g + 7 > j) {
#pragma unroll
                        for (int u = 8 * g; u < 8 * g + 8; u += 2) {
                            const double2 p0 = *reinterpret_cast<const double2*>(pp + 32 * hA + u);
                            const double2 p1 = *reinterpret_cast<const double2*>(pp + 64 + 32 * hA + u);
                            a[u] = fma(-vi, p0.x + p1.x, fma(-wi, vc[u], a[u]));
                            a[u + 1] = fma(-vi, p0.y + p1.y, fma(-wi, vc[u + 1], a[u + 1]));
                        }
                    }
            }
            EIGH_SUB(3);
            // row j + 2 as it now stands, for the next step's look-ahead
            if (j + 2 < n) stash_row(j + 2, cb ^ 1);
            EIGH_SUB(4);
        } else {
            if (tj != 0.0 && !EIGH_NOQ) {
                // Q <- Q H_j: q -= tau (q . v) v^T (rows of the pair: halves combined by a shuffle)
                double vc[32], acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int u = 0; u < 32; u += 2) {
                    const double2 t2 = *reinterpret_cast<const double2*>(v + 34 * hQ + u);
                    vc[u] = t2.x;
                    vc[u + 1] = t2.y;
                }
#pragma unroll
                for (int u = 0; u < 32; ++u) acc[u & 3] = fma(a[u], vc[u], acc[u & 3]);
                double dq = (acc[0] + acc[1]) + (acc[2] + acc[3]);
                dq += __shfl_xor_sync(0xffffffffu, dq, 1);
                dq *= -tj;
#pragma unroll
                for (int u = 0; u < 32; ++u) a[u] = fma(dq, vc[u], a[u]);
            }
            if (warp == 4) {
                // look-ahead: row j + 1 of the updated matrix from its stashed copy,
                // p and K (the same expressions as the A warps' update, so the same
                // bits), then reflector j + 1 while the A warps run their update
                asm volatile("bar.sync 1, 160;" ::: "memory");
                const int r = j + 1;
                const double* rw = rowbuf + 72 * cb;
                double x[2];
                if (tj != 0.0 && !EIGH_NOUPD) {
                    const double K = -0.5 * tj * ((RED_A(0) + RED_A(1)) + (RED_A(2) + RED_A(3)));
                    const double vi = v[vo(r)];
                    const double wi = fma(K, vi, fma(K, vi, pp[r] + pp[64 + r]));
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int c = lane + 32 * h;
                        x[h] = c < n ? fma(-vi, pp[c] + pp[64 + c], fma(-wi, v[vo(c)], rw[vo(c)])) : 0.0;
                    }
                } else {
#pragma unroll
                    for (int h = 0; h < 2; ++h) x[h] = lane + 32 * h < n ? rw[vo(lane + 32 * h)] : 0.0;
                }
                finish_reflector(r, cb ^ 1, x);
            }
        }
        __syncthreads();
        EIGH_SUB(5);
    }
    EIGH_SUB_DONE
    // the last diagonal entry, and Q to shared memory (rows, ld kLd)
    if (isA && n >= 2) {
        const int r = n - 1;
        if ((warp & 1) == (r >> 5) && lane == (r & 31)) {
#pragma unroll
            for (int u = 0; u < 32; ++u)
                if (32 * hA + u == r) d[r] = a[u];
        }
    }
    if (!isA) {
#pragma unroll
        for (int u = 0; u < 32; u += 2)
            *reinterpret_cast<double2*>(A + rQ * kLd + 32 * hQ + u) = make_double2(a[u], a[u + 1]);
    }
    __syncthreads();
    EIGH_CLK(1);
    if (tid < n) ee[tid] = tid + 1 < n ? e[tid] * e[tid] : 0.0;
    __syncthreads();
    // Gershgorin interval (every warp computes it, same order)
    double glo, ghi;
    {
        double lo = 1e300, hi = -1e300;
        for (int i = lane; i < n; i += 32) {
            const double rad = fabs(i > 0 ? e[i - 1] : 0.0) + fabs(i + 1 < n ? e[i] : 0.0);
            lo = fmin(lo, d[i] - rad);
            hi = fmax(hi, d[i] + rad);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        const double tn = fmax(fabs(lo), fabs(hi));
        glo = lo - 4.0 * 2.220446049250313e-16 * tn - 1e-300;
        ghi = hi + 4.0 * 2.220446049250313e-16 * tn + 1e-300;
    }
    const double tnorm = fmax(fabs(glo), fabs(ghi));

    // ---- 2. the kk largest eigenvalues: multisection, warp-local -----------------
    // ceil(kk / 8) eigenvalues per warp, gs = 32 / that lanes per eigenvalue,
    // one Sturm count per lane per iteration (the recurrence is latency-bound;
    // fewer, longer iterations cost less fp64 issue than wider ones).  The new
    // bracket follows from a ballot of "count <= target" (counts are monotone
    // in x), so no shared memory and no CTA barrier.
    {
        const int epw = (kv + 7) / 8;
        const int gs = 32 / epw;
        const int gi = lane / gs, mem = lane - gi * gs;
        const int g = warp * epw + gi;  // eigenvalue (descending index)
        const bool act = gi < epw && g < kv;
        const unsigned gmask = (gi < epw ? ((gs == 32 ? 0xffffffffu : ((1u << gs) - 1u)) << (gi * gs)) : 0u);
        const int target = n - 1 - g;  // ascending index
        double a = glo, b = ghi;
        const double rshrink = 1.0 / (double)(gs + 1);
        int iters = 1;
        for (double w = ghi - glo; w > 4.0 * 2.220446049250313e-16 * tnorm && iters < 200; w *= rshrink) ++iters;
        for (int it = 0; it < iters; ++it) {
            const double h = (b - a) * rshrink;
            const double x = fma((double)(mem + 1), h, a);
            int c = n;
            if (act) {
                double pa = 1.0, pb = d[0] - x;
                int sg = __double2hiint(pb) >> 31;
                int cn = sg;
                int i = 1;
                for (; i + 8 <= n; i += 8) {
                    double dd[8], e2[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        dd[u] = d[i + u];
                        e2[u] = ee[i + u - 1];
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const double q = fma(dd[u] - x, pb, -e2[u] * pa);
                        const int s2 = __double2hiint(q) >> 31;
                        cn += s2 ^ sg;
                        sg = s2;
                        pa = pb;
                        pb = q;
                    }
                    const double f = renorm_factor(pa, pb);
                    pa *= f;
                    pb *= f;
                }
                for (; i < n; ++i) {
                    const double q = fma(d[i] - x, pb, -ee[i - 1] * pa);
                    const int s2 = __double2hiint(q) >> 31;
                    cn += s2 ^ sg;
                    sg = s2;
                    pa = pb;
                    pb = q;
                }
                c = -cn;
            }
            const unsigned ok = __ballot_sync(0xffffffffu, act && c <= target) & gmask;
            const int nt = __popc(ok);  // points at or below the eigenvalue
            const double na = nt > 0 ? fma((double)nt, h, a) : a;
            const double nb = nt < gs ? fma((double)(nt + 1), h, a) : b;
            a = na;
            b = nb;
        }
        if (act && mem == 0) lam[g] = 0.5 * (a + b);
    }
    __syncthreads();
    EIGH_CLK(2);

    // ---- 3. inverse iteration: eigenvalue lam[t] on lane t / 8 of warp t % 8 ------
    // (a few lanes in each of the eight warps: the chains issue in parallel)
    const int t_inv = (lane << 3) | warp;
    if (t_inv < kk) {
        const int t = t_inv;
        const double lt = lam[t];
        const double pivmin = 2.220446049250313e-16 * tnorm + 1e-300;
        double* Ud = LUb;             // 1 / U_ii
        double* U1 = LUb + 64 * kk;   // U_{i,i+1}
        double* U2 = LUb + 128 * kk;  // U_{i,i+2}
        double* Lm = LUb + 192 * kk;  // multipliers
        uint64_t piv = 0;
        // dgttrf of T - lt I with the forward half of the first solve (P, L applied
        // to a pseudo-random start vector) fused in: y_i leaves row i final
        double a = d[0] - lt, bsup = n > 1 ? e[0] : 0.0;
        double ycur = start_entry(0, t);
        for (int i = 0; i + 1 < n; ++i) {
            const double c = e[i], a1 = d[i + 1] - lt, b1 = i + 2 < n ? e[i + 1] : 0.0;
            double ynext = start_entry(i + 1, t);
            // branch-free (the few lanes of a warp pivot on different rows): the same
            // operations as the two cases of dgttrf, operands picked by selects
            const bool keep = fabs(a) >= fabs(c);
            const double ui = fabs(a) < pivmin ? (a < 0.0 ? -pivmin : pivmin) : a;
            const double ru = rcp_nr(keep ? ui : c);
            const double l = (keep ? c : a) * ru;
            const double u1 = keep ? bsup : a1;
            const double u2 = keep ? 0.0 : b1;
            a = fma(-l, keep ? bsup : a1, keep ? a1 : bsup);
            bsup = keep ? b1 : -l * b1;
            const double ykeep = keep ? ycur : ynext;  // row i of P L^-1 y (rows i, i + 1 swap on a pivot)
            ynext = fma(-l, ykeep, keep ? ynext : ycur);
            ycur = ykeep;
            piv |= keep ? 0ull : (1ull << i);
            Ud[i * kk + t] = ru;
            U1[i * kk + t] = u1;
            U2[i * kk + t] = u2;
            Lm[i * kk + t] = l;
            Z[i * kLdZ + t] = ycur;
            ycur = ynext;
        }
        {
            const double ui = fabs(a) < pivmin ? (a < 0.0 ? -pivmin : pivmin) : a;
            Ud[(n - 1) * kk + t] = rcp_nr(ui);
            U1[(n - 1) * kk + t] = 0.0;
            U2[(n - 1) * kk + t] = 0.0;
            Z[(n - 1) * kLdZ + t] = ycur;
        }
        // two solves: lam is accurate to ~4 eps ||T||, so each solve scales the
        // other eigencomponents by ~eps ||T|| / gap relative to this one; the
        // second makes the result independent of how the start vector projects
        for (int sweep = 0; sweep < 2; ++sweep) {
            if (sweep == 1) {  // P, L of the second solve
                double xi = Z[t];
                for (int i = 0; i + 1 < n; ++i) {
                    double x1 = Z[(i + 1) * kLdZ + t];
                    if ((piv >> i) & 1) {
                        const double tmp = xi;
                        xi = x1;
                        x1 = tmp;
                    }
                    Z[i * kLdZ + t] = xi;
                    xi = fma(-Lm[i * kk + t], xi, x1);
                }
                Z[(n - 1) * kLdZ + t] = xi;
            }
            double z2 = 0.0, z1 = 0.0, big = 0.0;
            for (int i = n - 1; i >= 0; --i) {  // U
                const double zi = fma(-U2[i * kk + t], z2, fma(-U1[i * kk + t], z1, Z[i * kLdZ + t])) * Ud[i * kk + t];
                Z[i * kLdZ + t] = zi;
                big = fmax(big, fabs(zi));
                z2 = z1;
                z1 = zi;
            }
            if (sweep == 0) {  // rescale between the solves (the first grows ~1 / (eps ||T||))
                const double inv = big > 0.0 ? rcp_nr(big) : 1.0;
                for (int i = 0; i < n; ++i) Z[i * kLdZ + t] *= inv;
            }
        }
    }
    __syncthreads();
    EIGH_CLK(3);

    // ---- 4a. Cholesky QR of Z (n x kk): B = Z^T Z, R = chol(B), Z = Z R^-1 --------
    double* B = LUb;  // kk x kk, ld kLd (the LU factors are no longer needed)
    for (int x = tid; x < kk * kk; x += kThreads) {
        const int ia = x / kk, ib = x - ia * kk;
        if (ia <= ib) {
            double s[4] = {0.0, 0.0, 0.0, 0.0};
            for (int i = 0; i < n; i += 4) {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (i + u < n) s[u] = fma(Z[(i + u) * kLdZ + ia], Z[(i + u) * kLdZ + ib], s[u]);
            }
            B[ia * kLd + ib] = (s[0] + s[1]) + (s[2] + s[3]);
        }
    }
    __syncthreads();
    // right-looking Cholesky of B on the whole CTA, one barrier per column; B's
    // upper triangle keeps the unscaled rows, br[64 + a] = R_aa^-1, so
    // R[a][c] = B[a][c] br[64 + a].  A column keeping less than 1e-2 of its
    // length once the earlier ones are removed was (nearly) parallel to them:
    // two eigenvalues too close for inverse iteration to separate (status 2).
    for (int c = tid; c < kk; c += kThreads) br[c] = B[c * kLd + c];
    if (tid == 0) status = 0;
    __syncthreads();
    // vectors already orthogonal to ~eps (well separated eigenvalues: the usual
    // case) only need normalising; otherwise the Cholesky QR below
    {
        bool far = false;
        for (int x = tid; x < kk * kk; x += kThreads) {
            const int ia = x / kk, ib = x - ia * kk;
            if (ia < ib && !(fabs(B[ia * kLd + ib]) <= 1e-13 * sqrt(br[ia] * br[ib]))) far = true;
        }
        if (!__syncthreads_or(far)) {
            for (int x = tid; x < n * kk; x += kThreads) {
                const int i = x / kk, t = x - i * kk;
                Z[i * kLdZ + t] *= rsqrt_nr(br[t]);
            }
            __syncthreads();
            goto orthonormal;
        }
    }
    // nearly orthogonal (every normalised inner product below 1e-8: eigenvalues
    // apart by more than ~1e-8 ||T||): one symmetric orthogonalisation step
    // Z <- Zn (I - E / 2), Zn the normalised vectors, E = Zn^T Zn - I, leaves a
    // defect ~ kk |E|^2 <= 2e-15 and is one n x kk x kk product with no
    // sequential dependence (the Cholesky QR below is kk dependent columns)
    {
        bool farther = false;
        for (int x = tid; x < kk * kk; x += kThreads) {
            const int ia = x / kk, ib = x - ia * kk;
            if (ia < ib && !(fabs(B[ia * kLd + ib]) <= 1e-8 * sqrt(br[ia] * br[ib]))) farther = true;
        }
        if (!__syncthreads_or(farther)) {
            double* Zt = LUb + 64 * kLd;  // n x kk scratch (ld kLdZ) beyond B
            if (tid < kk) br[64 + tid] = rsqrt_nr(br[tid]);
            __syncthreads();
            for (int x = tid; x < n * kk; x += kThreads) {
                const int i = x / kk, t = x - i * kk;
                const double rt = br[64 + t];
                double acc0 = 0.0, acc1 = 0.0;
                int sidx = 0;
                for (; sidx + 1 < kk; sidx += 2) {
                    const int s0 = sidx, s1 = sidx + 1;
                    const double e0 = s0 == t ? 0.0 : B[(s0 < t ? s0 : t) * kLd + (s0 < t ? t : s0)] * br[64 + s0];
                    const double e1 = s1 == t ? 0.0 : B[(s1 < t ? s1 : t) * kLd + (s1 < t ? t : s1)] * br[64 + s1];
                    acc0 = fma(Z[i * kLdZ + s0] * br[64 + s0], e0, acc0);
                    acc1 = fma(Z[i * kLdZ + s1] * br[64 + s1], e1, acc1);
                }
                if (sidx < kk && sidx != t)
                    acc0 = fma(Z[i * kLdZ + sidx] * br[64 + sidx],
                               B[(sidx < t ? sidx : t) * kLd + (sidx < t ? t : sidx)] * br[64 + sidx], acc0);
                // E[s][t] = B[s][t] rs_s rs_t: acc carries rs_s^2 B[s][t], the factor rs_t is applied once
                Zt[i * kLdZ + t] = rt * fma(-0.5, acc0 + acc1, Z[i * kLdZ + t]);
            }
            __syncthreads();
            for (int x = tid; x < n * kk; x += kThreads) {
                const int i = x / kk, t = x - i * kk;
                Z[i * kLdZ + t] = Zt[i * kLdZ + t];
            }
            __syncthreads();
            goto orthonormal;
        }
    }
    for (int jj = 0; jj < kk; ++jj) {
        const double djj = B[jj * kLd + jj];
        if (!(djj > 1e-4 * br[jj])) {  // uniform (one Cholesky QR pass leaves ~eps / this ratio: 1e-12)
            if (tid == 0) status = 2;
            break;
        }
        const double inv2 = rcp_nr(djj);
        if (tid == 0) {
            br[64 + jj] = rsqrt_nr(djj);
            vs[jj] = inv2;  // (the tridiagonalisation's vectors are dead)
        }
        const int w = kk - jj - 1;
        for (int x = tid; x < w * w; x += kThreads) {
            const int c = jj + 1 + x / w, c2 = jj + 1 + x % w;
            if (c2 >= c) B[c * kLd + c2] = fma(-B[jj * kLd + c] * inv2, B[jj * kLd + c2], B[c * kLd + c2]);
        }
        __syncthreads();
    }
    __syncthreads();
    if (status) return status;
    if (kk <= 24) {
        // Z = Z R^-1, a row per thread in registers, right-looking: y_c = z_c / R_cc,
        // then z_c' -= y_c R_cc' = (z_c / d_cc) B[c][c'] for the later columns (the
        // chain is one multiply and one fma per column)
        if (tid < n) {
            double z[24];
#pragma unroll
            for (int c = 0; c < 24; ++c) z[c] = c < kk ? Z[tid * kLdZ + c] : 0.0;
#pragma unroll
            for (int c = 0; c < 24; ++c) {
                if (c < kk) {
                    const double t2 = z[c] * vs[c];
                    z[c] *= br[64 + c];
#pragma unroll
                    for (int c2 = c + 1; c2 < 24; ++c2)
                        if (c2 < kk) z[c2] = fma(-t2, B[c * kLd + c2], z[c2]);
                }
            }
#pragma unroll
            for (int c = 0; c < 24; ++c)
                if (c < kk) Z[tid * kLdZ + c] = z[c];
        }
    } else {
    // Z = Z R^-1: 4 threads per row (same warp), columns in order, the sums over
    // earlier columns split four ways
    {
        const int i = tid >> 2, q = tid & 3;
        for (int c = 0; c < kk; ++c) {
            double s0 = 0.0, s1 = 0.0;
            if (i < n) {
                int a = q;
                for (; a + 4 < c; a += 8) {
                    s0 = fma(Z[i * kLdZ + a], B[a * kLd + c] * br[64 + a], s0);
                    s1 = fma(Z[i * kLdZ + a + 4], B[(a + 4) * kLd + c] * br[68 + a], s1);
                }
                if (a < c) s0 = fma(Z[i * kLdZ + a], B[a * kLd + c] * br[64 + a], s0);
            }
            double sum = s0 + s1;
            sum += __shfl_xor_sync(0xffffffffu, sum, 1);
            sum += __shfl_xor_sync(0xffffffffu, sum, 2);
            if (i < n && q == 0) Z[i * kLdZ + c] = (Z[i * kLdZ + c] - sum) * br[64 + c];
            __syncwarp();
        }
    }
    }
    __syncthreads();
orthonormal:
    // residual in T's basis (T is tridiagonal: three terms per entry)
    {
        double worst = 0.0;
        for (int x = tid; x < n * kk; x += kThreads) {
            const int i = x / kk, t = x - i * kk;
            double r = fma(d[i] - lam[t], Z[i * kLdZ + t], 0.0);
            if (i > 0) r = fma(e[i - 1], Z[(i - 1) * kLdZ + t], r);
            if (i + 1 < n) r = fma(e[i], Z[(i + 1) * kLdZ + t], r);
            worst = fmax(worst, fabs(r));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
        if (lane == 0) red[8 + warp] = worst;
        __syncthreads();
        double w = 0.0;
        for (int i = 0; i < 8; ++i) w = fmax(w, red[8 + i]);
        if (!(w <= 1e-12 * fmax(tnorm, 1e-300))) return 3;
    }
    EIGH_CLK(4);

    // ---- 4b. back to G's basis: X = Q Z (Q in the A area, rows, ld kLd) ----------
    // thread (row i, column phase g) accumulates X[i][g + 4 s] over c in order
    auto back_transform = [&](auto ncols) {
        constexpr int kS = decltype(ncols)::value;
        const int i = tid >> 2, g = tid & 3;
        double acc[kS];
#pragma unroll
        for (int s2 = 0; s2 < kS; ++s2) acc[s2] = 0.0;
        if (i < n) {
            const double* qr = A + i * kLd;
            for (int c = 0; c < n; ++c) {
                const double qc = qr[c];
                const double* zr = Z + c * kLdZ + g;
#pragma unroll
                for (int s2 = 0; s2 < kS; ++s2)
                    if (g + 4 * s2 < kk) acc[s2] = fma(qc, zr[4 * s2], acc[s2]);
            }
        }
        __syncthreads();
        if (i < n) {
#pragma unroll
            for (int s2 = 0; s2 < kS; ++s2)
                if (g + 4 * s2 < kk) Z[i * kLdZ + g + 4 * s2] = acc[s2];
        }
    };
    if (kk <= 24) back_transform(std::integral_constant<int, 6>());
    else back_transform(std::integral_constant<int, (KMAX + 3) / 4>());
    __syncthreads();
    EIGH_CLK(5);
    EIGH_CLK(6);
    return 0;
#undef RED_A
}

}  // namespace eigh
}  // namespace zsvd
