// eigh.cuh — symmetric eigensolver for one n x n matrix (n <= 64) on one CTA
// of 256 threads, built for latency: the stitch of a range query has exactly
// one such problem (the Gram G = S^T S of the stacked sigma_p V_p^T,
// query.hpp:113-124), and sigma = sqrt(lambda), V = the eigenvectors.
//
// The one-sided Jacobi it replaces (svd_engine.cu mid-2) needs ~8 sweeps of
// n - 1 dependent rounds (~500 rounds of ~1,000 cycles at n = 64).  Here the
// sequential depth is ~n steps:
//
//  1. Householder tridiagonalisation T = Q^T G Q (LAPACK dsytd2, lower):
//     warp 0 forms each reflector from the column it updates itself while the
//     other warps finish the trailing rank-2 update, so a step costs two CTA
//     barriers (matvec, update);
//  2. the kk largest eigenvalues of T by Sturm-count multisection: each
//     eigenvalue gets 256 / kk threads, each thread counts four points with a
//     division-free three-term recurrence (power-of-two renormalisation every
//     eight terms), one CTA barrier per iteration, to ~4 eps ||T||;
//  3. inverse iteration (two solves, LU with partial pivoting as dgttrf, the
//     first solve's forward half fused into the factorisation) for each
//     eigenvalue on its own thread;
//  4. the eigenvectors of T made orthonormal (Cholesky QR: close eigenvalues
//     give vectors that are only nearly orthogonal; a vector nearly parallel
//     to earlier ones fails the task), then taken back to G's basis through
//     the stored reflectors;
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

#ifndef EIGH_CLK
#define EIGH_CLK(i)
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
    static constexpr int V = D + 5 * 64;         // reflector / p vectors, double-buffered: 2 x (v, p)
    static constexpr int RED = V + 4 * 64;       // 32 scratch
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
    double* vbuf = sm + P::V;  // [buf * 128 + 0..63] = v, [buf * 128 + 64..127] = p
    double* red = sm + P::RED;
    double* br = sm + P::BR;
    __shared__ int status;

    // ---- load the upper triangle, mirror, scale ---------------------------------
    for (int x = tid; x < n * n; x += kThreads) {
        const int i = x / n, j = x - i * n;
        const int a = i <= j ? i : j, b = i <= j ? j : i;
        A[i * kLd + j] = scale * G[(int64_t)a * ldg + b];
    }
    if (tid == 0) status = 0;
    __syncthreads();
    EIGH_CLK(0);

    // ---- 1. tridiagonalisation ---------------------------------------------------
    // Step j: H_j = I - tau_j v v^T (v_0 = 1) zeroes A[j+2.., j]; v_j[i] (i >= 1)
    // is stored at A[j+1+i][j].  Warp 0 makes the reflector of step j + 1 from
    // column j + 1, which it updates itself; warps 1..7 update the block
    // A[j+2..][j+2..] (the next step's A22).
    if (warp == 0) {
        if (n >= 2) {
            const int m = n - 1;
            double xr[2], s = 0.0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int r = lane + 32 * h;
                xr[h] = r < m ? A[(1 + r) * kLd] : 0.0;
                if (r >= 1 && r < m) s = fma(xr[h], xr[h], s);
            }
            s = warp_sum(s);
            const double alpha = __shfl_sync(0xffffffffu, xr[0], 0);
            double beta, tj, sc;
            reflector(alpha, s, beta, tj, sc);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int r = lane + 32 * h;
                if (r < m) {
                    const double vi = r == 0 ? 1.0 : xr[h] * sc;
                    vbuf[r] = vi;
                    if (r > 0) A[(1 + r) * kLd] = vi;
                }
            }
            if (lane == 0) {
                tau[0] = tj;
                e[0] = beta;
                d[0] = A[0];
            }
        } else if (lane == 0) {
            d[0] = A[0];
            e[0] = 0.0;
        }
    }
    __syncthreads();
    for (int j = 0; j + 1 < n; ++j) {
        const int m = n - j - 1;  // rows of A22 = A[j+1..][j+1..]
        const int cb = j & 1;
        const double* v = vbuf + cb * 128;
        double* p = vbuf + cb * 128 + 64;
        const double tj = tau[j];
        double K = 0.0;
        if (tj != 0.0) {
            // p = tau A22 v: 4 threads per row, columns q, q + 4, ...
            const int r = tid >> 2, q = tid & 3;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            if (r < m) {
                const double* Ar = A + (j + 1 + r) * kLd + j + 1;
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                    const int c = q + 4 * t;
                    if (c < m) acc[t & 3] = fma(Ar[c], v[c], acc[t & 3]);
                }
            }
            double a = (acc[0] + acc[1]) + (acc[2] + acc[3]);
            a += __shfl_xor_sync(0xffffffffu, a, 1);
            a += __shfl_xor_sync(0xffffffffu, a, 2);
            const double pr = tj * a;
            double pv = 0.0;
            if (r < m && q == 0) {
                p[r] = pr;
                pv = pr * v[r];
            }
            pv += __shfl_xor_sync(0xffffffffu, pv, 4);
            pv += __shfl_xor_sync(0xffffffffu, pv, 8);
            pv += __shfl_xor_sync(0xffffffffu, pv, 16);
            if (lane == 0) red[warp] = pv;
            __syncthreads();
            K = ((red[0] + red[1]) + (red[2] + red[3])) + ((red[4] + red[5]) + (red[6] + red[7]));
            K *= -0.5 * tj;
        }
        if (warp > 0) {
            if (tj != 0.0) {
                // A[r][c] -= v_r w_c + w_r v_c, w = p + K v, rows / cols >= 1 of A22
                const int t2 = tid - 32;
                const int c0 = 1 + (t2 & 3);
                double vc[16], wc[16];
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                    const int c = c0 + 4 * t;
                    vc[t] = c < m ? v[c] : 0.0;
                    wc[t] = c < m ? fma(K, vc[t], p[c]) : 0.0;
                }
                for (int rr = 1 + (t2 >> 2); rr < m; rr += 56) {
                    const double vr = v[rr], wr = fma(K, vr, p[rr]);
                    double* Ar = A + (j + 1 + rr) * kLd + j + 1;
#pragma unroll
                    for (int t = 0; t < 16; ++t) {
                        const int c = c0 + 4 * t;
                        if (c < m) Ar[c] = fma(-vr, wc[t], fma(-wr, vc[t], Ar[c]));
                    }
                }
            }
        } else if (m >= 2) {
            // column j + 1 of the updated A22 (rows j+1..n-1): x_r = A - v_r w_0 - w_r v_0
            const int nb = cb ^ 1;
            const double v0 = v[0], w0 = fma(K, v0, p[0]);
            double xr[2], s = 0.0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int rr = lane + 32 * h;
                double x = 0.0;
                if (rr < m) {
                    x = A[(j + 1 + rr) * kLd + j + 1];
                    if (tj != 0.0) {
                        const double vr = v[rr], wr = fma(K, vr, p[rr]);
                        x = fma(-vr, w0, fma(-wr, v0, x));
                    }
                }
                xr[h] = x;
                if (rr >= 2 && rr < m) s = fma(x, x, s);
            }
            s = warp_sum(s);
            const double dd = __shfl_sync(0xffffffffu, xr[0], 0);     // A[j+1][j+1]
            const double alpha = __shfl_sync(0xffffffffu, xr[0], 1);  // A[j+2][j+1]
            double beta, tn, sc;
            reflector(alpha, s, beta, tn, sc);
            double* vn = vbuf + nb * 128;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int rr = lane + 32 * h;  // reflector index rr - 1
                if (rr >= 1 && rr < m) {
                    const double vi = rr == 1 ? 1.0 : xr[h] * sc;
                    vn[rr - 1] = vi;
                    if (rr >= 2) A[(j + 1 + rr) * kLd + j + 1] = vi;
                }
            }
            if (lane == 0) {
                tau[j + 1] = tn;
                e[j + 1] = beta;
                d[j + 1] = dd;
            }
        } else if (lane == 0) {
            // last step (m == 1): the final diagonal entry
            double x = A[(j + 1) * kLd + j + 1];
            if (tj != 0.0) {
                const double v0 = v[0], w0 = fma(K, v0, p[0]);
                x = fma(-v0, w0, fma(-w0, v0, x));
            }
            d[j + 1] = x;
            e[j + 1] = 0.0;
            tau[j + 1] = 0.0;
        }
        __syncthreads();
    }
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

    // ---- 3. inverse iteration: thread t < kk, eigenvalue lam[t] -------------------
    if (tid < kk) {
        const int t = tid;
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
            double u1, u2, ru, l;
            if (fabs(a) >= fabs(c)) {
                const double ui = fabs(a) < pivmin ? (a < 0.0 ? -pivmin : pivmin) : a;
                ru = rcp_nr(ui);
                l = c * ru;
                u1 = bsup;
                u2 = 0.0;
                a = fma(-l, bsup, a1);
                bsup = b1;
                ynext = fma(-l, ycur, ynext);
            } else {
                piv |= 1ull << i;
                ru = rcp_nr(c);
                l = a * ru;
                u1 = a1;
                u2 = b1;
                a = fma(-l, a1, bsup);
                bsup = -l * b1;
                const double yi = ynext;  // rows i and i+1 swap
                ynext = fma(-l, yi, ycur);
                ycur = yi;
            }
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
    // R[a][c] = B[a][c] br[64 + a].  A column keeping less than 1e-3 of its
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
    for (int jj = 0; jj < kk; ++jj) {
        const double djj = B[jj * kLd + jj];
        if (!(djj > 1e-6 * br[jj])) {  // uniform
            if (tid == 0) status = 2;
            break;
        }
        const double inv2 = rcp_nr(djj);
        if (tid == 0) br[64 + jj] = rsqrt_nr(djj);
        const int w = kk - jj - 1;
        for (int x = tid; x < w * w; x += kThreads) {
            const int c = jj + 1 + x / w, c2 = jj + 1 + x % w;
            if (c2 >= c) B[c * kLd + c2] = fma(-B[jj * kLd + c] * inv2, B[jj * kLd + c2], B[c * kLd + c2]);
        }
        __syncthreads();
    }
    __syncthreads();
    if (status) return status;
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

    // ---- 4b. back to G's basis: X = H_0 H_1 ... H_{n-3} Z ------------------------
    // warp w owns columns 4w..4w+3 (+32); lane = (column 4w + (lane >> 3), row
    // part lane & 7), rows part + 8u.  No CTA barrier: columns are disjoint.
    for (int c0 = 4 * warp; c0 < kk; c0 += 32) {
        const int c = c0 + (lane >> 3), part = lane & 7;
        const bool cok = c < kk;
        for (int jr = n - 3; jr >= 0; --jr) {
            const double tj = tau[jr];
            if (tj == 0.0) continue;
            const int m = n - jr - 1;
            const double* vcol = A + (jr + 1) * kLd + jr;  // v_i at vcol[i * kLd], v_0 = 1
            double* zc = Z + (jr + 1) * kLdZ + c;
            double vv[8], zz[8], s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = part + 8 * u;
                vv[u] = i < m ? (i == 0 ? 1.0 : vcol[i * kLd]) : 0.0;
                zz[u] = (i < m && cok) ? zc[i * kLdZ] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; u += 2) {
                s0 = fma(vv[u], zz[u], s0);
                s1 = fma(vv[u + 1], zz[u + 1], s1);
            }
            double s = s0 + s1;
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            s += __shfl_xor_sync(0xffffffffu, s, 2);
            s += __shfl_xor_sync(0xffffffffu, s, 4);
            s *= tj;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = part + 8 * u;
                if (i < m && cok) zc[i * kLdZ] = fma(-s, vv[u], zz[u]);
            }
            __syncwarp();
        }
    }
    __syncthreads();
    EIGH_CLK(5);
    EIGH_CLK(6);
    return 0;
}

}  // namespace eigh
}  // namespace zsvd
