// eigh_warp.cuh — the kk <= 24 leading eigenpairs of a symmetric n x n matrix
// (n <= 64) on ONE WARP, built for throughput: a storage flush has hundreds of
// independent block Grams (svd_engine.cu eigen phase), so each gets a warp and
// ~53 KB of shared memory and four of them share an SM — all 500 blocks of a
// cfg2 flush are resident at once.  (eigh.cuh is the latency build of the same
// algorithm: one problem on a whole CTA with the matrix in registers.)
//
//   1. Householder tridiagonalisation (dsytd2 order, both triangles kept): lane
//      l owns rows l and l + 32 in shared memory (row stride 66, 16-byte loads);
//      a step is the reflector (one warp reduction), p = tau A v, w, and the
//      rank-2 update — no barrier but __syncwarp.  Reflector j goes to row j
//      (dead once eliminated), contiguous for the back-transform.
//   2. eigenvalue g on lane g: a 32-point Sturm scan brackets every eigenvalue,
//      then trisection (two independent division-free recurrences per lane,
//      power-of-two renormalised) to 4 eps ||T||.
//   3. inverse iteration on lane g (dgttrf with partial pivoting, two solves),
//      factors in local memory.
//   4. residual check, Cholesky QR of the vectors (a pivot below 1e-6 fails),
//      back-transform through the stored reflectors (lane = column).
// Returns 0 on success; nonzero = the caller keeps its own path.
#pragma once

#include <cfloat>
#include <cstdint>

namespace zsvd {
namespace eighw {

constexpr int LDA = 66;   // row stride of A: rows 16-byte aligned, a quarter-warp's 16-byte loads hit 8 bank groups
constexpr int LDZ = 66;   // stride of an eigenvector (column-major Z), same property
constexpr int KMAX = 24;
// shared doubles: A | Z | B (KMAX x 25) | d e ee tau (64 each) | v w (64 each) | lam (32) | cnt (32 ints)
constexpr int OFF_Z = 64 * LDA;
constexpr int OFF_B = OFF_Z + KMAX * LDZ;
constexpr int OFF_D = OFF_B + KMAX * 25;
constexpr int OFF_V = OFF_D + 4 * 64;
constexpr int OFF_L = OFF_V + 2 * 64;
constexpr int TOTAL = OFF_L + 32 + 16;
constexpr int bytes() { return TOTAL * 8; }

__device__ __forceinline__ double wsum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}
__device__ __forceinline__ double rcp_nr(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x, y, 1.0);
    return fma(y * e, 1.0 + e, y);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x * y, y, 1.0);
    return fma(y * e, fma(0.375, e, 0.5), y);
}
__device__ __forceinline__ double renorm(double a, double b) {
    const int ea = (__double2hiint(a) >> 20) & 0x7ff, eb = (__double2hiint(b) >> 20) & 0x7ff;
    const int e = ea > eb ? ea : eb;
    return e == 0 ? 1.0 : __hiloint2double((2046 - e) << 20, 0);
}
__device__ __forceinline__ double start_entry(int i, int t) {
    unsigned h = (unsigned)(i * 0x9E3779B1u) ^ (unsigned)((t + 1) * 0x85EBCA77u);
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    const double u = 0.5 + (double)(h & 0xFFFFFu) * (1.0 / 1048576.0);
    return (h & 0x100000u) ? -u : u;
}

// Eigenvalues of T below x (Sturm count), d / ee = e^2 in shared memory.
__device__ __forceinline__ int sturm(const double* d, const double* ee, int n, double x) {
    double pa = 1.0, pb = d[0] - x;
    int sg = __double2hiint(pb) >> 31;
    int cn = sg;
    int i = 1;
    for (; i + 8 <= n; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double q = fma(d[i + u] - x, pb, -ee[i + u - 1] * pa);
            const int s2 = __double2hiint(q) >> 31;
            cn += s2 ^ sg;
            sg = s2;
            pa = pb;
            pb = q;
        }
        const double f = renorm(pa, pb);
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
    return -cn;
}

// Two Sturm counts at once (independent recurrences interleaved: the chain is
// one dependent DFMA per term).
__device__ __forceinline__ void sturm2(const double* d, const double* ee, int n, const double (&x)[2], int (&out)[2]) {
    constexpr int NC = 2;
    double pa[NC], pb[NC];
    int sg[NC], cn[NC];
#pragma unroll
    for (int m = 0; m < NC; ++m) {
        pa[m] = 1.0;
        pb[m] = d[0] - x[m];
        sg[m] = __double2hiint(pb[m]) >> 31;
        cn[m] = sg[m];
    }
    int i = 1;
    for (; i + 8 <= n; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double di = d[i + u], e2 = ee[i + u - 1];
#pragma unroll
            for (int m = 0; m < NC; ++m) {
                const double q = fma(di - x[m], pb[m], -e2 * pa[m]);
                const int s2 = __double2hiint(q) >> 31;
                cn[m] += s2 ^ sg[m];
                sg[m] = s2;
                pa[m] = pb[m];
                pb[m] = q;
            }
        }
#pragma unroll
        for (int m = 0; m < NC; ++m) {
            const double f = renorm(pa[m], pb[m]);
            pa[m] *= f;
            pb[m] *= f;
        }
    }
    for (; i < n; ++i) {
        const double di = d[i], e2 = ee[i - 1];
#pragma unroll
        for (int m = 0; m < NC; ++m) {
            const double q = fma(di - x[m], pb[m], -e2 * pa[m]);
            const int s2 = __double2hiint(q) >> 31;
            cn[m] += s2 ^ sg[m];
            sg[m] = s2;
            pa[m] = pb[m];
            pb[m] = q;
        }
    }
#pragma unroll
    for (int m = 0; m < NC; ++m) out[m] = -cn[m];
}

// G: n x n, row-major, ld ldg even and >= 64 columns readable, both triangles
// stored, 16-byte aligned; scale: power of two with
// max |scale G| ~ 1.  X (n x kk, ld ldx) receives the orthonormal eigenvectors of
// the kk largest eigenvalues (descending).  One warp; sm: bytes().
__device__ int eigh_warp_top(const double* __restrict__ G, int ldg, int n, int kk, double scale, double* sm,
                             double* __restrict__ X, int ldx, long long* clk = nullptr) {
    const int lane = threadIdx.x & 31;
#define EW_CLK(i) if (clk && lane == 0) clk[i] = clock64()
    EW_CLK(0);
    double* A = sm;
    double* Z = sm + OFF_Z;
    double* B = sm + OFF_B;
    double* d = sm + OFF_D;
    double* e = d + 64;
    double* ee = d + 128;
    double* tau = d + 192;
    double* vs = sm + OFF_V;
    double* wv = vs + 64;
    double* lam = sm + OFF_L;
    int* cnt = reinterpret_cast<int*>(lam + 32);

    // (both triangles of G are stored: rows are read as they lie, 16 bytes per lane)
    // 16 rows' loads are issued before their stores (a load is not hoisted over a store
    // through a generic pointer: one L2 round trip per row otherwise, 22K cycles)
    for (int i0 = 0; i0 < 64; i0 += 16) {
        const int j = 2 * lane;
        double2 gv[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            gv[u] = make_double2(0.0, 0.0);
            if (i0 + u < n) gv[u] = __ldg(reinterpret_cast<const double2*>(G + (int64_t)(i0 + u) * ldg + j));
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            A[(i0 + u) * LDA + j] = j < n ? scale * gv[u].x : 0.0;
            A[(i0 + u) * LDA + j + 1] = j + 1 < n ? scale * gv[u].y : 0.0;
        }
    }
    for (int i = lane; i < 64; i += 32) d[i] = e[i] = tau[i] = 0.0;
    __syncwarp();

    EW_CLK(1);
    // ---- 1. tridiagonalisation ---------------------------------------------------
    const int r0 = lane, r1 = lane + 32;
    double* a0 = A + r0 * LDA;
    double* a1 = A + r1 * LDA;
    for (int j = 0; j + 2 < n; ++j) {
        // reflector from column j below the diagonal (= row j by symmetry; own rows)
        const double x0 = (r0 > j && r0 < n) ? a0[j] : 0.0, x1 = (r1 > j && r1 < n) ? a1[j] : 0.0;
        const double x0d = a0[j & 63], x1d = a1[j & 63];  // (the owner of row j keeps its diagonal entry)
        const double alpha = A[(j + 1) * LDA + j];  // (read by every lane before the shuffles below)
        const double ssq = wsum((r0 > j + 1 ? x0 * x0 : 0.0) + (r1 > j + 1 ? x1 * x1 : 0.0));
        double beta = alpha, tj = 0.0, sc = 0.0;
        if (ssq > 0.0) {
            const double h = fma(alpha, alpha, ssq);
            const double nrm = h * rsqrt_nr(h);
            beta = alpha >= 0.0 ? -nrm : nrm;
            tj = fma(-alpha, rcp_nr(beta), 1.0);
            sc = rcp_nr(alpha - beta);
        }
        const double v0 = r0 <= j ? 0.0 : (r0 == j + 1 ? 1.0 : x0 * sc);
        const double v1 = (r1 <= j || r1 >= n) ? 0.0 : (r1 == j + 1 ? 1.0 : x1 * sc);
        vs[r0] = v0;
        vs[r1] = v1;
        A[j * LDA + r0] = v0;  // reflector storage: row j (dead from here on), contiguous
        A[j * LDA + r1] = v1;
        if (lane == 0) {
            e[j] = beta;
            tau[j] = tj;
        }
        if (lane == (j & 31)) d[j] = j < 32 ? x0d : x1d;
        __syncwarp();
        if (tj != 0.0) {
            // p = tau A v over the trailing block (own two rows; whole groups of 8 columns:
            // v is zero up to column j), 16-byte loads, 16 chains
            double2 s0a = make_double2(0.0, 0.0), s0b = s0a, s1a = s0a, s1b = s0a;
            double2 s0c = s0a, s0d = s0a, s1c = s0a, s1d = s0a;
            for (int c = (j + 1) & ~7; c < 64; c += 8) {
                double2 vv[4], q0[4], q1[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    vv[u] = *reinterpret_cast<const double2*>(vs + c + 2 * u);
                    q0[u] = *reinterpret_cast<const double2*>(a0 + c + 2 * u);
                    q1[u] = *reinterpret_cast<const double2*>(a1 + c + 2 * u);
                }
                s0a.x = fma(q0[0].x, vv[0].x, s0a.x);
                s0a.y = fma(q0[0].y, vv[0].y, s0a.y);
                s0b.x = fma(q0[1].x, vv[1].x, s0b.x);
                s0b.y = fma(q0[1].y, vv[1].y, s0b.y);
                s0c.x = fma(q0[2].x, vv[2].x, s0c.x);
                s0c.y = fma(q0[2].y, vv[2].y, s0c.y);
                s0d.x = fma(q0[3].x, vv[3].x, s0d.x);
                s0d.y = fma(q0[3].y, vv[3].y, s0d.y);
                s1a.x = fma(q1[0].x, vv[0].x, s1a.x);
                s1a.y = fma(q1[0].y, vv[0].y, s1a.y);
                s1b.x = fma(q1[1].x, vv[1].x, s1b.x);
                s1b.y = fma(q1[1].y, vv[1].y, s1b.y);
                s1c.x = fma(q1[2].x, vv[2].x, s1c.x);
                s1c.y = fma(q1[2].y, vv[2].y, s1c.y);
                s1d.x = fma(q1[3].x, vv[3].x, s1d.x);
                s1d.y = fma(q1[3].y, vv[3].y, s1d.y);
            }
            s0a.x += s0c.x;
            s0a.y += s0c.y;
            s0b.x += s0d.x;
            s0b.y += s0d.y;
            s1a.x += s1c.x;
            s1a.y += s1c.y;
            s1b.x += s1d.x;
            s1b.y += s1d.y;
            const double p0 = r0 > j ? tj * ((s0a.x + s0a.y) + (s0b.x + s0b.y)) : 0.0;
            const double p1 = (r1 > j && r1 < n) ? tj * ((s1a.x + s1a.y) + (s1b.x + s1b.y)) : 0.0;
            const double K = -0.5 * tj * wsum(p0 * v0 + p1 * v1);
            const double w0 = fma(K, v0, p0), w1 = fma(K, v1, p1);
            wv[r0] = w0;
            wv[r1] = w1;
            __syncwarp();
            // A -= v w^T + w v^T (trailing block, own rows; v, w are zero up to column j and
            // beyond n, so whole groups of 8 columns are updated).  Loads of a group are issued
            // before its stores: the compiler cannot hoist shared-memory loads over the
            // stores of a previous iteration (same base pointer), which had serialised this loop.
            const bool u0 = r0 > j, u1 = r1 > j && r1 < n;
            for (int c2 = (j + 1) & ~7; c2 < 64; c2 += 8) {
                double2 wc[4], vc[4], q0[4], q1[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    wc[u] = *reinterpret_cast<const double2*>(wv + c2 + 2 * u);
                    vc[u] = *reinterpret_cast<const double2*>(vs + c2 + 2 * u);
                    q0[u] = *reinterpret_cast<const double2*>(a0 + c2 + 2 * u);
                    q1[u] = *reinterpret_cast<const double2*>(a1 + c2 + 2 * u);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    q0[u].x = fma(-v0, wc[u].x, fma(-w0, vc[u].x, q0[u].x));
                    q0[u].y = fma(-v0, wc[u].y, fma(-w0, vc[u].y, q0[u].y));
                    q1[u].x = fma(-v1, wc[u].x, fma(-w1, vc[u].x, q1[u].x));
                    q1[u].y = fma(-v1, wc[u].y, fma(-w1, vc[u].y, q1[u].y));
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (u0) *reinterpret_cast<double2*>(a0 + c2 + 2 * u) = q0[u];
                    if (u1) *reinterpret_cast<double2*>(a1 + c2 + 2 * u) = q1[u];
                }
            }
        }
        __syncwarp();
    }
    if (lane == 0) {
        if (n >= 2) {
            d[n - 2] = A[(n - 2) * LDA + n - 2];
            e[n - 2] = A[(n - 1) * LDA + n - 2];
        }
        d[n - 1] = A[(n - 1) * LDA + n - 1];
        e[n - 1] = 0.0;
    }
    __syncwarp();
    for (int i = lane; i < 64; i += 32) ee[i] = e[i] * e[i];
    __syncwarp();
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
        glo = lo - 4.0 * DBL_EPSILON * tn - 1e-300;
        ghi = hi + 4.0 * DBL_EPSILON * tn + 1e-300;
    }
    const double tnorm = fmax(fabs(glo), fabs(ghi));
    if (!(tnorm < 1e300)) return 1;

    EW_CLK(2);
    // ---- 2. eigenvalues: one 32-point scan, then bisection on lane g ------------
    const double h33 = (ghi - glo) * (1.0 / 33.0);
    cnt[lane] = sturm(d, ee, n, fma((double)(lane + 1), h33, glo));
    __syncwarp();
    const int g = lane;
    const bool mine = g < kk;
    double lg = 0.0;
    {
        const int target = n - 1 - (mine ? g : 0);  // ascending index
        int nt = 0;                                 // scan points at or below the eigenvalue
        for (int m = 0; m < 32; ++m) nt += cnt[m] <= target;
        double a = nt > 0 ? fma((double)nt, h33, glo) : glo;
        double b = nt < 32 ? fma((double)(nt + 1), h33, glo) : ghi;
        // trisection: two independent recurrences per lane hide the DFMA latency; more
        // points per step only add issue slots (measured: 5-way 81K cycles)
        int iters = 0;
        for (double w = h33; w > 4.0 * DBL_EPSILON * tnorm && iters < 60; w *= (1.0 / 3.0)) ++iters;
        for (int it = 0; it < iters; ++it) {
            const double h = (b - a) * (1.0 / 3.0);
            double x[2];
            int c2[2];
            x[0] = a + h;
            x[1] = fma(2.0, h, a);
            sturm2(d, ee, n, x, c2);
            const int k2 = (c2[0] <= target) + (c2[1] <= target);
            const double na = k2 > 0 ? fma((double)k2, h, a) : a;
            const double nb = k2 < 2 ? fma((double)(k2 + 1), h, a) : b;
            a = na;
            b = nb;
        }
        lg = 0.5 * (a + b);
        if (mine) lam[g] = lg;
    }
    __syncwarp();

    EW_CLK(3);
    // ---- 3. inverse iteration on lane g ---------------------------------------------
    bool bad = false;
    if (mine) {
        double Ud[64], U1[64], U2[64], Lm[64];
        uint64_t piv = 0;
        const double pivmin = DBL_EPSILON * tnorm + 1e-300;
        double* z = Z + g * LDZ;
        double a = d[0] - lg, bsup = n > 1 ? e[0] : 0.0;
        double ycur = start_entry(0, g);
        for (int i = 0; i + 1 < n; ++i) {
            const double c = e[i], a1v = d[i + 1] - lg, b1 = i + 2 < n ? e[i + 1] : 0.0;
            double ynext = start_entry(i + 1, g);
            // branch-free (every lane pivots on its own rows, so a branch would run both
            // sides on most rows): the same operations as the two cases of dgttrf,
            // operands picked by selects
            const bool keep = fabs(a) >= fabs(c);
            const double ui = fabs(a) < pivmin ? (a < 0.0 ? -pivmin : pivmin) : a;
            const double ru = rcp_nr(keep ? ui : c);
            const double l = (keep ? c : a) * ru;
            const double u1 = keep ? bsup : a1v;
            const double u2 = keep ? 0.0 : b1;
            a = fma(-l, keep ? bsup : a1v, keep ? a1v : bsup);
            bsup = keep ? b1 : -l * b1;
            const double ykeep = keep ? ycur : ynext;  // rows i, i + 1 swap on a pivot
            ynext = fma(-l, ykeep, keep ? ynext : ycur);
            ycur = ykeep;
            piv |= keep ? 0ull : (1ull << i);
            Ud[i] = ru;
            U1[i] = u1;
            U2[i] = u2;
            Lm[i] = l;
            z[i] = ycur;
            ycur = ynext;
        }
        {
            const double ui = fabs(a) < pivmin ? (a < 0.0 ? -pivmin : pivmin) : a;
            Ud[n - 1] = rcp_nr(ui);
            U1[n - 1] = 0.0;
            U2[n - 1] = 0.0;
            z[n - 1] = ycur;
        }
        for (int sweep = 0; sweep < 2; ++sweep) {
            if (sweep == 1) {
                double xi = z[0];
                for (int i = 0; i + 1 < n; ++i) {
                    double x1 = z[i + 1];
                    if ((piv >> i) & 1) {
                        const double tmp = xi;
                        xi = x1;
                        x1 = tmp;
                    }
                    z[i] = xi;
                    xi = fma(-Lm[i], xi, x1);
                }
                z[n - 1] = xi;
            }
            double z2 = 0.0, z1 = 0.0, big = 0.0;
            for (int i = n - 1; i >= 0; --i) {
                const double zi = fma(-U2[i], z2, fma(-U1[i], z1, z[i])) * Ud[i];
                z[i] = zi;
                big = fmax(big, fabs(zi));
                z2 = z1;
                z1 = zi;
            }
            if (sweep == 0) {
                const double inv = big > 0.0 ? rcp_nr(big) : 1.0;
                for (int i = 0; i < n; ++i) z[i] *= inv;
            }
        }
        // normalise; residual in T's basis
        double nn = 0.0;
        for (int i = 0; i < n; ++i) nn = fma(z[i], z[i], nn);
        if (!(nn > 0.0) || !(nn < 1e300)) {
            bad = true;
        } else {
            const double rn = rsqrt_nr(nn);
            double worst = 0.0, zm = 0.0, zc = z[0] * rn;
            for (int i = 0; i < n; ++i) {
                const double zn = i + 1 < n ? z[i + 1] * rn : 0.0;
                double r = (d[i] - lg) * zc;
                if (i > 0) r = fma(e[i - 1], zm, r);
                if (i + 1 < n) r = fma(e[i], zn, r);
                worst = fmax(worst, fabs(r));
                z[i] = zc;
                zm = zc;
                zc = zn;
            }
            if (!(worst <= 1e-11 * fmax(tnorm, 1e-300))) bad = true;
        }
    }
    if (__any_sync(0xffffffffu, bad)) return 2;
    __syncwarp();

    EW_CLK(4);
    // ---- 4a. Cholesky QR of Z, a second time when the first met a pivot below 1e-2 (one
    // pass leaves an orthogonality error ~eps / smallest pivot: the vectors of an
    // eigenvalue cluster come out of inverse iteration far from orthogonal) -----------
    for (int pass = 0; pass < 2; ++pass) {
        for (int x = lane; x < kk * kk; x += 32) {
            const int ia = x / kk, ib = x - ia * kk;
            if (ia <= ib) {
                const double* za = Z + ia * LDZ;
                const double* zb = Z + ib * LDZ;
                double s0 = 0.0, s1 = 0.0;
                int i = 0;
                for (; i + 1 < n; i += 2) {
                    s0 = fma(za[i], zb[i], s0);
                    s1 = fma(za[i + 1], zb[i + 1], s1);
                }
                if (i < n) s0 = fma(za[i], zb[i], s0);
                B[ia * 25 + ib] = s0 + s1;
            }
        }
        __syncwarp();
        bool chol_bad = false;
        double minpiv = 1.0;
        for (int jj = 0; jj < kk; ++jj) {  // right-looking, lane = column (kk <= 32)
            const double djj = B[jj * 25 + jj];
            if (!(djj > 1e-6)) {  // (unit vectors) uniform
                chol_bad = true;
                break;
            }
            minpiv = fmin(minpiv, djj);
            const double inv2 = rcp_nr(djj);
            const double bjl = lane < kk ? B[jj * 25 + lane] : 0.0;
            for (int c = jj + 1; c < kk; ++c) {
                const double f = B[jj * 25 + c] * inv2;
                if (lane >= c && lane < kk) B[c * 25 + lane] = fma(-f, bjl, B[c * 25 + lane]);
            }
            __syncwarp();
        }
        if (chol_bad) return 3;
        // R[a][c] = B[a][c] / sqrt(B[a][a]); Z <- Z R^-1, lane = row (two rows each)
        for (int a = lane; a < kk; a += 32) lam[a] = rsqrt_nr(B[a * 25 + a]);  // 1 / R_aa (lam is free now)
        __syncwarp();
        for (int rr = 0; rr < 2; ++rr) {
            const int i = lane + 32 * rr;
            if (i < n) {
                double zr[KMAX];
    #pragma unroll
                for (int c = 0; c < KMAX; ++c) zr[c] = c < kk ? Z[c * LDZ + i] : 0.0;
    #pragma unroll
                for (int c = 0; c < KMAX; ++c) {
                    if (c < kk) {  // uniform
                        double s0 = zr[c], s1 = 0.0;
    #pragma unroll
                        for (int a = 0; a < c; ++a) {
                            const double rac = B[a * 25 + c] * lam[a];
                            if (a & 1) s1 = fma(-zr[a], rac, s1);
                            else s0 = fma(-zr[a], rac, s0);
                        }
                        zr[c] = (s0 + s1) * lam[c];
                    }
                }
    #pragma unroll
                for (int c = 0; c < KMAX; ++c)
                    if (c < kk) Z[c * LDZ + i] = zr[c];
            }
        }
        __syncwarp();

        if (minpiv >= 1e-2) break;  // uniform
    }
    EW_CLK(5);
    // ---- 4b. back-transform X = H_0 ... H_{n-3} Z, lane = column; reflector j is row j
    // of A (zero up to column j, one at j + 1, zero beyond n): 16-byte broadcast loads
    {
        // (every lane runs the loop — the loads are broadcasts — lanes beyond kk on zeros)
        const double* zc = Z + (mine ? g : 0) * LDZ;
        double z[64];
#pragma unroll
        for (int i = 0; i < 64; ++i) z[i] = (mine && i < n) ? zc[i] : 0.0;
        for (int j = n - 3; j >= 0; --j) {
            const double tj = tau[j];
            if (tj == 0.0) continue;  // uniform
            const double* v = A + j * LDA;
            // (v is zero up to column j: the whole row is used, branch-free, so the loads
            // of a phase are issued together; eight accumulation chains)
            double sa[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) sa[u] = 0.0;
#pragma unroll
            for (int r = 0; r < 64; r += 8) {
                const double2 v0 = *reinterpret_cast<const double2*>(v + r);
                const double2 v1 = *reinterpret_cast<const double2*>(v + r + 2);
                const double2 v2 = *reinterpret_cast<const double2*>(v + r + 4);
                const double2 v3 = *reinterpret_cast<const double2*>(v + r + 6);
                sa[0] = fma(v0.x, z[r], sa[0]);
                sa[1] = fma(v0.y, z[r + 1], sa[1]);
                sa[2] = fma(v1.x, z[r + 2], sa[2]);
                sa[3] = fma(v1.y, z[r + 3], sa[3]);
                sa[4] = fma(v2.x, z[r + 4], sa[4]);
                sa[5] = fma(v2.y, z[r + 5], sa[5]);
                sa[6] = fma(v3.x, z[r + 6], sa[6]);
                sa[7] = fma(v3.y, z[r + 7], sa[7]);
            }
            const double f = -tj * (((sa[0] + sa[1]) + (sa[2] + sa[3])) + ((sa[4] + sa[5]) + (sa[6] + sa[7])));
#pragma unroll
            for (int r = 0; r < 64; r += 8) {
                const double2 v0 = *reinterpret_cast<const double2*>(v + r);
                const double2 v1 = *reinterpret_cast<const double2*>(v + r + 2);
                const double2 v2 = *reinterpret_cast<const double2*>(v + r + 4);
                const double2 v3 = *reinterpret_cast<const double2*>(v + r + 6);
                z[r] = fma(f, v0.x, z[r]);
                z[r + 1] = fma(f, v0.y, z[r + 1]);
                z[r + 2] = fma(f, v1.x, z[r + 2]);
                z[r + 3] = fma(f, v1.y, z[r + 3]);
                z[r + 4] = fma(f, v2.x, z[r + 4]);
                z[r + 5] = fma(f, v2.y, z[r + 5]);
                z[r + 6] = fma(f, v3.x, z[r + 6]);
                z[r + 7] = fma(f, v3.y, z[r + 7]);
            }
        }
        if (mine) {
            double* zo = Z + g * LDZ;
#pragma unroll
            for (int i = 0; i < 64; ++i) zo[i] = z[i];
        }
    }
    __syncwarp();
    for (int x = lane; x < n * kk; x += 32) {
        const int i = x / kk, t = x - i * kk;
        X[(int64_t)i * ldx + t] = Z[t * LDZ + i];
    }
    EW_CLK(6);
#undef EW_CLK
    return 0;
}

}  // namespace eighw
}  // namespace zsvd
