// wide_engine.cu — batched fp64 thin SVD for work matrices wider than the
// shared-memory engine (64 < q <= kWideMax): the cfg3 / cfg5 blocks
// (4000 x 256, 8192 x 1024), their open tails, and stitches of K x c stacks
// (query.hpp:95-144) with c = 256 / 1024.
//
// W (p x q, p >= q) is A or A^T as in svd_engine.cu.  Each step is one batched
// kernel over the tasks:
//   pass 1  G = W^T W on DMMA; G = V1 diag V1^T by two-sided block Jacobi:
//           the q columns form q/32 blocks, every round pairs the blocks
//           (circle method), each pair's 64 x 64 sub-matrix is diagonalised in
//           shared memory by scalar two-sided Jacobi (rotation T_P), then
//           G <- J^T G J and V <- V J with J = blockdiag(T_P) on DMMA; sweeps of
//           q/32 - 1 rounds repeat until one rotates nothing.  Rotations stop
//           at the Gram's own rounding level (16 eps max_i g_ii).
//   pass 2  Y = W V1 (columns orthogonal to ~eps cond^2), G = Y^T Y recomputed
//           from Y, and the same block Jacobi again (V2), now with small angles
//           and a purely relative threshold: this is one-sided Jacobi on W
//           preconditioned by V1, so sigma and U keep one-sided accuracy
//           (relative error ~ eps sigma_1 / sigma_i, U orthogonal to ~eps).
//   out     sigma = sqrt(diag G) sorted; rank cutoff 1e-12 sigma_1 and
//           truncation (svd.hpp:118-124, 135-164); V = V1 V2_k (times vpre for
//           trims); canonical sign (svd.hpp:179-203); U = Y V2_k Sigma^-1.
//   check   U^T U against the reference's 1e-10 contract (svd.hpp:25).
#include <cfloat>
#include <cstdint>
#include <cstdio>

#include "zsvd_internal.h"

namespace zsvd {
namespace {

constexpr int T = 256;
constexpr int NW = T / 32;

struct WGeo {
    int m, n, p, q, tall;
};

__device__ __forceinline__ WGeo wgeo(const SvdTask& t) {
    WGeo g;
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

__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(a), "l"(gmem));
}
__device__ __forceinline__ void cp_wait_all() {
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// W(i, j) of a task (A or A^T, column scaling applied).
__device__ __forceinline__ double w_elem(const SvdTask& t, bool tall, int i, int j) {
    const int r = tall ? i : j, c = tall ? j : i;
    const double x = t.a[(int64_t)r * t.lda + c];
    return t.colscale ? x * t.colscale[c] : x;
}

}  // namespace

// ---------------------------------------------------------------- layout
int wide_qp(int64_t q_bound) { return (int)((q_bound + 63) / 64 * 64); }

// Per task: G | V (pass rotation) | V1 | M (q x k operands) | Y (p x qp) |
// T (64 x 64 per pair) | sigma | sign | flags | Gram partials.
int64_t wide_ws_doubles(int64_t p_bound, int64_t q_bound, int nsplit) {
    const int64_t qp = wide_qp(q_bound);
    const int64_t nb64 = qp / 64, nbp = nb64 * (nb64 + 1) / 2, npair = qp / 64;
    int64_t w = 4 * qp * qp + p_bound * qp + npair * 4096 + 2 * qp + 16;
    w += 8 * qp + 64 * 6 * qp + 64 * qp + 64 * 64;  // direct route scratch (wide_eig.cuh: weig_doubles)
    if (nsplit > 1) w += (int64_t)nsplit * nbp * 4096;
    return w;
}

namespace {

struct WLay {
    int qp, nb32, npair, nb64, nbp;
    double *g, *v, *v1, *m, *y, *t, *sig, *sgn, *ez, *gp;
    int* flags;      // [0], [1] rotated in sweep parity; [2] done; [3] direct route (wide_eig.cuh)
    double* gscale;  // max diagonal of the pass's initial G
};

__device__ __forceinline__ WLay wlay(const SvdTask& t, const WParams& P) {
    WLay L;
    L.qp = (P.q_bound + 63) / 64 * 64;
    L.nb32 = L.qp / 32;
    L.npair = L.nb32 / 2;
    L.nb64 = L.qp / 64;
    L.nbp = L.nb64 * (L.nb64 + 1) / 2;
    const int64_t q2 = (int64_t)L.qp * L.qp;
    L.g = t.ws;
    L.v = L.g + q2;
    L.v1 = L.v + q2;
    L.m = L.v1 + q2;
    L.y = L.m + q2;
    L.t = L.y + (int64_t)P.p_bound * L.qp;
    L.sig = L.t + (int64_t)L.npair * 4096;
    L.sgn = L.sig + L.qp;
    L.flags = reinterpret_cast<int*>(L.sgn + L.qp);
    L.gscale = L.sgn + L.qp + 8;
    L.ez = L.sgn + L.qp + 16;
    L.gp = L.ez + 8 * (int64_t)L.qp + 64 * 6 * (int64_t)L.qp + 64 * (int64_t)L.qp + 64 * 64;
    return L;
}

// Block pair (I <= J) of the nb upper 64-column blocks from a linear index.
__device__ __forceinline__ void upper_pair(int idx, int nb, int& I, int& J) {
    int r = 0;
    while (idx >= nb - r) {
        idx -= nb - r;
        ++r;
    }
    I = r;
    J = r + idx;
}

// Circle-method pairing of n (even) items, round r in [0, n - 1), slot i in [0, n/2).
__device__ __forceinline__ void circle_pair(int n, int r, int i, int& a, int& b) {
    if (i == 0) {
        a = n - 1;
        b = r;
    } else {
        a = (r + i) % (n - 1);
        b = (r - i + (n - 1)) % (n - 1);
    }
    if (a > b) {
        const int x = a;
        a = b;
        b = x;
    }
}

// Source of a Gram / GEMM left operand: W through w_elem, or a plain row-major
// matrix.
struct Src {
    const double* base;
    int64_t ld;
    int rows, cols;
    bool work;
    bool tall;
};

__device__ __forceinline__ double src_at(const SvdTask& t, const Src& s, int i, int j) {
    if (s.work) return w_elem(t, s.tall, i, j);
    return s.base[(int64_t)i * s.ld + j];
}

constexpr int GCH = 32;        // rows per staged chunk
}  // namespace

// Circle-method pairs of the 64 local columns of a pair solve: round r, slot i
// -> (lo, hi), built once on the host (integer division in the inner loops
// had made the pair solves index-bound).
__constant__ unsigned char c_pair64[63][32][2];


namespace {
constexpr int GLD = 128 + 4;   // staged row: 64 columns of block I | 64 of block J
constexpr int SLD = 65;        // scalar Jacobi arrays (odd stride)
constexpr int MLD = 68;        // DMMA operands in smem (4 mod 16: conflict-free fragments)

}  // namespace

// ---------------------------------------------------------------- kernels
// V <- I (the pass's rotation accumulator); flags reset (grid: qp/64 x tasks).
__global__ void __launch_bounds__(T) wide_init_kernel(SvdTask* tasks, WParams P) {
    SvdTask& t = tasks[blockIdx.y];
    if (t.status != TASK_OK) return;
    const WLay L = wlay(t, P);
    const int r0 = blockIdx.x * 64;
    for (int idx = threadIdx.x; idx < 64 * L.qp; idx += T) {
        const int r = r0 + idx / L.qp, c = idx % L.qp;
        L.v[(int64_t)r * L.qp + c] = r == c ? 1.0 : 0.0;
    }
    if (blockIdx.x == 0 && threadIdx.x < 4) L.flags[threadIdx.x] = 0;
}

// 64 x 64 block (I, J) of S^T S over a row split (grid: nbp * gsplit x tasks).
// src 0: S = W (q columns) into G; 2: S = Y (q columns) into G; 1: S = the
// formed factor (k columns, U for tall tasks, V for wide ones) into the G
// region.  Warp w computes tile row w of the block.
__global__ void __launch_bounds__(T, 2) wide_gram_kernel(SvdTask* tasks, WParams P, int gsplit, int src) {
    extern __shared__ __align__(16) double sm[];
    SvdTask& t = tasks[blockIdx.y];
    if (t.status != TASK_OK || (src == 1 && t.krank <= 0) || (src == 2 && t.onepass)) return;
    const WGeo g = wgeo(t);
    const WLay L = wlay(t, P);
    Src s;
    if (src == 0) s = Src{nullptr, 0, g.p, g.q, true, (bool)g.tall};
    else if (src == 2) s = Src{L.y, L.qp, g.p, g.q, false, true};
    else s = Src{g.tall ? t.u : t.v, g.tall ? t.ldu : t.ldv, g.p, t.krank, false, true};
    const int nb64 = (s.cols + 63) / 64;
    const int bp = blockIdx.x / gsplit, split = blockIdx.x % gsplit;
    int I, J;
    upper_pair(bp, L.nb64, I, J);
    const bool live = J < nb64;
    if (src == 1 && !live) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rps = ((s.rows + gsplit - 1) / gsplit + GCH - 1) / GCH * GCH;
    const int r0 = split * rps, r1 = min(s.rows, r0 + rps);
    double acc[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
    // Fast path (row-major operand, even ld and column count, 16-byte aligned): the
    // chunks go through a 3-deep cp.async ring, so the loads of two chunks are in
    // flight while one is multiplied (the synchronous staging below left the DMMA
    // pipe idle for ~80% of a chunk).
    const double* fbase = s.work ? t.a : s.base;
    const int64_t fld = s.work ? t.lda : s.ld;
    const bool fast = (!s.work || (s.tall && !t.colscale)) && (fld & 1) == 0 && (s.cols & 1) == 0 &&
                      (reinterpret_cast<uintptr_t>(fbase) & 15) == 0;
    if (live && r1 > r0 && fast) {
        const int nch = (r1 - r0 + GCH - 1) / GCH;
        auto issue = [&](int ci) {
            if (ci < nch) {
                double* buf = sm + (ci % 3) * (GCH * GLD);
                const int c0 = r0 + ci * GCH;
                for (int idx = threadIdx.x; idx < GCH * 64; idx += T) {
                    const int r = idx >> 6, cc = 2 * (idx & 63);
                    const int col = cc < 64 ? 64 * I + cc : 64 * J + cc - 64;
                    const int row = c0 + r;
                    double* dst = buf + r * GLD + cc;
                    if (row < r1 && col < s.cols) cp16(dst, fbase + (int64_t)row * fld + col);
                    else dst[0] = dst[1] = 0.0;
                }
            }
            asm volatile("cp.async.commit_group;");
        };
        issue(0);
        issue(1);
        for (int ci = 0; ci < nch; ++ci) {
            issue(ci + 2);
            asm volatile("cp.async.wait_group 2;" ::: "memory");
            __syncthreads();
            const double* buf = sm + (ci % 3) * (GCH * GLD);
#pragma unroll
            for (int h = 0; h < GCH / 4; ++h) {
                const double* rw = buf + (4 * h + (lane & 3)) * GLD;
                const double a = rw[8 * warp + (lane >> 2)];
#pragma unroll
                for (int j = 0; j < 8; ++j) dmma(acc[j][0], acc[j][1], a, rw[64 + 8 * j + (lane >> 2)]);
            }
            __syncthreads();
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    } else if (live && r1 > r0) {
        double* buf = sm;
        const bool rowwise = !s.work || s.tall;
        for (int c0 = r0; c0 < r1; c0 += GCH) {
            // stage rows [c0, c0 + 32) of the two column blocks, coalesced along
            // the source's contiguous direction
            for (int idx = threadIdx.x; idx < GCH * 128; idx += T) {
                int r, cc;
                if (rowwise) {
                    r = idx / 128;
                    cc = idx % 128;
                } else {
                    cc = idx / GCH;
                    r = idx % GCH;
                }
                const int col = cc < 64 ? 64 * I + cc : 64 * J + cc - 64;
                const int row = c0 + r;
                buf[r * GLD + cc] = (row < r1 && col < s.cols) ? src_at(t, s, row, col) : 0.0;
            }
            __syncthreads();
#pragma unroll
            for (int h = 0; h < GCH / 4; ++h) {
                const double* rw = buf + (4 * h + (lane & 3)) * GLD;
                const double a = rw[8 * warp + (lane >> 2)];
#pragma unroll
                for (int j = 0; j < 8; ++j) dmma(acc[j][0], acc[j][1], a, rw[64 + 8 * j + (lane >> 2)]);
            }
            __syncthreads();
        }
    }
    const int rr = 8 * warp + (lane >> 2);
    if (gsplit > 1) {
        double* dst = L.gp + ((int64_t)split * L.nbp + bp) * 4096;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int cc = 8 * j + 2 * (lane & 3);
            dst[rr * 64 + cc] = acc[j][0];
            dst[rr * 64 + cc + 1] = acc[j][1];
        }
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int gi = 64 * I + rr, gj = 64 * J + 8 * j + 2 * (lane & 3);
            L.g[(int64_t)gi * L.qp + gj] = acc[j][0];
            L.g[(int64_t)gi * L.qp + gj + 1] = acc[j][1];
            if (I != J) {
                L.g[(int64_t)gj * L.qp + gi] = acc[j][0];
                L.g[(int64_t)(gj + 1) * L.qp + gi] = acc[j][1];
            }
        }
    }
}

// Sum of the row-split partials of block pair bp (fixed order) into G.
__global__ void __launch_bounds__(T) wide_gram_reduce_kernel(SvdTask* tasks, WParams P, int gsplit, int src) {
    SvdTask& t = tasks[blockIdx.y];
    if (t.status != TASK_OK || (src == 1 && t.krank <= 0) || (src == 2 && t.onepass)) return;
    const WLay L = wlay(t, P);
    const int bp = blockIdx.x;
    int I, J;
    upper_pair(bp, L.nb64, I, J);
    for (int idx = threadIdx.x; idx < 4096; idx += T) {
        double s = 0.0;
        for (int sp = 0; sp < gsplit; ++sp) s += L.gp[((int64_t)sp * L.nbp + bp) * 4096 + idx];
        const int gi = 64 * I + idx / 64, gj = 64 * J + idx % 64;
        L.g[(int64_t)gi * L.qp + gj] = s;
        if (I != J) L.g[(int64_t)gj * L.qp + gi] = s;
    }
}

// Max diagonal of G (scale of pass 1's absolute rotation threshold).
__global__ void __launch_bounds__(T) wide_scale_kernel(SvdTask* tasks, WParams P) {
    __shared__ double red[NW];
    SvdTask& t = tasks[blockIdx.x];
    if (t.status != TASK_OK) return;
    const WGeo g = wgeo(t);
    const WLay L = wlay(t, P);
    double m = 0.0;
    for (int i = threadIdx.x; i < g.q; i += T) m = fmax(m, L.g[(int64_t)i * L.qp + i]);
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 0; w < NW; ++w) m = fmax(m, red[w]);
        *L.gscale = m;
    }
}

// Pair solve of round r (grid: npair x tasks): the 64 x 64 sub-matrix of G on
// blocks (a, b) is diagonalised by cyclic two-sided Jacobi; T_P (row-major,
// G_P' = T_P^T G_P T_P) goes to the workspace.  Rotation when
// |s_ij| > 64 eps sqrt(s_ii s_jj), and in pass 1 also |s_ij| > 16 eps max g_ii
// (below that the Gram's rounding carries no information).
__global__ void __launch_bounds__(T, 3) wide_pair_kernel(SvdTask* tasks, WParams P, int round, int sweep, int pass) {
    extern __shared__ __align__(16) double sm[];
    double* S = sm;             // G_P (ld SLD)
    double* R = sm + 64 * SLD;  // T_P being accumulated
    __shared__ double2 cs[32];
    __shared__ int any_rot, sweep_rot;
    __shared__ unsigned char s_pair[63][32][2];  // per-lane table lookups: shared, not constant
    SvdTask& t = tasks[blockIdx.y];
    if (t.status != TASK_OK) return;
    const WLay L = wlay(t, P);
    if (L.flags[2]) return;  // converged
    for (int i = threadIdx.x; i < 63 * 32 * 2; i += T) (&s_pair[0][0][0])[i] = (&c_pair64[0][0][0])[i];

    const WGeo g = wgeo(t);
    int a, b;
    circle_pair(L.nb32, round, blockIdx.x, a, b);
    double* Tout = L.t + (int64_t)blockIdx.x * 4096;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    auto gidx = [&](int l) { return l < 32 ? 32 * a + l : 32 * b + l - 32; };
    for (int idx = threadIdx.x; idx < 4096; idx += T) {
        const int i = idx / 64, j = idx % 64;
        S[i * SLD + j] = L.g[(int64_t)gidx(i) * L.qp + gidx(j)];
        R[i * SLD + j] = i == j ? 1.0 : 0.0;
    }
    if (threadIdx.x == 0) any_rot = 0;
    __syncthreads();
    const double tol = pass == 1 ? P.tol1 : 64.0 * DBL_EPSILON;
    const double abs_floor = pass == 1 ? 16.0 * DBL_EPSILON * (*L.gscale) : 0.0;
    const bool dead = 32 * a >= g.q && 32 * b >= g.q;
    const int max_inner = P.pad > 0 ? P.pad : 20;
    for (int isw = 0; isw < max_inner && !dead; ++isw) {
        if (threadIdx.x == 0) sweep_rot = 0;
        __syncthreads();
        long long tA = 0, tB = 0, tC = 0, tD = 0;
        for (int rr = 0; rr < 63; ++rr) {
            long long t0 = clock64();
            if (warp == 0) {
                const int i = s_pair[rr][lane][0], j = s_pair[rr][lane][1];
                const double sii = S[i * SLD + i], sjj = S[j * SLD + j], sij = S[i * SLD + j];
                double c = 1.0, sn = 0.0;
                if (fabs(sij) > abs_floor && sij * sij > tol * tol * fmax(sii, 0.0) * fmax(sjj, 0.0)) {
                    // t = 2 s_ij sign(d) / (|d| + sqrt(d^2 + 4 s_ij^2)), d = s_jj - s_ii: the angle only
                    // steers convergence (approximate rsqrt / rcp + one Newton step); c, s from a
                    // full-precision rsqrt keep every rotation orthogonal to working precision
                    const double d = sjj - sii;
                    const double h2 = fma(d, d, 4.0 * sij * sij);
                    double rh, rd;
                    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rh) : "d"(h2));
                    const double den = fma(h2, rh, fabs(d));
                    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rd) : "d"(den));
                    rd = rd * fma(-den, rd, 2.0);
                    double tt = 2.0 * sij * rd;
                    if (d < 0.0) tt = -tt;
                    c = rsqrt(fma(tt, tt, 1.0));
                    sn = c * tt;
                    sweep_rot = 1;
                }
                cs[lane] = make_double2(c, sn);
            }
            __syncthreads();
            long long t1 = clock64();
            // rows i, j of S (S <- J^T S), then columns i, j of S and of T (S <- S J,
            // T <- T J).  Thread (x = tid % 64) handles pairs tid / 64 + 4 m, m < 8,
            // four at a time with every load of a batch issued before its stores
            // (the pairs' rows and columns are disjoint), so a batch is one memory
            // round trip instead of four
            {
                const int x = threadIdx.x & 63, p0 = threadIdx.x >> 6;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    double2 r[4];
                    int ii[4], jj[4];
                    double si[4], sj[4];
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        const int pr = p0 + 4 * (4 * h + m);
                        r[m] = cs[pr];
                        ii[m] = s_pair[rr][pr][0];
                        jj[m] = s_pair[rr][pr][1];
                    }
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        si[m] = S[ii[m] * SLD + x];
                        sj[m] = S[jj[m] * SLD + x];
                    }
#pragma unroll
                    for (int m = 0; m < 4; ++m)
                        if (r[m].y != 0.0) {
                            S[ii[m] * SLD + x] = r[m].x * si[m] - r[m].y * sj[m];
                            S[jj[m] * SLD + x] = r[m].y * si[m] + r[m].x * sj[m];
                        }
                }
                __syncthreads();
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    double2 r[4];
                    int ii[4], jj[4];
                    double si[4], sj[4], ti[4], tj[4];
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        const int pr = p0 + 4 * (4 * h + m);
                        r[m] = cs[pr];
                        ii[m] = s_pair[rr][pr][0];
                        jj[m] = s_pair[rr][pr][1];
                    }
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        si[m] = S[x * SLD + ii[m]];
                        sj[m] = S[x * SLD + jj[m]];
                        ti[m] = R[x * SLD + ii[m]];
                        tj[m] = R[x * SLD + jj[m]];
                    }
#pragma unroll
                    for (int m = 0; m < 4; ++m)
                        if (r[m].y != 0.0) {
                            S[x * SLD + ii[m]] = r[m].x * si[m] - r[m].y * sj[m];
                            S[x * SLD + jj[m]] = r[m].y * si[m] + r[m].x * sj[m];
                            R[x * SLD + ii[m]] = r[m].x * ti[m] - r[m].y * tj[m];
                            R[x * SLD + jj[m]] = r[m].y * ti[m] + r[m].x * tj[m];
                        }
                }
                __syncthreads();
            }
        }
        const int sr = sweep_rot;
        if (threadIdx.x == 0 && sr) any_rot = 1;
        __syncthreads();
        if (!sr) break;
    }
    for (int idx = threadIdx.x; idx < 4096; idx += T) Tout[idx] = R[(idx / 64) * SLD + idx % 64];
    if (threadIdx.x == 0 && any_rot) atomicOr(&L.flags[sweep & 1], 1);
}

namespace {
// C (64 x 64, registers: warp w owns tile row w, 8 tiles) = op(A) B, A and B in
// smem (ld MLD); TA: A read transposed.
template <bool TA>
__device__ __forceinline__ void mm64(const double* A, const double* B, double (&c)[8][2]) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = 0.0;
#pragma unroll 4
    for (int s = 0; s < 16; ++s) {
        const int k = 4 * s + (lane & 3);
        const double av = TA ? A[k * MLD + 8 * warp + (lane >> 2)] : A[(8 * warp + (lane >> 2)) * MLD + k];
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma(c[j][0], c[j][1], av, B[k * MLD + 8 * j + (lane >> 2)]);
    }
}

__device__ __forceinline__ void store64(double* D, const double (&c)[8][2]) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        double* d = D + (8 * warp + (lane >> 2)) * MLD + 8 * j + 2 * (lane & 3);
        d[0] = c[j][0];
        d[1] = c[j][1];
    }
}
}  // namespace

// G <- J^T G J for round r: block (P, P') of G (rows of pair P, columns of
// pair P') becomes T_P^T G[P, P'] T_P'.
namespace {
__device__ __forceinline__ void update_body(SvdTask& t, const WParams& PP, int round, int bx, double* sm) {
    const WLay L = wlay(t, PP);
    int P, P2;
    upper_pair(bx, L.npair, P, P2);
    int a1, b1, a2, b2;
    circle_pair(L.nb32, round, P, a1, b1);
    circle_pair(L.nb32, round, P2, a2, b2);
    double* B = sm;
    double* T1 = sm + 64 * MLD;
    double* T2 = sm + 2 * 64 * MLD;
    auto gi = [&](int l, int a, int b) { return l < 32 ? 32 * a + l : 32 * b + l - 32; };
    const double* t1 = L.t + (int64_t)P * 4096;
    const double* t2 = L.t + (int64_t)P2 * 4096;
    // 16-byte asynchronous copies: G rows are two 32-column segments, T_P contiguous
    for (int idx = threadIdx.x; idx < 2048; idx += T) {
        const int i = idx >> 5, c = idx & 31;  // row, 16-byte chunk of the row
        const int col = c < 16 ? 32 * a2 + 2 * c : 32 * b2 + 2 * (c - 16);
        cp16(B + i * MLD + 2 * c, L.g + (int64_t)gi(i, a1, b1) * L.qp + col);
        cp16(T1 + i * MLD + 2 * c, t1 + 2 * idx);
        cp16(T2 + i * MLD + 2 * c, t2 + 2 * idx);
    }
    cp_wait_all();
    __syncthreads();
    double c[8][2];
    mm64<false>(B, T2, c);  // G[P, P'] T_P'
    __syncthreads();
    store64(B, c);
    __syncthreads();
    mm64<true>(T1, B, c);   // T_P^T (...)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int i = 8 * warp + (lane >> 2), jj = 8 * j + 2 * (lane & 3);
        const int r = gi(i, a1, b1);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int cc = gi(jj + e, a2, b2);
            L.g[(int64_t)r * L.qp + cc] = c[j][e];
            if (P != P2) L.g[(int64_t)cc * L.qp + r] = c[j][e];
        }
    }
}

// V <- V J for round r: V tile (64 rows, columns of pair P).
__device__ __forceinline__ void vupdate_body(SvdTask& t, const WParams& PP, int round, int bx, double* sm) {
    const WLay L = wlay(t, PP);
    const int P = bx % L.npair, r0 = 64 * (bx / L.npair);
    int a, b;
    circle_pair(L.nb32, round, P, a, b);
    double* Vb = sm;
    double* Tm = sm + 64 * MLD;
    auto gj = [&](int l) { return l < 32 ? 32 * a + l : 32 * b + l - 32; };
    const double* tp = L.t + (int64_t)P * 4096;
    for (int idx = threadIdx.x; idx < 2048; idx += T) {
        const int i = idx >> 5, c = idx & 31;
        const int col = c < 16 ? 32 * a + 2 * c : 32 * b + 2 * (c - 16);
        cp16(Vb + i * MLD + 2 * c, L.v + (int64_t)(r0 + i) * L.qp + col);
        cp16(Tm + i * MLD + 2 * c, tp + 2 * idx);
    }
    cp_wait_all();
    __syncthreads();
    double c[8][2];
    mm64<false>(Vb, Tm, c);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int i = 8 * warp + (lane >> 2), jj = 8 * j + 2 * (lane & 3);
        L.v[(int64_t)(r0 + i) * L.qp + gj(jj)] = c[j][0];
        L.v[(int64_t)(r0 + i) * L.qp + gj(jj + 1)] = c[j][1];
    }
}

}  // namespace

// One launch per round for both rotation updates (grid: npair (npair + 1) / 2
// G blocks + npair * qp/64 V tiles, x tasks): G <- J^T G J and V <- V J.
__global__ void __launch_bounds__(T, 2) wide_apply_kernel(SvdTask* tasks, WParams PP, int round) {
    extern __shared__ __align__(16) double sm[];
    SvdTask& t = tasks[blockIdx.y];
    if (t.status != TASK_OK) return;
    const WLay L = wlay(t, PP);
    if (L.flags[2]) return;
    const int nupd = L.npair * (L.npair + 1) / 2;
    if ((int)blockIdx.x < nupd) update_body(t, PP, round, blockIdx.x, sm);
    else vupdate_body(t, PP, round, blockIdx.x - nupd, sm);
}

// End of sweep s: a task that rotated nothing is done; counts active tasks.
__global__ void wide_sweep_end_kernel(SvdTask* tasks, int n, WParams P, int sweep, int* active) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        SvdTask& t = tasks[i];
        if (t.status != TASK_OK) continue;
        const WLay L = wlay(t, P);
        if (!L.flags[2] && !L.flags[sweep & 1]) L.flags[2] = 1;
        L.flags[(sweep + 1) & 1] = 0;
        if (!L.flags[2]) atomicAdd(active, 1);
    }
}

// One-pass decision after pass 1 (one CTA per task).  Pass 1 diagonalises the
// Gram to its own rounding (eps max g_ii), so the kept sigma_j = sqrt(g_jj)
// and U = W V1_k Sigma^-1 are accurate to ~eps (sigma_1 / sigma_j)^2 (the
// narrow engine's one-pass argument, mid2_body).  Under FIXED_RANK(k) with
// sigma_1 <= 1000 sigma_k (lambda ratio 1e6) pass 2 (Y^T Y and its sweeps) is
// skipped: V2 stays I and G keeps pass 1's diagonal; the check kernel still
// enforces the 1e-10 orthonormality contract (fallback otherwise).
__device__ int g_wide_onepass = 1;
__global__ void __launch_bounds__(T) wide_onepass_kernel(SvdTask* tasks, WParams P) {
    __shared__ double lam[1024];
    __shared__ double kth;
    SvdTask& t = tasks[blockIdx.x];
    if (t.status != TASK_OK) return;
    const WGeo g = wgeo(t);
    const WLay L = wlay(t, P);
    const int q = g.q;
    if (!g_wide_onepass || t.trunc.kind != TRUNC_FIXED || t.vpre) {  // (trims keep two passes)
        if (threadIdx.x == 0) t.onepass = 0;
        return;
    }
    const int k = min(t.trunc.k, q);
    for (int i = threadIdx.x; i < q; i += T) lam[i] = L.g[(int64_t)i * L.qp + i];
    if (threadIdx.x == 0) kth = -1.0;
    __syncthreads();
    double lmax = 0.0;
    for (int i = threadIdx.x; i < q; i += T) {
        const double li = lam[i];
        lmax = fmax(lmax, li);
        int r = 0;
        for (int j = 0; j < q; ++j) r += (lam[j] > li) || (lam[j] == li && j < i);
        if (r == k - 1) kth = li;
    }
    for (int o = 16; o > 0; o >>= 1) lmax = fmax(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    __shared__ double red[NW];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = lmax;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 0; w < NW; ++w) lmax = fmax(lmax, red[w]);
        t.onepass = (k >= 1 && kth > 0.0 && lmax <= 1e6 * kth) ? 1 : 0;
    }
}

// Start of pass 2: one-pass tasks are marked converged (their pair / apply /
// sweep-end kernels skip them).
__global__ void wide_pass2_mark_kernel(SvdTask* tasks, int n, WParams P) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        SvdTask& t = tasks[i];
        if (t.status != TASK_OK || !t.onepass) continue;
        const WLay L = wlay(t, P);
        L.flags[2] = 1;
    }
}

// End of pass 1: V1 <- V (grid: qp/64 x tasks).
__global__ void __launch_bounds__(T) wide_keep_v1_kernel(SvdTask* tasks, WParams P) {
    SvdTask& t = tasks[blockIdx.y];
    if (t.status != TASK_OK) return;
    const WLay L = wlay(t, P);
    const int64_t r0 = 64 * blockIdx.x;
    for (int idx = threadIdx.x; idx < 64 * L.qp; idx += T) L.v1[r0 * L.qp + idx] = L.v[r0 * L.qp + idx];
}

// sigma = sqrt(diag G) sorted (ties by index), rank cutoff, truncation; writes
// sigma, k, and M = V2[:, order] (q x k, ld qp).  One CTA per task.
__global__ void __launch_bounds__(T) wide_finalize_kernel(SvdTask* tasks, WParams P) {
    __shared__ double sg[1024];
    __shared__ int ord[1024];
    __shared__ int kk;
    SvdTask& t = tasks[blockIdx.x];
    if (t.status != TASK_OK) return;
    const WGeo g = wgeo(t);
    const WLay L = wlay(t, P);
    const int q = g.q;
    for (int i = threadIdx.x; i < q; i += T) sg[i] = sqrt(fmax(L.g[(int64_t)i * L.qp + i], 0.0));
    __syncthreads();
    for (int i = threadIdx.x; i < q; i += T) {
        int r = 0;
        const double si = sg[i];
        for (int j = 0; j < q; ++j) r += (sg[j] > si) || (sg[j] == si && j < i);
        ord[r] = i;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // svd.hpp:118-124 cutoff, then svd.hpp:135-164 (sequential energy sum)
        const double smax = q > 0 ? sg[ord[0]] : 0.0;
        int knum = 0;
        while (knum < q && sg[ord[knum]] > 0.0 && sg[ord[knum]] >= kNumericalRankCutoff * smax) ++knum;
        int k = knum;
        if (t.trunc.kind == TRUNC_FIXED) {
            k = min(knum, t.trunc.k);
        } else if (t.trunc.kind == TRUNC_ENERGY && knum > 0) {
            double total = 0.0;
            for (int i = 0; i < knum; ++i) total += sg[ord[i]] * sg[ord[i]];
            if (total == 0.0) {
                k = 0;
            } else {
                double acc = 0.0;
                k = knum;
                for (int i = 0; i < knum; ++i) {
                    acc += sg[ord[i]] * sg[ord[i]];
                    if (acc / total >= t.trunc.xi) {
                        k = i + 1;
                        break;
                    }
                }
            }
        }
        if (k > t.kcap) {
            t.status = TASK_CAPACITY;
            k = 0;
        }
        if (t.vpre && !g.tall && k > 0) t.status = TASK_UNSUPPORTED;  // trim narrower than its rank, rank > 64
        kk = k;
        *t.k_out = (double)(t.status == TASK_OK ? k : 0);
        t.krank = t.status == TASK_OK ? k : 0;
    }
    __syncthreads();
    const int k = kk;
    if (t.status != TASK_OK) return;
    for (int r = threadIdx.x; r < k; r += T) {
        t.s[r] = sg[ord[r]];
        L.sig[r] = sg[ord[r]];
        L.sgn[r] = 1.0;
    }
    for (int idx = threadIdx.x; idx < L.qp * k; idx += T) {
        const int i = idx / k, r = idx % k;
        L.m[(int64_t)i * L.qp + r] = i < q ? L.v[(int64_t)i * L.qp + ord[r]] : 0.0;
    }
}

// out (rows x cols tile 64 x 64; grid: rows/64 x cols/64 x tasks) = S B:
//   which 0: Y = W V1 (p x qp)
//   which 1: V_k = V1 M (q x k): A's V (tall, no vpre), A's U (wide), or the
//            G region (tall with vpre)
//   which 2: A's V = vpre (G region) (nvpre x k) for trims
//   which 3: U = Y M diag(sign / sigma) (p x k): A's U (tall) or A's V (wide)
//   which 4: Y = W X (p x kk), X in the V1 region (direct route, wide_eig.cuh)
//   which 5: X Z (q x k), Z in the M region (direct route)
__global__ void __launch_bounds__(T, 2) wide_gemm_kernel(SvdTask* tasks, WParams P, int which) {
    extern __shared__ __align__(16) double sm[];
    SvdTask& t = tasks[blockIdx.z];
    if (t.status != TASK_OK) return;
    const WGeo g = wgeo(t);
    const WLay L = wlay(t, P);
    const int k = t.krank;
    Src s;
    const double* B;
    int ncols, kdim;
    double* out;
    int64_t ldo;
    switch (which) {
        case 0:
            s = Src{nullptr, 0, g.p, g.q, true, (bool)g.tall};
            B = L.v1;
            ncols = L.qp;
            kdim = g.q;
            out = L.y;
            ldo = L.qp;
            break;
        case 1:
            s = Src{L.v1, L.qp, g.q, g.q, false, true};
            B = L.m;
            ncols = k;
            kdim = g.q;
            if (!g.tall) {
                out = t.u;
                ldo = t.ldu;
            } else if (t.vpre) {
                out = L.g;
                ldo = L.qp;
            } else {
                out = t.v;
                ldo = t.ldv;
            }
            break;
        case 4:  // Y = W X (p x kk) of the direct route
            if (L.flags[3] != 1) return;
            s = Src{nullptr, 0, g.p, g.q, true, (bool)g.tall};
            B = L.v1;
            ncols = k;
            kdim = g.q;
            out = L.y;
            ldo = L.qp;
            break;
        case 5:  // A's V (tall) or A's U (wide) = X Z of the direct route, Z in the M region
            if (L.flags[3] != 1 && L.flags[3] != 3) return;
            s = Src{L.v1, L.qp, g.q, min(t.trunc.k, g.q), false, true};
            B = L.m;
            ncols = k;
            kdim = s.cols;
            out = g.tall ? t.v : t.u;
            ldo = g.tall ? t.ldv : t.ldu;
            break;
        case 2:
            if (!(g.tall && t.vpre)) return;
            s = Src{t.vpre, t.ldvpre, t.nvpre, g.q, false, true};
            B = L.g;
            ncols = k;
            kdim = g.q;
            out = t.v;
            ldo = t.ldv;
            break;
        default:
            s = Src{L.y, L.qp, g.p, g.q, false, true};
            B = L.m;
            ncols = k;
            kdim = g.q;
            out = g.tall ? t.u : t.v;
            ldo = g.tall ? t.ldu : t.ldv;
            break;
    }
    const int r0 = 64 * blockIdx.x, c0 = 64 * blockIdx.y;
    if (r0 >= s.rows || c0 >= ncols) return;
    double* Wb = sm;             // 64 rows x 32 (ld 36)
    double* Mb = sm + 64 * 36;   // 32 x 64 columns (ld MLD)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool rowwise = !s.work || s.tall;
    double c[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = 0.0;
    // Fast path (row-major left operand, even ld / inner dimension, aligned): both
    // operands go through a 3-deep cp.async ring (two k-chunks in flight per multiply).
    const double* fbase = s.work ? t.a : s.base;
    const int64_t fld = s.work ? t.lda : s.ld;
    const bool fast = (!s.work || (s.tall && !t.colscale)) && (fld & 1) == 0 && (kdim & 1) == 0 &&
                      (reinterpret_cast<uintptr_t>(fbase) & 15) == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0;
    if (fast) {
        constexpr int STG = 64 * 36 + 32 * MLD;
        const int nch = (kdim + 31) / 32;
        auto issue = [&](int ci) {
            if (ci < nch) {
                double* wb = sm + (ci % 3) * STG;
                double* mb = wb + 64 * 36;
                const int kb = 32 * ci;
                for (int idx = threadIdx.x; idx < 64 * 16; idx += T) {  // W tile: 64 rows x 16 pairs
                    const int r = idx >> 4, kx = 2 * (idx & 15);
                    const int row = r0 + r, col = kb + kx;
                    double* dst = wb + r * 36 + kx;
                    if (row < s.rows && col < kdim) cp16(dst, fbase + (int64_t)row * fld + col);
                    else dst[0] = dst[1] = 0.0;
                }
                for (int idx = threadIdx.x; idx < 32 * 32; idx += T) {  // B tile: 32 rows x 32 pairs
                    const int kx = idx >> 5, cc = 2 * (idx & 31);
                    double* dst = mb + kx * MLD + cc;
                    if (c0 + cc < ncols && kb + kx < kdim) cp16(dst, B + (int64_t)(kb + kx) * L.qp + c0 + cc);
                    else dst[0] = dst[1] = 0.0;
                }
            }
            asm volatile("cp.async.commit_group;");
        };
        issue(0);
        issue(1);
        for (int ci = 0; ci < nch; ++ci) {
            issue(ci + 2);
            asm volatile("cp.async.wait_group 2;" ::: "memory");
            __syncthreads();
            const double* wb = sm + (ci % 3) * STG;
            const double* mb = wb + 64 * 36;
#pragma unroll
            for (int sx = 0; sx < 8; ++sx) {
                const int kx = 4 * sx + (lane & 3);
                const double av = wb[(8 * warp + (lane >> 2)) * 36 + kx];
#pragma unroll
                for (int j = 0; j < 8; ++j) dmma(c[j][0], c[j][1], av, mb[kx * MLD + 8 * j + (lane >> 2)]);
            }
            __syncthreads();
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    for (int kb = 0; kb < kdim && !fast; kb += 32) {
        for (int idx = threadIdx.x; idx < 64 * 32; idx += T) {
            int r, kx;
            if (rowwise) {
                r = idx / 32;
                kx = idx % 32;
            } else {
                kx = idx / 64;
                r = idx % 64;
            }
            const int row = r0 + r, col = kb + kx;
            Wb[r * 36 + kx] = (row < s.rows && col < kdim) ? src_at(t, s, row, col) : 0.0;
        }
        for (int idx = threadIdx.x; idx < 32 * 64; idx += T) {
            const int kx = idx / 64, cc = idx % 64;
            Mb[kx * MLD + cc] = (c0 + cc < ncols && kb + kx < kdim) ? B[(int64_t)(kb + kx) * L.qp + c0 + cc] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int sx = 0; sx < 8; ++sx) {
            const int kx = 4 * sx + (lane & 3);
            const double av = Wb[(8 * warp + (lane >> 2)) * 36 + kx];
#pragma unroll
            for (int j = 0; j < 8; ++j) dmma(c[j][0], c[j][1], av, Mb[kx * MLD + 8 * j + (lane >> 2)]);
        }
        __syncthreads();
    }
    const int row = r0 + 8 * warp + (lane >> 2);
    if (row < s.rows) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = c0 + 8 * j + 2 * (lane & 3) + e;
                if (col < ncols) {
                    double x = c[j][e];
                    if (which == 3) x *= L.sgn[col] / L.sig[col];
                    out[(int64_t)row * ldo + col] = x;
                }
            }
        }
    }
}

namespace {
// Pivot of column r of F (rows x ., ld): first index of max |F(i, r)|; warp-wide.
__device__ __forceinline__ int col_pivot(const double* F, int64_t ld, int rows, int r) {
    const int lane = threadIdx.x & 31;
    double best = -1.0;
    int bi = 0;
    for (int i = lane; i < rows; i += 32) {
        const double x = fabs(F[(int64_t)i * ld + r]);
        if (x > best) {
            best = x;
            bi = i;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
        }
    }
    return bi;
}
}  // namespace

// Canonical sign (svd.hpp:179-203).  stage 0 (tall tasks, before U is
// formed): pivot of A's V, flip it, record the sign for U.  stage 1 (wide
// tasks, after): pivot of the formed A's V, flip it and A's U.  One warp per
// column; grid: tasks.
__global__ void __launch_bounds__(T) wide_sign_kernel(SvdTask* tasks, WParams P, int stage) {
    SvdTask& t = tasks[blockIdx.x];
    if (t.status != TASK_OK || !t.sign) return;
    const WGeo g = wgeo(t);
    if ((stage == 0) != (bool)g.tall) return;
    const WLay L = wlay(t, P);
    const int k = t.krank;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nv = stage == 0 ? (t.vpre ? t.nvpre : g.q) : g.p;
    for (int r = warp; r < k; r += NW) {
        const int bi = col_pivot(t.v, t.ldv, nv, r);
        const bool neg = t.v[(int64_t)bi * t.ldv + r] < 0.0;
        __syncwarp();
        if (neg) {
            for (int i = lane; i < nv; i += 32) t.v[(int64_t)i * t.ldv + r] = -t.v[(int64_t)i * t.ldv + r];
            if (stage == 1)
                for (int i = lane; i < g.q; i += 32) t.u[(int64_t)i * t.ldu + r] = -t.u[(int64_t)i * t.ldu + r];
        }
        if (stage == 0 && lane == 0) L.sgn[r] = neg ? -1.0 : 1.0;
    }
}

// Orthonormality of the formed factor (its Gram is in the G region, k x k at
// ld qp): max |F^T F - I| <= 1e-10 (svd.hpp:25).
__global__ void __launch_bounds__(T) wide_check_kernel(SvdTask* tasks, WParams P) {
    __shared__ int bad;
    SvdTask& t = tasks[blockIdx.x];
    if (t.status != TASK_OK) return;
    const WLay L = wlay(t, P);
    const int k = t.krank;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    for (int idx = threadIdx.x; idx < k * k; idx += T) {
        const int i = idx / k, j = idx % k;
        const double d = L.g[(int64_t)i * L.qp + j] - (i == j ? 1.0 : 0.0);
        if (!(fabs(d) <= kOrthonormalityTol)) bad = 1;
    }
    __syncthreads();
    if (threadIdx.x == 0 && bad) {
        t.status = TASK_NEEDS_FALLBACK;
        t.reason = 8;
    }
}

#include "wide_eig.cuh"

// ---------------------------------------------------------------- host side
int wide_tridiag_smem(int qp) { return 8 * 4 * qp; }
int wide_trieig_smem(int qp) { return 8 * (4 * qp + (3 * qp > 2 * 64 * 65 ? 3 * qp : 2 * 64 * 65)); }

// Launches the two cluster kernels of the direct route over n tasks: clusters
// of 8 CTAs, or of 16 (non-portable size) when the batch is small enough for
// 16-CTA clusters to run side by side (a single stitch gets 16 SMs).
int wide_eig_launch(SvdTask* d, int n, WParams P, int qp, cudaStream_t st) {
    static int cl16 = -1;  // 16-CTA clusters schedulable on this device?
    if (cl16 < 0) {
        const int smax = wide_trieig_smem(1024);
        if (cudaFuncSetAttribute(wide_tridiag_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, wide_tridiag_smem(1024)) != cudaSuccess ||
            cudaFuncSetAttribute(wide_tridiag_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, wide_tridiag_smem(1024)) != cudaSuccess ||
            cudaFuncSetAttribute(wide_trieig_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax) != cudaSuccess ||
            cudaFuncSetAttribute(wide_trieig_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax) != cudaSuccess ||
            cudaFuncSetAttribute(wide_trieig_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax) != cudaSuccess)
            return 1;
        bool ok = cudaFuncSetAttribute(wide_tridiag_kernel<512>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
                  cudaFuncSetAttribute(wide_tridiag_kernel<256>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
                  cudaFuncSetAttribute(wide_trieig_kernel<8>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
                  cudaFuncSetAttribute(wide_trieig_kernel<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
                  cudaFuncSetAttribute(wide_trieig_kernel<32>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
        if (ok) {
            cudaLaunchConfig_t q = {};
            q.gridDim = dim3(16, 1);
            q.blockDim = dim3(512);
            q.dynamicSmemBytes = wide_tridiag_smem(1024);
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = 16;
            qa[0].val.clusterDim.y = 1;
            qa[0].val.clusterDim.z = 1;
            q.attrs = qa;
            q.numAttrs = 1;
            int nc = 0;
            ok = cudaOccupancyMaxActiveClusters(&nc, wide_tridiag_kernel<512>, &q) == cudaSuccess && nc >= 1;
        }
        cudaGetLastError();
        cl16 = ok ? 1 : 0;
    }
    // cluster size: 16 CTAs for a lone task or two (queries), 4 for large batches of
    // small problems (more tasks in flight; a step is latency-bound), else 8
    const int cl = (cl16 && n <= 4) ? 16 : (qp <= 256 && n >= 19) ? 4 : 8;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl, n);
    cfg.blockDim = dim3(qp <= 256 ? 256 : 512);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.dynamicSmemBytes = wide_tridiag_smem(qp);
    if ((qp <= 256 ? cudaLaunchKernelEx(&cfg, wide_tridiag_kernel<256>, d, P)
                   : cudaLaunchKernelEx(&cfg, wide_tridiag_kernel<512>, d, P)) != cudaSuccess)
        return 1;
    cfg.blockDim = dim3(T);
    if (cl < 8) {  // one warp per eigenpair: 64 of them need 8 CTAs
        cfg.gridDim = dim3(8, n);
        at[0].val.clusterDim.x = 8;
    }
    cfg.dynamicSmemBytes = wide_trieig_smem(qp);
    cudaError_t e;
    if (qp <= 256) e = cudaLaunchKernelEx(&cfg, wide_trieig_kernel<8>, d, P);
    else if (qp <= 512) e = cudaLaunchKernelEx(&cfg, wide_trieig_kernel<16>, d, P);
    else e = cudaLaunchKernelEx(&cfg, wide_trieig_kernel<32>, d, P);
    return e == cudaSuccess ? 0 : 1;
}

int wide_init_tables() {
    unsigned char h[63][32][2];
    for (int r = 0; r < 63; ++r)
        for (int i = 0; i < 32; ++i) {
            int a, b;
            if (i == 0) {
                a = 63;
                b = r;
            } else {
                a = (r + i) % 63;
                b = (r - i + 63) % 63;
            }
            h[r][i][0] = (unsigned char)(a < b ? a : b);
            h[r][i][1] = (unsigned char)(a < b ? b : a);
        }
    return cudaMemcpyToSymbol(c_pair64, h, sizeof(h)) == cudaSuccess ? 0 : 1;
}

int wide_gram_smem() { return 3 * 8 * GCH * GLD; }
int wide_pair_smem() { return 8 * 2 * 64 * SLD; }
int wide_mm_smem() { return 8 * 3 * 64 * MLD; }
int wide_gemm_smem() { return 3 * 8 * (64 * 36 + 32 * MLD); }

}  // namespace zsvd
