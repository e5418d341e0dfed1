// sym_eig.cuh — latency-optimised symmetric eigensolver for one N x N Gram
// (N = 16, 32, 64) on one CTA: parallel two-sided cyclic Jacobi.
//
// Used by the Gram stitch of range_query (gram_stitch.cu): the stitched stack
// S (query.hpp:113-122) enters only through G = S^T S, whose eigenpairs give
// sigma = sqrt(lambda) and V (query.hpp:124) — the same Gram-level accuracy
// as one-pass CholeskyQR.  A single query has exactly one such
// problem, so the solver is built for latency, not throughput:
//
//  * (N/2)^2 threads; thread (p, q) owns the 2 x 2 block of rows of pair p and
//    columns of pair q and applies J_p^T B J_q to it in registers each round;
//  * G is kept in "slot order": the round-robin (circle method) pairs of round
//    r sit in slots (2i, 2i + 1), and every element is written straight to its
//    slot of the next round (ping-pong buffers).  The position of an index in
//    the circle advances by one per round, so the next slot of a slot does not
//    depend on the round: each thread's four write addresses are fixed;
//  * the thread whose block holds the off-diagonal element of a pair of the
//    NEXT round (it is unique) also recomputes that pair's two rotated
//    diagonal entries and its rotation angle in the same round, so one
//    barrier per round suffices;
//  * angles come from fp32 (MUFU) arithmetic and are made exactly orthogonal
//    in fp64 (c^2 + s^2 = 1 to working precision); the rotated pair's
//    off-diagonal is then the true residual, kept (not zeroed);
//  * convergence is tested on the whole matrix at the end of each sweep, so
//    no confirming rotation-free sweep is needed.
#pragma once

#include <cstdint>

namespace zsvd {
namespace eig {

template <int N>
struct Shared {
    static constexpr int NP = N / 2;
    static constexpr int NT = NP * NP;
    double G[2][N * N];  // slot order, ping-pong
    double V[N * N];     // V[row * N + x], x = original index
    double2 cs[2][NP];   // (c, s) of the pairs of the current / next round
    double d[2][N];      // diagonal, slot order
    double lam[N];       // eigenvalues by original index
    int flag;
    int sweeps;
};

__device__ __forceinline__ int pos_of_slot(int s, int n) { return (s & 1) ? n - 1 - (s >> 1) : (s >> 1); }
__device__ __forceinline__ int slot_of_pos(int pos, int n) { return pos < n / 2 ? 2 * pos : 2 * (n - 1 - pos) + 1; }
__device__ __forceinline__ int next_pos(int pos, int n) { return pos == 0 ? 0 : (pos == n - 1 ? 1 : pos + 1); }
__device__ __forceinline__ int next_slot(int s, int n) { return slot_of_pos(next_pos(pos_of_slot(s, n), n), n); }
// original index at circle position pos in round r (0 <= r < n - 1)
__device__ __forceinline__ int orig_at(int pos, int r, int n) {
    if (pos == 0) return 0;
    int x = pos - 1 - r;
    if (x < 0) x += n - 1;
    return x + 1;
}

// Rotation (c, s) annihilating g in [[a, g], [g, b]]: theta = (b - a) / 2g,
// t = sgn(theta) / (|theta| + sqrt(theta^2 + 1)) in fp32, then (c, s) scaled
// to unit norm in fp64 (one third-order correction of an fp32-accurate pair).
// Returns false (c = 1, s = 0) below the threshold.
__device__ __forceinline__ bool angle(double a, double b, double g, double tol2, double tolabs, double& c,
                                      double& s) {
    if (g * g <= tol2 * a * b || fabs(g) <= tolabs) {
        c = 1.0;
        s = 0.0;
        return false;
    }
    const float x = (float)(b - a);
    const float y = (float)(g + g);
    const float th = __fdividef(x, y);
    const float r = __fsqrt_rn(fmaf(th, th, 1.0f));
    const float t = __fdividef(th >= 0.0f ? 1.0f : -1.0f, fabsf(th) + r);
    const float cf = rsqrtf(fmaf(t, t, 1.0f));
    const double c0 = (double)cf, s0 = (double)(t * cf);
    const double e = fma(c0, c0, fma(s0, s0, -1.0));
    const double nrm = fma(e, fma(e, 0.375, -0.5), 1.0);
    c = c0 * nrm;
    s = s0 * nrm;
    return true;
}

// Eigen-decomposition of the symmetric matrix A (n x n, row-major, lda; n <= N)
// scaled by `scale`, padded with zeros to N.  On return (all threads):
// S.lam[x] = eigenvalue of original index x (unsorted, of the scaled matrix),
// S.V[i * N + x] = component i of its eigenvector; S.sweeps.  tol: relative
// threshold sqrt(g^2 / (a b)); absolute threshold tolabs_rel * max diagonal.
// blockDim.x must be Shared<N>::NT.
template <int N>
__device__ void jacobi_eig(const double* A, int64_t lda, int n, double scale, Shared<N>& S, double tol,
                           double tolabs_rel, int max_sweeps) {
    constexpr int NP = N / 2;
    const int tid = threadIdx.x;
    const int p = tid / NP, q = tid % NP;
    // load (slot order of round 0: slot s holds index pos_of_slot(s))
    for (int e = tid; e < N * N; e += Shared<N>::NT) {
        const int si = e / N, sj = e % N;
        const int i = pos_of_slot(si, N), j = pos_of_slot(sj, N);
        S.G[0][e] = (i < n && j < n) ? scale * A[(int64_t)i * lda + j] : 0.0;
        S.V[e] = (si == sj) ? 1.0 : 0.0;
    }
    __syncthreads();
    if (tid < N) S.d[0][tid] = S.G[0][tid * N + tid];
    if (tid == 0) S.flag = 0;
    __syncthreads();
    double dmax = 0.0;
    for (int i = 0; i < N; ++i) dmax = fmax(dmax, S.d[0][i]);
    const double tol2 = tol * tol;
    const double tolabs = tolabs_rel * dmax;
    if (tid < NP) {
        double c, s;
        angle(S.d[0][2 * tid], S.d[0][2 * tid + 1], S.G[0][(2 * tid) * N + 2 * tid + 1], tol2, tolabs, c, s);
        S.cs[0][tid] = make_double2(c, s);
    }
    // fixed per thread: next-round slots of my rows / columns, ownership
    const int rs0 = next_slot(2 * p, N), rs1 = next_slot(2 * p + 1, N);
    const int cs0 = next_slot(2 * q, N), cs1 = next_slot(2 * q + 1, N);
    int own_u = -1, own_v = -1;
    {
        const int rr[2] = {rs0, rs1}, cc[2] = {cs0, cs1};
        for (int u = 0; u < 2; ++u)
            for (int v = 0; v < 2; ++v)
                if (p != q && (rr[u] & 1) == 0 && cc[v] == rr[u] + 1) {
                    own_u = u;
                    own_v = v;
                }
    }
    const int own_n = own_u >= 0 ? (own_u ? rs1 : rs0) >> 1 : 0;
    // V work: pair pv, rows rv and rv + NP
    const int pv = tid % NP, rv = tid / NP;
    const int vpos_a = pos_of_slot(2 * pv, N), vpos_b = pos_of_slot(2 * pv + 1, N);
    __syncthreads();

    int cur = 0;
    int sweep = 0;
    for (; sweep < max_sweeps; ++sweep) {
        for (int r = 0; r < N - 1; ++r) {
            const int nxt = cur ^ 1;
            const double2 cp = S.cs[cur][p], cq = S.cs[cur][q];
            const double* Gc = S.G[cur];
            double* Gn = S.G[nxt];
            const double2 b0 = *reinterpret_cast<const double2*>(Gc + (2 * p) * N + 2 * q);
            const double2 b1 = *reinterpret_cast<const double2*>(Gc + (2 * p + 1) * N + 2 * q);
            if (p == q) {
                // the pair's own block: its off-diagonal after the (exactly
                // orthogonal, approximately annihilating) rotation
                const double d0 = S.d[cur][2 * p], d1 = S.d[cur][2 * p + 1];
                const double c = cp.x, s = cp.y;
                const double g1 = fma(c * s, d0 - d1, (c - s) * (c + s) * b0.y);
                Gn[rs0 * N + rs1] = g1;
                Gn[rs1 * N + rs0] = g1;
            } else {
                const double cc = cp.x * cq.x, csq = cp.x * cq.y, sc = cp.y * cq.x, ss = cp.y * cq.y;
                const double n00 = fma(cc, b0.x, -csq * b0.y) + fma(ss, b1.y, -sc * b1.x);
                const double n01 = fma(csq, b0.x, cc * b0.y) - fma(ss, b1.x, sc * b1.y);
                const double n10 = fma(sc, b0.x, -ss * b0.y) + fma(cc, b1.x, -csq * b1.y);
                const double n11 = fma(ss, b0.x, sc * b0.y) + fma(csq, b1.x, cc * b1.y);
                Gn[rs0 * N + cs0] = n00;
                Gn[rs0 * N + cs1] = n01;
                Gn[rs1 * N + cs0] = n10;
                Gn[rs1 * N + cs1] = n11;
                if (own_u >= 0) {
                    // rotated diagonals of the two elements that form pair own_n next
                    auto rot_diag = [&](int pr, int w, double2 csp) {
                        const double d0 = S.d[cur][2 * pr], d1 = S.d[cur][2 * pr + 1];
                        const double g = Gc[(2 * pr) * N + 2 * pr + 1];
                        const double c2 = csp.x * csp.x, s2 = csp.y * csp.y, cs2 = 2.0 * csp.x * csp.y;
                        return w == 0 ? fma(c2, d0, fma(-cs2, g, s2 * d1)) : fma(s2, d0, fma(cs2, g, c2 * d1));
                    };
                    const double da = rot_diag(p, own_u, cp);
                    const double db = rot_diag(q, own_v, cq);
                    const double g = own_u == 0 ? (own_v == 0 ? n00 : n01) : (own_v == 0 ? n10 : n11);
                    double c, s;
                    angle(da, db, g, tol2, tolabs, c, s);
                    S.cs[nxt][own_n] = make_double2(c, s);
                    S.d[nxt][2 * own_n] = da;
                    S.d[nxt][2 * own_n + 1] = db;
                }
            }
            {
                const double2 cv = S.cs[cur][pv];
                const int a = orig_at(vpos_a, r, N), b = orig_at(vpos_b, r, N);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    double* row = S.V + (rv + h * NP) * N;
                    const double x = row[a], y = row[b];
                    row[a] = fma(cv.x, x, -cv.y * y);
                    row[b] = fma(cv.y, x, cv.x * y);
                }
            }
            cur = nxt;
            __syncthreads();
        }
        // whole-matrix convergence test in the next round's layout
        bool bad = false;
        {
            const double* Gc = S.G[cur];
            if (p == q) {
                const double g = Gc[(2 * p) * N + 2 * p + 1];
                bad = !(g * g <= tol2 * S.d[cur][2 * p] * S.d[cur][2 * p + 1] || fabs(g) <= tolabs);
            } else {
#pragma unroll
                for (int u = 0; u < 2; ++u)
#pragma unroll
                    for (int v = 0; v < 2; ++v) {
                        const double g = Gc[(2 * p + u) * N + 2 * q + v];
                        bad |= !(g * g <= tol2 * S.d[cur][2 * p + u] * S.d[cur][2 * q + v] || fabs(g) <= tolabs);
                    }
            }
        }
        if (!__syncthreads_or(bad)) {
            ++sweep;
            break;
        }
    }
    // a whole number of sweeps: round 0 again, slot s holds index pos_of_slot(s)
    if (tid < N) S.lam[pos_of_slot(tid, N)] = S.d[cur][tid];
    if (tid == 0) S.sweeps = sweep;
    __syncthreads();
}

}  // namespace eig
}  // namespace zsvd
