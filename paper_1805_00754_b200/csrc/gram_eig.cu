// gram_eig.cu — the SVD of a range query's Gram stitch (gram_stitch.cu) by the
// symmetric eigensolver of eigh.cuh: one task, so latency is what counts, and
// the narrow engine's mid-phases (Cholesky of G, then ~500 dependent rounds of
// one-sided Jacobi on R, all on one SM) were ~80% of a cfg2 query.
//
// It writes what mid-2 writes: V (t.v, sign-canonical, svd.hpp:179-203), sigma
// and M = V_k Sigma_k^-1 (workspace, ld kQMax) and the kept rank (numerical-rank
// cutoff 1e-12 sigma_1, svd.hpp:118-124, then FIXED_RANK k).
//
// Accuracy is that of one-pass CholeskyQR: the kept sigma_j and
// U = S V Sigma^-1 carry ~eps (sigma_1 / sigma_j)^2 errors, so a kept spread
// beyond sigma_1 > 3000 sigma_k, an unresolvable truncation boundary or a
// failed eigensolver check flags the task and the host redoes the query on the
// trim + stack engine path (zsvd_api.cu).  (The storage flush uses the warp
// build of the same solver, eigh_warp.cuh, only for the starting basis of a
// k-column Jacobi on R X: a Gram-level U alone misses the 1e-10 contract at
// cfg2's spreads of 600-900.)
#include <cstdint>

namespace zsvd {
__device__ long long g_qeig_clk[8];  // eigh_top's phase stamps of the last query (diagnostics)
}
#define EIGH_CLK(i)                                        \
    do {                                                   \
        if (threadIdx.x == 0) zsvd::g_qeig_clk[i] = clock64(); \
    } while (0)
#include "eigh.cuh"
#include "zsvd_internal.h"

namespace zsvd {
namespace {

// After eigh_top: rank, sign, outputs.  Returns the kept rank, or -1 if the
// spread exceeds `spread` (nothing written).
template <int KMAX>
__device__ int eig_outputs(SvdTask& t, int q, int kk, int kv, double scale, double spread, const double* esm) {
    using P = eigh::Plan<KMAX>;
    __shared__ double sgn[64];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double* lam = esm + P::D + 256;
    const double* Z = esm + P::Z;
    const double inv_scale = 1.0 / scale;
    const double s0 = sqrt(fmax(lam[0], 0.0) * inv_scale);
    int kout = 0;
    while (kout < kk) {
        const double sj = sqrt(fmax(lam[kout], 0.0) * inv_scale);
        if (!(sj > 0.0) || sj < 1e-12 * s0) break;
        ++kout;
    }
    if (kout > 0 && s0 > spread * sqrt(fmax(lam[kout - 1], 0.0) * inv_scale)) return -1;
    // a truncation boundary (rank kept < numerical rank) must be resolvable at the
    // Gram's accuracy: sigma_k+1 close to sigma_k turns the eps ||G|| / gap angle
    // error of the k-th vector into a reconstruction error ~ angle sigma_k /
    // sigma_1; keep that 10x under the 1e-9 bar (else the one-sided Jacobi on R,
    // whose error is eps sigma_1 / gap, decides)
    if (kout == kk && kv > kk && lam[kk] > 0.0) {
        const double gap = lam[kk - 1] - lam[kk];
        const double sk = sqrt(fmax(lam[kk - 1], 0.0));
        if (!(gap > 0.0) || 4.0 * 2.220446049250313e-16 * lam[0] * sk > 1e-10 * gap * sqrt(lam[0])) return -1;
    }
    // canonical sign: pivot = first index of max |V(:, j)|
    for (int j = warp; j < kout; j += 8) {
        double best = -1.0;
        int idx = 0x7fffffff;
        for (int i = lane; i < q; i += 32) {
            const double mag = fabs(Z[i * P::LDZ + j]);
            if (mag > best) {
                best = mag;
                idx = i;
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
        if (lane == 0) sgn[j] = Z[idx * P::LDZ + j] < 0.0 ? -1.0 : 1.0;
    }
    __syncthreads();
    const int nsp = t.nsplit;
    double* mg = t.ws + ws_off_m(nsp);
    double* sg = t.ws + ws_off_sig(nsp);
    for (int x = tid; x < q * kout; x += 256) {
        const int a = x / kout, r = x - a * kout;
        t.v[(int64_t)a * t.ldv + r] = sgn[r] * Z[a * P::LDZ + r];
    }
    for (int x = tid; x < kQMax * kQMax; x += 256) {
        const int l = x >> 6, r = x & 63;
        double m = 0.0;
        if (l < q && r < kout) m = sgn[r] * Z[l * P::LDZ + r] * rsqrt(fmax(lam[r], 0.0) * inv_scale);
        mg[l * kQMax + r] = m;
    }
    if (tid < kout) sg[tid] = sqrt(fmax(lam[tid], 0.0) * inv_scale);
    return kout;
}

// Power of two bringing max |G| (upper triangle, q x q, ld kQMax) to [0.5, 1);
// 0 for a zero matrix, -1 for non-finite entries.
__device__ double gram_scale(const double* G, int q) {
    __shared__ double red[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double amax = 0.0;
    for (int x = tid; x < q * q; x += 256) {
        const int i = x / q, j = x - i * q;
        if (i <= j) amax = fmax(amax, fabs(G[i * kQMax + j]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if (lane == 0) red[warp] = amax;
    __syncthreads();
    amax = 0.0;
    for (int w = 0; w < 8; ++w) amax = fmax(amax, red[w]);
    __syncthreads();
    if (!(amax < 1e300)) return -1.0;
    if (amax == 0.0) return 0.0;
    const int e2 = ((__double2hiint(amax) >> 20) & 0x7ff) - 1022;  // amax in [2^(e2-1), 2^e2)
    return ldexp(1.0, -e2);
}
}  // namespace

int gram_eig_smem_bytes() { return eigh::Plan<64>::bytes(); }

// The Gram stitch's SVD (one CTA): G = t.ws partial 0 (c x c, ld kQMax, upper
// triangle); k = min(FIXED_RANK k, c); a kept spread beyond 3000 or a failed
// eigensolver check flags the task (the host redoes the query on the engine path).
__global__ void __launch_bounds__(256) gram_eig_kernel(SvdTask* task, int c) {
    ZSVD_PDL_WAIT();
    extern __shared__ __align__(16) double esm[];
    SvdTask& t = *task;
    if (t.status != TASK_OK) return;
    auto flag = [&](int reason) {
        if (threadIdx.x == 0) {
            t.status = TASK_NEEDS_FALLBACK;
            t.reason = reason;
            t.krank = 0;
        }
    };
    if (t.trunc.kind != TRUNC_FIXED) {
        flag(20);
        return;
    }
    const double scale = gram_scale(t.ws, c);
    if (scale < 0.0) {
        flag(20);
        return;
    }
    if (scale == 0.0) {  // a zero stack: rank 0 (query.hpp:109-111)
        if (threadIdx.x == 0) t.krank = 0;
        return;
    }
    const int kk = t.trunc.k < c ? t.trunc.k : c;
    const int kv = kk < c ? kk + 1 : kk;  // one more eigenvalue: the truncation boundary's gap
    const int st = eigh::eigh_top<64>(t.ws, kQMax, c, kk, kv, scale, esm);
    if (st) {
        flag(20 + st);
        return;
    }
    const int kout = eig_outputs<64>(t, c, kk, kv, scale, 3000.0, esm);
    __syncthreads();
    if (kout < 0) flag(23);
    else if (threadIdx.x == 0) t.krank = kout;
}

}  // namespace zsvd
