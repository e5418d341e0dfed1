// wide_eig.cuh — the wide path's direct route for FIXED_RANK(k <= 64) tasks
// (included by wide_engine.cu inside namespace zsvd).
//
// thin_svd + truncate_rank (svd.hpp:90-164) of a tall W (p x q, 64 < q <= 1024)
// only keeps k <= 64 triplets, so instead of diagonalising the whole Gram by
// block Jacobi (~15 sweeps of q/32 - 1 rounds, two launches each and a host
// wait per sweep) the kept subspace is taken directly:
//
//   1. G = W^T W (wide_gram_kernel), then T = Q^T G Q by Householder
//      tridiagonalisation (dsytd2 order) on one thread-block cluster per task:
//      the rows of G are dealt round-robin to the cluster's CTAs and warps; a
//      step is ONE fused pass over the trailing matrix (apply the previous
//      step's rank-2 update, write it back, multiply by the new reflector) and
//      ONE cluster barrier; the vectors every CTA needs (the next row, p = G v)
//      go through L2.
//   2. the kk = min(k, q) largest eigenvalues of T by warp-wide 32-way Sturm
//      multisection, one warp per eigenvalue across the cluster; inverse
//      iteration (dgttrf with partial pivoting, two solves) on the same warp,
//      the sequential recurrences run redundantly on all lanes with the
//      factors streamed through L2 in 32-entry chunks; a residual check;
//      Cholesky QR of the kk vectors (close eigenvalues leave them only nearly
//      orthogonal); back-transform through the stored reflectors, the column
//      in registers, reflectors staged per CTA by cp.async.
//   3. Y = W X (p x kk, DMMA) and the NARROW engine on Y (svd_engine.cu:
//      CholeskyQR + one-sided Jacobi + U formation + 1e-10 check + robust
//      fallback): sigma and U with thin_svd's rank cutoff and FIXED_RANK
//      truncation exactly as on q <= 64; V = X Z (DMMA), then canonical_sign.
//
// X spans the dominant invariant subspace to the Gram's accuracy
// (eps sigma_1^2 / (sigma_k^2 - sigma_k+1^2), the one-pass accuracy the wide
// path already accepted); sigma, U and V inside it come from the one-sided
// engine.  A wide A (m < n, W = A^T: short stitches, K < c) takes the same
// route with the roles of U and V exchanged.  Tasks the route cannot take
// (energy truncation or none, k > 64, trims, a failed residual / Cholesky)
// keep the block-Jacobi path.
#pragma once

namespace {

constexpr int WE_KMAX = 64;  // most eigenpairs (one warp each: 8 warps x 8 CTAs)
constexpr int kParked = 100; // task finished by this route; restored to TASK_OK at the end

// Scratch of the route inside the task workspace (doubles), after sig / sgn / flags.
struct WEig {
    double *d, *e, *tau, *lam, *pbuf, *res, *lu, *z, *b;
};
__host__ __device__ constexpr int64_t weig_doubles(int64_t qp) {
    return 8 * qp + (int64_t)WE_KMAX * 6 * qp + (int64_t)WE_KMAX * qp + WE_KMAX * WE_KMAX;
}
__device__ __forceinline__ WEig weig(const WLay& L) {
    WEig E;
    const int64_t qp = L.qp;
    E.d = L.ez;
    E.e = E.d + qp;
    E.tau = E.e + qp;
    E.lam = E.tau + qp;        // kk eigenvalues (of the scaled T)
    E.res = E.lam + qp / 2;    // per-eigenvalue failure flags (as doubles)
    E.pbuf = E.lam + qp;       // 2 x qp: p = tau G v, double-buffered by step parity
    E.lu = E.d + 8 * qp;       // per vector: 1/U_ii, U_i,i+1, U_i,i+2, L_i, pivot bit, start/solve vector
    E.z = E.lu + (int64_t)WE_KMAX * 6 * qp;  // eigenvectors of T, one per row (kk x qp)
    E.b = E.z + (int64_t)WE_KMAX * qp;       // Z Z^T (kk x kk, ld 64)
    return E;
}

__device__ __forceinline__ void we_cluster_sync() {
    __threadfence();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ double we_warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// Sum over the CTA (fixed order: lanes by butterfly, warps in order); every
// thread gets the same bits.  red: NW doubles of shared memory.
__device__ __forceinline__ double we_block_sum(double x, double* red) {
    x = we_warp_sum(x);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += red[w];
    return s;
}

__device__ __forceinline__ double we_rcp(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x, y, 1.0);
    return fma(y * e, 1.0 + e, y);
}

// 2^-(exponent of max(|a|, |b|)) (1 when both are zero / denormal).
__device__ __forceinline__ double we_renorm(double a, double b) {
    const int ea = (__double2hiint(a) >> 20) & 0x7ff, eb = (__double2hiint(b) >> 20) & 0x7ff;
    const int e = ea > eb ? ea : eb;
    return e == 0 ? 1.0 : __hiloint2double((2046 - e) << 20, 0);
}

__device__ __forceinline__ double we_start(int i, int t) {
    unsigned h = (unsigned)(i * 0x9E3779B1u) ^ (unsigned)((t + 1) * 0x85EBCA77u);
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    const double u = 0.5 + (double)(h & 0xFFFFFu) * (1.0 / 1048576.0);
    return (h & 0x100000u) ? -u : u;
}

}  // namespace

__device__ int g_wide_eig = 1;
extern __device__ unsigned long long g_direct_tasks;  // svd_engine.cu

// Which tasks take the direct route (flags[3] = 1); one thread per task.
__global__ void wide_eig_select_kernel(SvdTask* tasks, int n, WParams P) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        SvdTask& t = tasks[i];
        if (t.status != TASK_OK) continue;
        const WGeo g = wgeo(t);
        const WLay L = wlay(t, P);
        const bool ok = g_wide_eig && t.trunc.kind == TRUNC_FIXED && t.trunc.k >= 1 && t.trunc.k <= WE_KMAX && !t.vpre && !t.qr_only && g.q > kQMax && g.q <= 1024;
        L.flags[3] = ok ? 1 : 0;
    }
}

// Householder tridiagonalisation of G (q x q, both triangles, ld qp) on a
// cluster of gridDim.x CTAs of 512 threads (grid: cluster x tasks).  Out: d, e,
// tau in the scratch, reflector j (v_{j+1} = 1, support j+1..q-1) in row j of
// the V region.  The pass is L2-bandwidth work: a warp streams four of its rows
// at once with 16-byte loads, two column chunks in flight (8 loads per lane).
template <int TNW>
__device__ __forceinline__ double we_block_sum_n(double x, double* red) {
    x = we_warp_sum(x);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < TNW; ++w) s += red[w];
    return s;
}

template <int TT>
__global__ void __launch_bounds__(TT, 1) wide_tridiag_kernel(SvdTask* tasks, WParams P) {
    constexpr int TNW = TT / 32, PCN = 1024 / TT;
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[TNW];
    SvdTask& t = tasks[blockIdx.y];
    if (t.status != TASK_OK) return;
    const WLay L = wlay(t, P);
    if (L.flags[3] != 1) return;  // the same for every CTA of the cluster
    const WEig E = weig(L);
    const int n = wgeo(t).q, ld = L.qp;
    const int CL = gridDim.x, rank = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* A = L.g;
    double* vj = sm;            // current reflector
    double* vp = sm + ld;       // previous reflector
    double* wp = sm + 2 * ld;   // previous w
    double* row = sm + 3 * ld;  // row j with the pending update applied
    for (int c = tid; c < ld; c += TT) vp[c] = wp[c] = vj[c] = 0.0;
    __syncthreads();
    const int stride = CL * TNW;          // rows between two rows of one warp
    const int base = rank + CL * warp;    // row i belongs to CTA i % CL, warp (i / CL) % TNW
    for (int j = 0; j + 2 < n; ++j) {
        // ---- row j of the current matrix (every CTA, same bits), reflector j
        const double vpj = vp[j], wpj = wp[j];
        double ssq = 0.0;
        for (int c = j + tid; c < n; c += TT) {
            const double x = fma(-wpj, vp[c], fma(-vpj, wp[c], __ldcg(A + (int64_t)j * ld + c)));
            row[c] = x;
            if (c >= j + 2) ssq = fma(x, x, ssq);
        }
        ssq = we_block_sum_n<TNW>(ssq, red);  // (its barriers publish row[])
        const double alpha = row[j + 1];
        double beta = alpha, tau = 0.0, sc = 0.0;
        if (ssq > 0.0) {
            const double nrm = sqrt(fma(alpha, alpha, ssq));
            beta = alpha >= 0.0 ? -nrm : nrm;
            tau = (beta - alpha) / beta;
            sc = 1.0 / (alpha - beta);
        }
        for (int c = j + 1 + tid; c < n; c += TT) {
            const double v = c == j + 1 ? 1.0 : row[c] * sc;
            vj[c] = v;
            if (rank == 0) L.v[(int64_t)j * ld + c] = v;
        }
        if (tid == 0) vj[j] = 0.0;
        if (rank == 0 && tid == 0) {
            E.d[j] = row[j];
            E.e[j] = beta;
            E.tau[j] = tau;
        }
        __syncthreads();
        // ---- fused pass over this CTA's rows i > j: apply update j - 1, p_i = tau (row_i . v_j).
        // Columns from the even boundary at or below j + 1: column j is dead (finite
        // leftovers) and v_j, v_{j-1}, w_{j-1} are zero there; columns in [n, ld) are
        // zero padding of G and of the vectors.
        double* pb = E.pbuf + (int64_t)(j & 1) * ld;
        const int i0 = j + 1, c0 = i0 & ~1, cend = (n + 1) & ~1;
        const int s0 = i0 > base ? (i0 - base + stride - 1) / stride : 0;
        for (int ib = base + stride * s0; ib < n; ib += 4 * stride) {
            double* ar[4];
            double vpi[4], wpi[4], acc[4];
            bool live[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int i = ib + r * stride;
                live[r] = i < n;
                const int ic = live[r] ? i : ib;
                ar[r] = A + (int64_t)ic * ld;
                vpi[r] = vp[ic];
                wpi[r] = wp[ic];
                acc[r] = 0.0;
            }
            for (int c = c0 + 2 * lane; c < cend; c += 128) {
                const bool two = c + 64 < cend;
                double2 a[4][2];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    a[r][0] = live[r] ? __ldcg(reinterpret_cast<const double2*>(ar[r] + c)) : make_double2(0.0, 0.0);
                    a[r][1] = (live[r] && two) ? __ldcg(reinterpret_cast<const double2*>(ar[r] + c + 64))
                                               : make_double2(0.0, 0.0);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (h == 1 && !two) break;
                    const int cc = c + 64 * h;
                    const double2 v2 = *reinterpret_cast<const double2*>(vj + cc);
                    const double2 p2 = *reinterpret_cast<const double2*>(vp + cc);
                    const double2 w2 = *reinterpret_cast<const double2*>(wp + cc);
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        double2 x = a[r][h];
                        x.x = fma(-wpi[r], p2.x, fma(-vpi[r], w2.x, x.x));
                        x.y = fma(-wpi[r], p2.y, fma(-vpi[r], w2.y, x.y));
                        if (j > 0 && live[r]) __stcg(reinterpret_cast<double2*>(ar[r] + cc), x);
                        acc[r] = fma(x.x, v2.x, acc[r]);
                        acc[r] = fma(x.y, v2.y, acc[r]);
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const double pi = tau * we_warp_sum(acc[r]);
                if (lane == 0 && live[r]) __stcg(pb + ib + r * stride, pi);
            }
        }
        we_cluster_sync();
        // ---- w_j = p + K v_j, K = -tau/2 (p . v_j) (every CTA, same bits)
        double pc[PCN];
        double part = 0.0;
#pragma unroll
        for (int u = 0; u < PCN; ++u) {
            const int c = i0 + tid + u * TT;
            pc[u] = c < n ? __ldcg(pb + c) : 0.0;
            if (c < n) part = fma(pc[u], vj[c], part);
        }
        const double K = -0.5 * tau * we_block_sum_n<TNW>(part, red);
#pragma unroll
        for (int u = 0; u < PCN; ++u) {
            const int c = i0 + tid + u * TT;
            if (c < n) {
                wp[c] = fma(K, vj[c], pc[u]);
                vp[c] = vj[c];
            }
        }
        if (tid == 0) vp[j] = wp[j] = 0.0;
        __syncthreads();
    }
    // the trailing 2 x 2 block (pending update n - 3 applied)
    if (rank == 0 && tid == 0) {
        const int a = n - 2, b = n - 1;
        E.d[a] = __ldcg(A + (int64_t)a * ld + a) - 2.0 * vp[a] * wp[a];
        E.e[a] = __ldcg(A + (int64_t)a * ld + b) - vp[a] * wp[b] - wp[a] * vp[b];
        E.d[b] = __ldcg(A + (int64_t)b * ld + b) - 2.0 * vp[b] * wp[b];
        E.e[b] = 0.0;
        E.tau[a] = E.tau[b] = 0.0;
    }
}

// The kk largest eigenpairs of T and X = Q Z (q x kk, ld qp, into the V1
// region).  Cluster of gridDim.x (8 or 16) CTAs per task; eigenvalue g on
// warp g / cluster of CTA g % cluster.  NZ = ceil(q / 32) bound (registers of a column).
template <int NZ>
__global__ void __launch_bounds__(T, 1) wide_trieig_kernel(SvdTask* tasks, WParams P) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[NW];
    __shared__ int s_bad;
    SvdTask& t = tasks[blockIdx.y];
    if (t.status != TASK_OK) return;
    const WLay L = wlay(t, P);
    if (L.flags[3] != 1) return;
    const WEig E = weig(L);
    const int n = wgeo(t).q, ld = L.qp;
    const int rank = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int kk = min(t.trunc.k, n);
    const int g = rank + (int)gridDim.x * warp;  // this warp's eigenvalue (descending index)
    const bool mine = g < kk;
    double* d = sm;
    double* e = sm + ld;
    double* ee = sm + 2 * ld;
    double* tau = sm + 3 * ld;
    double* stage = sm + 4 * ld;  // 3 x ld reflector ring; first kk x 65 doubles double as B / R^-1
    // ---- T scaled by a power of two so that max |G| ~ 1
    const double gs = *L.gscale;
    const double scale = gs > 0.0 && isfinite(gs) ? we_renorm(gs, gs) : 1.0;
    for (int i = tid; i < n; i += T) {
        d[i] = scale * E.d[i];
        const double ei = i + 1 < n ? scale * E.e[i] : 0.0;
        e[i] = ei;
        ee[i] = ei * ei;
        tau[i] = E.tau[i];
    }
    if (tid == 0) s_bad = 0;
    __syncthreads();
    double glo, ghi;
    {
        double lo = 1e300, hi = -1e300;
        for (int i = lane; i < n; i += 32) {
            const double rad = fabs(i > 0 ? e[i - 1] : 0.0) + fabs(e[i]);
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
    const bool finite_t = isfinite(tnorm);
    double* lu = E.lu + (int64_t)g * 6 * ld;
    double* Ud = lu;
    double* U1 = lu + ld;
    double* U2 = lu + 2 * ld;
    double* Lm = lu + 3 * ld;
    double* Pv = lu + 4 * ld;
    double* Zs = lu + 5 * ld;
    double* zrow = E.z + (int64_t)g * ld;
    double z[NZ];
#pragma unroll
    for (int m = 0; m < NZ; ++m) z[m] = 0.0;
    bool bad = !finite_t;
    if (mine && finite_t) {
        // ---- eigenvalue g: 32-way multisection on Sturm counts (one point per lane)
        double lam;
        {
            const int target = n - 1 - g;  // ascending index
            double a = glo, b = ghi;
            const double rshrink = 1.0 / 33.0;
            int iters = 1;
            for (double w = ghi - glo; w > 4.0 * DBL_EPSILON * tnorm && iters < 200; w *= rshrink) ++iters;
            for (int it = 0; it < iters; ++it) {
                const double h = (b - a) * rshrink;
                const double x = fma((double)(lane + 1), h, a);
                double pa = 1.0, pb2 = d[0] - x;
                int sg = __double2hiint(pb2) >> 31;
                int cn = sg;
                int i = 1;
                for (; i + 8 <= n; i += 8) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const double q = fma(d[i + u] - x, pb2, -ee[i + u - 1] * pa);
                        const int s2 = __double2hiint(q) >> 31;
                        cn += s2 ^ sg;
                        sg = s2;
                        pa = pb2;
                        pb2 = q;
                    }
                    const double f = we_renorm(pa, pb2);
                    pa *= f;
                    pb2 *= f;
                }
                for (; i < n; ++i) {
                    const double q = fma(d[i] - x, pb2, -ee[i - 1] * pa);
                    const int s2 = __double2hiint(q) >> 31;
                    cn += s2 ^ sg;
                    sg = s2;
                    pa = pb2;
                    pb2 = q;
                }
                const int cnt = -cn;  // eigenvalues below x
                const unsigned ok = __ballot_sync(0xffffffffu, cnt <= target);
                const int nt = __popc(ok);
                const double na = nt > 0 ? fma((double)nt, h, a) : a;
                const double nb = nt < 32 ? fma((double)(nt + 1), h, a) : b;
                a = na;
                b = nb;
            }
            lam = 0.5 * (a + b);
            if (lane == 0) E.lam[g] = lam;
        }
        // ---- inverse iteration (dgttrf of T - lam I, partial pivoting; two solves).
        // The recurrences run on every lane alike; lane s keeps step 32 c + s of a
        // chunk and the chunk goes to / comes from L2 coalesced.
        const double pivmin = DBL_EPSILON * tnorm + 1e-300;
        const int nch = (n + 31) / 32;
        {
            double a = d[0] - lam, bsup = n > 1 ? e[0] : 0.0;
            double ycur = we_start(0, g);
            for (int c = 0; c < nch; ++c) {
                double k_ru = 0.0, k_u1 = 0.0, k_u2 = 0.0, k_l = 0.0, k_pv = 0.0, k_y = 0.0;
                const int lim = min(32, n - 32 * c);
                for (int s = 0; s < lim; ++s) {
                    const int i = 32 * c + s;
                    double ru, u1, u2, l, pv = 0.0, yout;
                    if (i + 1 < n) {
                        const double cc = e[i], a1 = d[i + 1] - lam, b1 = i + 2 < n ? e[i + 1] : 0.0;
                        double ynext = we_start(i + 1, g);
                        if (fabs(a) >= fabs(cc)) {
                            const double ui = fabs(a) < pivmin ? (a < 0.0 ? -pivmin : pivmin) : a;
                            ru = we_rcp(ui);
                            l = cc * ru;
                            u1 = bsup;
                            u2 = 0.0;
                            a = fma(-l, bsup, a1);
                            bsup = b1;
                            ynext = fma(-l, ycur, ynext);
                            yout = ycur;
                        } else {
                            pv = 1.0;
                            ru = we_rcp(cc);
                            l = a * ru;
                            u1 = a1;
                            u2 = b1;
                            a = fma(-l, a1, bsup);
                            bsup = -l * b1;
                            yout = ynext;  // rows i and i + 1 swap
                            ynext = fma(-l, yout, ycur);
                        }
                        ycur = ynext;
                    } else {
                        const double ui = fabs(a) < pivmin ? (a < 0.0 ? -pivmin : pivmin) : a;
                        ru = we_rcp(ui);
                        u1 = u2 = l = 0.0;
                        yout = ycur;
                    }
                    if (lane == s) {
                        k_ru = ru;
                        k_u1 = u1;
                        k_u2 = u2;
                        k_l = l;
                        k_pv = pv;
                        k_y = yout;
                    }
                }
                const int i = 32 * c + lane;
                if (i < n) {
                    Ud[i] = k_ru;
                    U1[i] = k_u1;
                    U2[i] = k_u2;
                    Lm[i] = k_l;
                    Pv[i] = k_pv;
                    Zs[i] = k_y;
                }
            }
        }
        __syncwarp();
        double inv = 1.0;
        for (int sweep = 0; sweep < 2; ++sweep) {
            if (sweep == 1) {  // P, L of the second solve on the rescaled first solution
                double xi = Zs[0] * inv;
                for (int c = 0; c < nch; ++c) {
                    const int il = 32 * c + lane;
                    const double r_l = il < n ? Lm[il] : 0.0, r_pv = il < n ? Pv[il] : 0.0;
                    const double r_z1 = il + 1 < n ? Zs[il + 1] * inv : 0.0;
                    double keep = 0.0;
                    const int lim = min(32, n - 32 * c);
                    for (int s = 0; s < lim; ++s) {
                        const int i = 32 * c + s;
                        const double l = __shfl_sync(0xffffffffu, r_l, s), pv = __shfl_sync(0xffffffffu, r_pv, s);
                        double x1 = __shfl_sync(0xffffffffu, r_z1, s);
                        double out;
                        if (i + 1 < n) {
                            if (pv != 0.0) {
                                const double tmp = xi;
                                xi = x1;
                                x1 = tmp;
                            }
                            out = xi;
                            xi = fma(-l, xi, x1);
                        } else {
                            out = xi;
                        }
                        if (lane == s) keep = out;
                    }
                    __syncwarp();
                    if (il < n) Zs[il] = keep;
                }
                __syncwarp();
            }
            double z2 = 0.0, z1 = 0.0, big = 0.0;
#pragma unroll
            for (int m = NZ - 1; m >= 0; --m) {
                if (m < nch) {
                    const int il = 32 * m + lane;
                    const double r_d = il < n ? Ud[il] : 0.0, r_1 = il < n ? U1[il] : 0.0, r_2 = il < n ? U2[il] : 0.0;
                    const double r_z = il < n ? Zs[il] : 0.0;
                    double keep = 0.0;
                    for (int s = min(31, n - 1 - 32 * m); s >= 0; --s) {
                        const double ud = __shfl_sync(0xffffffffu, r_d, s), u1 = __shfl_sync(0xffffffffu, r_1, s);
                        const double u2 = __shfl_sync(0xffffffffu, r_2, s), zi0 = __shfl_sync(0xffffffffu, r_z, s);
                        const double zi = fma(-u2, z2, fma(-u1, z1, zi0)) * ud;
                        big = fmax(big, fabs(zi));
                        z2 = z1;
                        z1 = zi;
                        if (lane == s) keep = zi;
                    }
                    z[m] = keep;
                    if (sweep == 0 && il < n) Zs[il] = keep;
                }
            }
            __syncwarp();
            if (sweep == 0) inv = big > 0.0 ? we_rcp(big) : 1.0;
        }
        // ---- normalise, residual in T's basis, publish the vector
        double nn = 0.0;
#pragma unroll
        for (int m = 0; m < NZ; ++m) nn = fma(z[m], z[m], nn);
        nn = we_warp_sum(nn);
        const double rn = nn > 0.0 && isfinite(nn) ? rsqrt(nn) : 0.0;
        if (rn == 0.0) bad = true;
#pragma unroll
        for (int m = 0; m < NZ; ++m) {
            z[m] *= rn;
            const int i = 32 * m + lane;
            if (i < n) zrow[i] = z[m];
        }
        __syncwarp();
        double worst = 0.0;
#pragma unroll
        for (int m = 0; m < NZ; ++m) {
            const int i = 32 * m + lane;
            if (i < n) {
                double r = (d[i] - lam) * z[m];
                if (i > 0) r = fma(e[i - 1], zrow[i - 1], r);
                if (i + 1 < n) r = fma(e[i], zrow[i + 1], r);
                worst = fmax(worst, fabs(r));
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
        if (!(worst <= 1e-11 * fmax(tnorm, 1e-300))) bad = true;
    }
    if (mine && lane == 0) E.res[g] = bad ? 1.0 : 0.0;
    // ---- Cholesky QR of the kk vectors, a second time when the first met a pivot below 1e-2:
    // one pass leaves an orthogonality error ~eps / (smallest pivot) — vectors of an
    // eigenvalue cluster come out of inverse iteration far from orthogonal, and a
    // single pass then missed the 1e-10 contract on V (1.8e-10 on a tenfold singular value)
    double* B = stage;            // kk x kk, ld 65
    double* Ri = stage + 64 * 65; // R^-1 (upper), ld 65
    for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) {
            we_cluster_sync();  // every warp has formed its vector from the first pass's Z
            if (mine) {
#pragma unroll
                for (int m = 0; m < NZ; ++m) {
                    const int i = 32 * m + lane;
                    if (i < n) zrow[i] = z[m];
                }
            }
        }
        we_cluster_sync();
        // B = Z Z^T rows of this warp's vector (z in registers against every vector)
        if (mine) {
            for (int h = 0; h < kk; ++h) {
                const double* zh = E.z + (int64_t)h * ld;
                double acc = 0.0;
#pragma unroll
                for (int m = 0; m < NZ; ++m) {
                    const int i = 32 * m + lane;
                    if (i < n) acc = fma(z[m], __ldcg(zh + i), acc);
                }
                acc = we_warp_sum(acc);
                if (lane == 0) __stcg(E.b + g * 64 + h, acc);
            }
        }
        we_cluster_sync();
        // Cholesky of B and R^-1 (every CTA, same bits); failures decided alike
        for (int x = tid; x < kk * kk; x += T) {
            const int a = x / kk, b = x - a * kk;
            B[a * 65 + b] = __ldcg(E.b + a * 64 + b);
        }
        for (int a = tid; a < kk; a += T)
            if (__ldcg(E.res + a) != 0.0) s_bad = 1;
        __syncthreads();
        double minpiv = 1.0;
        for (int jj = 0; jj < kk; ++jj) {
            const double djj = B[jj * 65 + jj];
            if (!(djj > 1e-6)) {  // (rows are unit vectors) uniform
                if (tid == 0) s_bad = 1;
                break;
            }
            minpiv = fmin(minpiv, djj);
            const double inv2 = 1.0 / djj;
            const int w = kk - jj - 1;
            for (int x = tid; x < w * w; x += T) {
                const int c = jj + 1 + x / w, c2 = jj + 1 + x % w;
                if (c2 >= c) B[c * 65 + c2] = fma(-B[jj * 65 + c] * inv2, B[jj * 65 + c2], B[c * 65 + c2]);
            }
            __syncthreads();
        }
        __syncthreads();
        if (s_bad) {
            if (rank == 0 && tid == 0) L.flags[3] = 2;  // the block-Jacobi path takes the task
            return;
        }
        // R[a][c] = B[a][c] / sqrt(B[a][a]) (a <= c).  R^-1 column c by back substitution.
        for (int c = tid; c < kk; c += T) {
            for (int a = c; a >= 0; --a) {
                double s0 = a == c ? 1.0 : 0.0, s1 = 0.0;
                const double ra = rsqrt(B[a * 65 + a]);
                int b = a + 1;
                for (; b + 1 <= c; b += 2) {
                    s0 = fma(-B[a * 65 + b] * ra, Ri[b * 65 + c], s0);
                    s1 = fma(-B[a * 65 + b + 1] * ra, Ri[(b + 1) * 65 + c], s1);
                }
                if (b <= c) s0 = fma(-B[a * 65 + b] * ra, Ri[b * 65 + c], s0);
                Ri[a * 65 + c] = (s0 + s1) * ra;  // / R[a][a] = sqrt(B[a][a])
            }
        }
        __syncthreads();
        // orthonormalised column g: z = sum_{a <= g} Ri[a][g] Z_a
        if (mine) {
#pragma unroll
            for (int m = 0; m < NZ; ++m) z[m] *= Ri[g * 65 + g];
            for (int a = 0; a < g; ++a) {
                const double f = Ri[a * 65 + g];
                const double* za = E.z + (int64_t)a * ld;
#pragma unroll
                for (int m = 0; m < NZ; ++m) {
                    const int i = 32 * m + lane;
                    if (i < n) z[m] = fma(f, __ldcg(za + i), z[m]);
                }
            }
        }
        __syncthreads();
        if (minpiv >= 1e-2) break;  // (the same on every CTA of the cluster)
    }
    __syncthreads();  // B / Ri done: the stage ring takes over
    // ---- back-transform X = H_0 H_1 ... H_{n-3} Z: reflectors n-3 .. 0, staged per CTA
    auto load_reflector = [&](int j) {
        if (j >= 0) {
            double* dst = stage + (int64_t)(j % 3) * ld;
            const double* src = L.v + (int64_t)j * ld;
            const int c0 = (j + 1) & ~1;
            for (int c = c0 + 2 * tid; c < ld; c += 2 * T) cp16(dst + c, src + c);
        }
        asm volatile("cp.async.commit_group;");
    };
    const int j0 = n - 3;
    load_reflector(j0);
    load_reflector(j0 - 1);
    for (int j = j0; j >= 0; --j) {
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        load_reflector(j - 2);
        const double tj = tau[j];
        if (mine && tj != 0.0) {
            const double* v = stage + (int64_t)(j % 3) * ld;
            double dot = 0.0;
#pragma unroll
            for (int m = 0; m < NZ; ++m) {
                const int i = 32 * m + lane;
                if (32 * m + 31 > j && i > j && i < n) dot = fma(v[i], z[m], dot);
            }
            const double f = -tj * we_warp_sum(dot);
#pragma unroll
            for (int m = 0; m < NZ; ++m) {
                const int i = 32 * m + lane;
                if (32 * m + 31 > j && i > j && i < n) z[m] = fma(f, v[i], z[m]);
            }
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (mine) {
#pragma unroll
        for (int m = 0; m < NZ; ++m) {
            const int i = 32 * m + lane;
            if (i < ld) L.v1[(int64_t)i * ld + g] = i < n ? z[m] : 0.0;
        }
    }
    if (rank == 0 && tid == 0) t.krank = kk;
}

// Narrow-engine tasks over Y = W X of the tasks on the direct route (one
// thread per task): SVD of Y (p x kk) = U' Sigma Z^T.  U' is A's U (tall A) or
// A's V (wide A, W = A^T) and goes straight to the outer task's factor; Z
// (kk x k, ld qp) goes to the M region for the X Z product.  Other tasks get
// an inert inner task.
__global__ void wide_eig_inner_kernel(SvdTask* tasks, SvdTask* inner, int n, WParams P, int nsplit, int rps,
                                      double* wsbase, int64_t wsstride) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const SvdTask& t = tasks[i];
        SvdTask in = {};
        in.status = kParked;
        in.m = in.n = 1;  // (an empty task would make mid-1 write its rank)
        if (t.status == TASK_OK) {
            const WLay L = wlay(t, P);
            if (L.flags[3] == 1) {
                const WGeo g = wgeo(t);
                in.a = L.y;
                in.lda = L.qp;
                in.m = g.p;
                in.n = t.krank;
                in.u = g.tall ? t.u : t.v;
                in.ldu = g.tall ? t.ldu : t.ldv;
                in.s = t.s;
                in.v = L.m;
                in.ldv = L.qp;
                in.k_out = t.k_out;
                in.kcap = t.kcap;
                in.trunc = t.trunc;
                in.sign = 0;
                in.status = TASK_OK;
                in.nsplit = nsplit;
                in.rows_per_split = rps;
                in.ws = wsbase + (int64_t)i * wsstride;
            }
        }
        inner[i] = in;
    }
}

// Results of the inner tasks back to the outer ones.  phase 0 (before the
// X Z product and the sign): rank and diagnostics; a task the inner engine
// finished on its robust path is marked flags[3] = 3, a failed one takes the
// inner status.  phase 1: finished tasks are parked (or DONE_FALLBACK) and the
// tasks the block-Jacobi path still has to take are counted.
__global__ void wide_eig_collect_kernel(SvdTask* tasks, const SvdTask* inner, int n, WParams P, int phase,
                                        int* remaining) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        SvdTask& t = tasks[i];
        if (t.status != TASK_OK) continue;
        const WLay L = wlay(t, P);
        if (phase == 0) {
            if (L.flags[3] != 1) continue;
            const SvdTask& in = inner[i];
            t.krank = in.krank;
            t.sweeps = in.sweeps;
            t.reason = in.reason;
            if (in.status == TASK_DONE_FALLBACK) L.flags[3] = 3;
            else if (in.status != TASK_OK) t.status = in.status;
        } else if (L.flags[3] == 1) {
            t.status = kParked;
            atomicAdd(&g_direct_tasks, 1ull);
        } else if (L.flags[3] == 3) {
            t.status = TASK_DONE_FALLBACK;
        } else {
            atomicAdd(remaining, 1);
        }
    }
}

// canonical_sign (svd.hpp:179-203) of the direct route's tasks, in two launches:
// the pivot (first largest |entry|) of each column of A's V decides the sign
// (grid: tasks; thread = (column tid % 64, row phase tid / 64), so a warp reads 32
// consecutive doubles of a row), then the flagged columns of V and U are flipped
// by row slices (grid: slices x tasks).
__global__ void __launch_bounds__(T) wide_eig_sign_kernel(SvdTask* tasks, WParams P) {
    __shared__ double s_best[4][64];
    __shared__ int s_idx[4][64];
    SvdTask& t = tasks[blockIdx.x];
    if (t.status != TASK_OK) return;
    const WLay L = wlay(t, P);
    if (L.flags[3] != 1 && L.flags[3] != 3) return;
    const WGeo g = wgeo(t);
    const int k = t.krank;  // <= 64
    const int c = threadIdx.x & 63, ph = threadIdx.x >> 6;
    const int nv = g.tall ? g.q : g.p;
    double best = -1.0;
    int bi = 0;
    if (c < k && t.sign) {
        int i = ph;
        for (; i + 12 < nv; i += 16) {
            double x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = fabs(t.v[(int64_t)(i + 4 * u) * t.ldv + c]);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (x[u] > best) {
                    best = x[u];
                    bi = i + 4 * u;
                }
        }
        for (; i < nv; i += 4) {
            const double x = fabs(t.v[(int64_t)i * t.ldv + c]);
            if (x > best) {
                best = x;
                bi = i;
            }
        }
    }
    s_best[ph][c] = best;
    s_idx[ph][c] = bi;
    __syncthreads();
    if (ph == 0 && c < 64) {
        bool neg = false;
        if (c < k && t.sign) {
            for (int h = 1; h < 4; ++h) {
                const double ob = s_best[h][c];
                const int oi = s_idx[h][c];
                if (ob > best || (ob == best && oi < bi)) {
                    best = ob;
                    bi = oi;
                }
            }
            neg = nv > 0 && t.v[(int64_t)bi * t.ldv + c] < 0.0;
        }
        L.sgn[c] = neg ? -1.0 : 1.0;
    }
}

__global__ void __launch_bounds__(T) wide_eig_flip_kernel(SvdTask* tasks, WParams P) {
    SvdTask& t = tasks[blockIdx.y];
    if (t.status != TASK_OK || !t.sign) return;
    const WLay L = wlay(t, P);
    if (L.flags[3] != 1 && L.flags[3] != 3) return;
    const WGeo g = wgeo(t);
    const int k = t.krank;
    const int c = threadIdx.x & 63, ph = threadIdx.x >> 6;
    if (c >= k || L.sgn[c] > 0.0) return;
    const int nv = g.tall ? g.q : g.p, nu = g.tall ? g.p : g.q;
    const int step = 4 * gridDim.x;
    for (int pass = 0; pass < 2; ++pass) {
        double* f = pass == 0 ? t.v : t.u;
        const int64_t ld = pass == 0 ? t.ldv : t.ldu;
        const int rows = pass == 0 ? nv : nu;
        int i = 4 * blockIdx.x + ph;
        for (; i + 3 * step < rows; i += 4 * step) {
            double x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = f[(int64_t)(i + u * step) * ld + c];
#pragma unroll
            for (int u = 0; u < 4; ++u) f[(int64_t)(i + u * step) * ld + c] = -x[u];
        }
        for (; i < rows; i += step) f[(int64_t)i * ld + c] = -f[(int64_t)i * ld + c];
    }
}

__global__ void wide_eig_unpark_kernel(SvdTask* tasks, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (tasks[i].status == kParked) tasks[i].status = TASK_OK;
}
