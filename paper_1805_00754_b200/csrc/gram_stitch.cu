// gram_stitch.cu — range_query (query.hpp:163-191) as a Gram stitch, for the
// narrow engine (c <= 64) under a truncation the boundary trims cannot change
// (FIXED_RANK k >= the blocks' rank capacity).
//
// The reference trims the head and tail blocks (trim_block, query.hpp:64-89),
// stacks sigma_p V_p^T of every part (query.hpp:113-122) and takes the SVD of
// the stack S (query.hpp:124).  S enters that SVD only through its Gram
// G = S^T S = sum_p V_p Sigma_p C_p Sigma_p V_p^T, where C_p = I for a stored
// block (U_p orthonormal) and C_p = U_s^T U_s for the row slice U_s of the
// head / tail block: a no-op trim (its truncation keeps every column) turns the
// slice U_s Sigma V^T into factors with exactly that Gram.  So
//
//   gram_parts_kernel   G's partial sums straight from the stored factors (no
//                       trims, no stack): each CTA folds a run of parts / slice
//                       chunks, the 8 CTAs of a cluster add their partials over
//                       distributed shared memory, one partial per cluster lands
//                       in the task workspace (the layout P1 would write);
//   gram_eig_kernel     the top-k eigenpairs of G (eigh.cuh: tridiagonalisation,
//                       bisection, inverse iteration): sigma = sqrt(lambda), V
//                       (sign-canonical, svd.hpp:179-203) and M = V_k Sigma_k^-1
//                       (with U_inner = S M);
//   uform_gram_kernel   U_out rows of part p = U_p (Sigma_p V_p^T M)
//                       (query.hpp:129-141 with U_inner's band formed in place),
//                       plus sigma and the rank.
//
// Accuracy is that of one-pass CholeskyQR: the kept sigma_j and
// V carry eps (sigma_1 / sigma_j)^2 errors, so a retained spectrum spread
// beyond sigma_1 > 3000 sigma_k (or a failed eigensolver check) flags the task
// and the host redoes the query on the trim + stack engine path (zsvd_api.cu).
#include <cstdint>

#include "zsvd_internal.h"

namespace zsvd {

constexpr int kGramCluster = 8;
constexpr int kGramChunk = 128;  // slice rows per work item
constexpr int kVL = 68;          // row stride of the j-major tiles (doubles; 16-byte aligned rows)
constexpr int kUL = 33;          // row stride of the staged U chunk
constexpr int kCL = 33;          // row stride of C

namespace {
__device__ __forceinline__ unsigned gs_cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void gs_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ const double* gs_peer(const double* p, unsigned rank) {
    const double* out;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(p), "r"(rank));
    return out;
}

// Shared-memory plan of gram_parts_kernel (doubles).
constexpr int kOffVS = 0;                          // VS^T: kp x c, ld kVL
constexpr int kOffT = kOffVS + 32 * kVL;           // T^T = (VS C)^T: kp x c, ld kVL
constexpr int kOffC = kOffT + 32 * kVL;            // C: kp x kp, ld kCL
constexpr int kOffU = kOffC + 32 * kCL;            // U chunk: rows x kp, ld kUL
constexpr int kOffCP = kOffU + kGramChunk * kUL;   // 4 row-group partials of C, 32 x 33 each
constexpr int kSmemD = kOffCP + 4 * 32 * 33;
static_assert(64 * 64 <= kGramChunk * kUL + 4 * 32 * 33, "final partial must fit the U / C-partial region");

// rows x cols block of a row-major source (ld sld) into shared memory, either
// row-major (dld) or transposed (dst[col * dld + row]), optionally times
// scale[col]; every load of the block is issued before the first store.
template <bool TRANS>
__device__ __forceinline__ void stage_block(double* dst, int dld, const double* src, int64_t sld, int rows, int cols,
                                            const double* scale) {
    const int n = rows * cols;
    for (int e0 = 0; e0 < n; e0 += 8 * 256) {
        double v[8];
        int rr[8], cc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int e = e0 + threadIdx.x + 256 * i;
            rr[i] = e / cols;
            cc[i] = e - rr[i] * cols;
            v[i] = e < n ? __ldg(src + (int64_t)rr[i] * sld + cc[i]) : 0.0;
        }
        if (scale) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (e0 + threadIdx.x + 256 * i < n) v[i] *= __ldg(scale + cc[i]);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (e0 + threadIdx.x + 256 * i < n) {
                if (TRANS) dst[cc[i] * dld + rr[i]] = v[i];
                else dst[rr[i] * dld + cc[i]] = v[i];
            }
    }
}

// acc (4 x 4 tile at rows tr, cols tc of a 64 x 64) += A^T B over j < kd, A and
// B j-major (ld kVL)
__device__ __forceinline__ void tile_rank_update(double (&acc)[4][4], const double* A, const double* B, int kd, int tr,
                                                 int tc) {
    for (int j = 0; j < kd; ++j) {
        const double2 x0 = *reinterpret_cast<const double2*>(A + j * kVL + tr);
        const double2 x1 = *reinterpret_cast<const double2*>(A + j * kVL + tr + 2);
        const double2 y0 = *reinterpret_cast<const double2*>(B + j * kVL + tc);
        const double2 y1 = *reinterpret_cast<const double2*>(B + j * kVL + tc + 2);
        const double x[4] = {x0.x, x0.y, x1.x, x1.y}, y[4] = {y0.x, y0.y, y1.x, y1.y};
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = fma(x[a], y[b], acc[a][b]);
    }
}
}  // namespace

int gram_parts_smem_bytes() { return 8 * kSmemD; }

// Thread t owns the 4 x 4 tile (rows 4 (t / 16) .., cols 4 (t % 16) ..) of the
// CTA's 64 x 64 partial Gram.  CTA b folds items [item_start[b],
// item_start[b + 1]) (kp <= 32):
//   stored block      G += VS VS^T, VS = V diag(sigma)
//   slice chunk       C = U_c^T U_c (four row groups, summed), T = VS C,
//                     G += T VS^T
// The 8 CTAs of a cluster add their partials over distributed shared memory
// (CTA r: rows [8r, 8r + 8), peers in rank order) into one cluster partial in
// global scratch; the last CTA of each row band to arrive (ticket) adds the
// cluster partials in cluster order into `out` (c x c, ld kQMax).  Every sum
// has a fixed order: the result is bitwise reproducible.
__global__ void __cluster_dims__(kGramCluster, 1, 1) __launch_bounds__(256, 2)
    gram_parts_kernel(const GramPart* parts, const GramItem* items, const int32_t* item_start, int c,
                      double* cluster_ws, unsigned* tickets, double* out) {
    ZSVD_PDL_WAIT();
    extern __shared__ __align__(16) double gsh[];
    double* VS = gsh + kOffVS;
    double* Tt = gsh + kOffT;
    double* Cm = gsh + kOffC;
    double* Uc = gsh + kOffU;
    double* Cp = gsh + kOffCP;
    const int tid = threadIdx.x;
    const int tr = (tid >> 4) * 4, tc = (tid & 15) * 4;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    const int i0 = item_start[blockIdx.x], i1 = item_start[blockIdx.x + 1];
    for (int it = i0; it < i1; ++it) {
        const GramItem item = items[it];
        const GramPart d = parts[item.part];
        const int kcap = (int)d.ldv;  // factors stored at capacity kcap (slot layout)
        __syncthreads();              // the previous item is done with the shared buffers
        // loads issued before the rank arrives: columns beyond it are never read
        stage_block<true>(VS, kVL, d.v, d.ldv, c, kcap, d.s);
        if (d.slice) stage_block<false>(Uc, kUL, d.u + (int64_t)item.row0 * d.ldu, d.ldu, item.nrows, kcap, nullptr);
        const int kp = (int)d.k_from[0];
        if (kp == 0) continue;
        if (!d.slice) {
            __syncthreads();
            tile_rank_update(acc, VS, VS, kp, tr, tc);
            continue;
        }
        const int nr = item.nrows;
        const int kp4 = (kp + 3) & ~3;
        if (kp4 > kp)  // zero the U columns up to the 4-wide tile edge
            for (int e = tid; e < nr * (kp4 - kp); e += 256) Uc[(e / (kp4 - kp)) * kUL + kp + e % (kp4 - kp)] = 0.0;
        __syncthreads();
        {
            // C = U_c^T U_c: thread = 4 x 4 tile of the 32 x 32 (tid % 64), row
            // group tid / 64 of four; the row-group partials summed in order
            const int tile = tid & 63, rg = tid >> 6;
            const int cr = (tile >> 3) * 4, cc = (tile & 7) * 4;
            if (cr < kp && cc < kp) {
                double cacc[4][4];
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) cacc[a][b] = 0.0;
                for (int r = rg; r < nr; r += 4) {
                    double x[4], y[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) {
                        x[a] = Uc[r * kUL + cr + a];
                        y[a] = Uc[r * kUL + cc + a];
                    }
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b) cacc[a][b] = fma(x[a], y[b], cacc[a][b]);
                }
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) Cp[rg * 32 * 33 + (cr + a) * 33 + cc + b] = cacc[a][b];
            }
            __syncthreads();
            for (int e = tid; e < kp4 * kp4; e += 256) {
                const int i = e / kp4, j = e % kp4;
                Cm[i * kCL + j] = (Cp[i * 33 + j] + Cp[32 * 33 + i * 33 + j]) +
                                  (Cp[2 * 32 * 33 + i * 33 + j] + Cp[3 * 32 * 33 + i * 33 + j]);
            }
        }
        __syncthreads();
        {
            // T^T[j][l] = sum_i C[i][j] VS^T[i][l]: thread tile (j rows 4 (tid / 16), l cols 4 (tid % 16))
            const int jr = (tid >> 4) * 4, lc = (tid & 15) * 4;
            if (jr < kp) {
                double tacc[4][4];
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) tacc[a][b] = 0.0;
                for (int i = 0; i < kp; ++i) {
                    double x[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) x[a] = Cm[i * kCL + jr + a];
                    const double2 y0 = *reinterpret_cast<const double2*>(VS + i * kVL + lc);
                    const double2 y1 = *reinterpret_cast<const double2*>(VS + i * kVL + lc + 2);
                    const double y[4] = {y0.x, y0.y, y1.x, y1.y};
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b) tacc[a][b] = fma(x[a], y[b], tacc[a][b]);
                }
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) Tt[(jr + a) * kVL + lc + b] = tacc[a][b];
            }
        }
        __syncthreads();
        tile_rank_update(acc, Tt, VS, kp, tr, tc);
    }
    // cluster reduction through distributed shared memory
    double* P = Uc;  // 64 x 64
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) P[(tr + a) * 64 + tc + b] = acc[a][b];
    gs_cluster_sync();
    const unsigned rank = gs_cluster_rank();
    const int cluster = blockIdx.x / kGramCluster, ncl = gridDim.x / kGramCluster;
    double* cw = cluster_ws + (int64_t)cluster * kWsQ2;
    for (int e = tid; e < 8 * 64; e += 256) {
        const int i = (int)rank * 8 + (e >> 6), j = e & 63;
        double sum = 0.0;
#pragma unroll
        for (unsigned pr = 0; pr < kGramCluster; ++pr) sum += gs_peer(P + i * 64 + j, pr)[0];
        cw[i * 64 + j] = sum;
    }
    gs_cluster_sync();  // peers read this CTA's partial until here
    // the last cluster to finish a row band adds all cluster partials of it
    __shared__ unsigned last;
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(tickets + rank, 1u) == (unsigned)(ncl - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int e = tid; e < 8 * 64; e += 256) {
        const int i = (int)rank * 8 + (e >> 6), j = e & 63;
        double sum = 0.0;
        for (int k0 = 0; k0 < ncl; k0 += 8) {  // eight loads in flight, added in cluster order
            double v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                v[k] = k0 + k < ncl ? __ldcg(cluster_ws + (int64_t)(k0 + k) * kWsQ2 + i * 64 + j) : 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k) sum += v[k];
        }
        if (i < c && j < c) out[i * kQMax + j] = sum;
    }
}

// Sharded Gram stitch (zsvd_sharded_range_query): every rank's buffer holds its
// local Gram (64 x 64, upper triangle valid) then [eligible, stacked rows]; the
// Grams are added in rank order (the same bits on every rank, so every rank's
// eigensolver returns the same sigma and V) into the task's partial 0.  A rank
// that cannot take the Gram path, or a global stack shorter than c, flags the
// task on every rank alike.
constexpr int kShardRec = kWsQ2 + 8;
__global__ void __launch_bounds__(256) gram_gather_sum_kernel(const double* recv, int nranks, int c, SvdTask* task) {
    ZSVD_PDL_WAIT();
    bool ok = true;
    double kall = 0.0;
    for (int r = 0; r < nranks; ++r) {
        ok = ok && recv[(int64_t)r * kShardRec + kWsQ2] != 0.0;
        kall += recv[(int64_t)r * kShardRec + kWsQ2 + 1];
    }
    if (!ok || kall < (double)c) {
        if (threadIdx.x == 0 && blockIdx.x == 0) {
            task->status = TASK_NEEDS_FALLBACK;
            task->reason = ok ? 31 : 30;  // 30: a rank cannot take the Gram path; 31: stack shorter than c
        }
        return;
    }
    double* G = task->ws;
    for (int e = blockIdx.x * 256 + threadIdx.x; e < c * kQMax; e += gridDim.x * 256) {
        const int i = e / kQMax, j = e - i * kQMax;
        if (j >= c || j < i) continue;
        double s = 0.0;
        for (int r = 0; r < nranks; ++r) s += recv[(int64_t)r * kShardRec + e];
        G[e] = s;
    }
}
int gram_shard_record() { return kShardRec; }

// U_inner's band of part p = Sigma_p V_p^T M (k_p x k_out, query.hpp:129-141
// with U_inner = S M): one CTA per part, written at band p * kb (ld kq) for
// uform_reg_kernel; CTA 0 also writes sigma and the rank.  Nothing is written
// when the engine flagged the task (the host redoes the query).
__global__ void __launch_bounds__(256) gram_band_kernel(const GramPart* parts, const SvdTask* task, int c, int kb,
                                                        int kq, double* bands, double* s_out, double* k_out) {
    ZSVD_PDL_WAIT();
    __shared__ double Vs[64][33], Ms[64][33];
    if (task->status != TASK_OK) return;
    const int kout = task->krank;
    const double* tws = task->ws;
    const int tns = task->nsplit;
    if (blockIdx.x == 0) {
        const double* sg = tws + ws_off_sig(tns);
        if (threadIdx.x < kout) s_out[threadIdx.x] = sg[threadIdx.x];
        if (threadIdx.x == 0) k_out[0] = (double)kout;
    }
    const GramPart d = parts[blockIdx.x];
    const int kcap = (int)d.ldv;
    const double* M = tws + ws_off_m(tns);  // c x k_out, ld kQMax
    for (int e0 = 0; e0 < 64 * 32; e0 += 8 * 256) {  // all loads in flight, then stores
        double a[8], m[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int e = e0 + threadIdx.x + 256 * i, l = e >> 5, j = e & 31;
            a[i] = l < c && j < kcap ? d.v[(int64_t)l * d.ldv + j] : 0.0;
            m[i] = l < c && j < kout ? M[l * kQMax + j] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int e = e0 + threadIdx.x + 256 * i, l = e >> 5, j = e & 31;
            Vs[l][j] = a[i];
            Ms[l][j] = m[i];
        }
    }
    const int kp = (int)d.k_from[0];
    __syncthreads();
    double* band = bands + (int64_t)blockIdx.x * kb * kq;
    for (int e = threadIdx.x; e < kp * kout; e += 256) {
        const int j = e / kout, n = e % kout;
        double a0 = 0.0, a1 = 0.0;
        for (int l = 0; l < c; l += 2) {
            a0 = fma(Vs[l][j], Ms[l][n], a0);
            a1 = fma(Vs[l + 1][j], Ms[l + 1][n], a1);  // row c (odd c) is zero
        }
        band[j * kq + n] = d.s[j] * (a0 + a1);
    }
}

}  // namespace zsvd
