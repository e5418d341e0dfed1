// query_kernels.cu — the non-SVD kernels of the query phase (sm_100a).
//
//   stack_kernel  stacks diag(sigma_p) V_p^T of every part (query.hpp:113-122)
//                 and derives the band offsets on the device (ranks are
//                 device-resident, so no host round trip between kernels).
//   uform_kernel  U_out[rows of part p] = U_p * U_inner[band p]
//                 (query.hpp:129-141) — the blockdiag(U_i) U' product; rank-0
//                 parts give zero rows.  HBM-streaming: reads U_p once, writes
//                 U_out once, one CTA per (part, 64-row tile).
//   validate_kernel  finiteness of appended rows (store.hpp:41-50).
//   truncate_kernel / sign_kernel  standalone truncate_rank (svd.hpp:135-164)
//                 and canonical_sign (svd.hpp:179-203) for the L1 ABI.
#include <cstdint>

#include "zsvd_internal.h"

namespace zsvd {

__global__ void stack_kernel(const PartDesc* parts, int nparts, int c, double* stack,
                             int32_t* offs, int32_t* m_out) {
    ZSVD_PDL_WAIT();
    const int p = blockIdx.x;
    __shared__ int off, kp;
    __shared__ int wsum[32];
    // band offset = sum of the ranks of the parts before p (parallel loads)
    int acc = 0;
    for (int t = threadIdx.x; t < p; t += blockDim.x) acc += (int)parts[t].k_from[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int o = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) o += wsum[w];
        off = o;
        kp = (int)parts[p].k_from[0];
        offs[p] = o;
        if (p == nparts - 1) {
            offs[nparts] = o + kp;
            *m_out = o + kp;
        }
    }
    __syncthreads();
    const PartDesc d = parts[p];
    const int n = kp * c;
    for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
        int i = idx / c, j = idx % c;
        stack[(int64_t)(off + i) * c + j] = d.s[i] * d.v[(int64_t)j * d.ldv + i];
    }
}

// U_out rows of part blockIdx.y, tile blockIdx.x (64 rows):
// U_out[rowoff[p] + r] = U_p[r] * U_inner[offs[p] .. offs[p] + k_p)   (query.hpp:129-141)
// on DMMA: both operands staged in shared memory (rank padded to a multiple of
// 4, row strides = 4 mod 16 doubles: conflict-free fragments), warp w computes
// rows 8w .. 8w + 7 of the tile; ranks (kpm) and k_out are at most 64.
__device__ __forceinline__ void uform_dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__host__ __device__ constexpr int uform_ld(int n) { return n + ((4 - n % 16) + 16) % 16; }

__global__ void __launch_bounds__(256) uform_kernel(const PartDesc* parts, const int64_t* rowoff, int nparts,
                                                    const int32_t* offs, const double* uin, int64_t ldin,
                                                    const double* kout_ptr, double* uout, int64_t L, int kcap,
                                                    int kpm) {
    ZSVD_PDL_WAIT();
    extern __shared__ double ushm[];
    const int kpm4 = (kpm + 3) & ~3;
    const int wld = uform_ld(64), uld = uform_ld(kpm4);
    double* Ws = ushm;               // kpm4 x 64 (ld wld)
    double* Us = ushm + kpm4 * wld;  // 64 x kpm4 (ld uld)
    const int p = blockIdx.y;
    const PartDesc d = parts[p];
    const int64_t rows = rowoff[p + 1] - rowoff[p];
    const int64_t r0 = (int64_t)blockIdx.x * 64;
    if (r0 >= rows) return;
    const int nr = (int)(rows - r0 < 64 ? rows - r0 : 64);
    const int kout = (int)kout_ptr[0];
    const int kp = (int)d.k_from[0];
    if (kout == 0) return;
    double* out = uout + (rowoff[p] + r0) * kout;
    if (kp == 0) {  // rank-0 part: zero rows (query.hpp:133-140)
        for (int e = threadIdx.x; e < nr * kout; e += blockDim.x) out[e] = 0.0;
        return;
    }
    const int kp4 = (kp + 3) & ~3;
    const double* w = uin + (int64_t)offs[p] * ldin;
    for (int e = threadIdx.x; e < kp4 * 64; e += blockDim.x) {
        const int t = e >> 6, c = e & 63;
        Ws[t * wld + c] = (t < kp && c < kout) ? w[(int64_t)t * ldin + c] : 0.0;
    }
    for (int e = threadIdx.x; e < 64 * kp4; e += blockDim.x) {
        const int r = e / kp4, t = e - r * kp4;
        Us[r * uld + t] = (r < nr && t < kp) ? d.u[(r0 + r) * d.ldu + t] : 0.0;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nct = (kout + 7) >> 3;
    double c[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = 0.0;
    for (int s = 0; s < kp4 / 4; ++s) {
        const int k = 4 * s + (lane & 3);
        const double a = Us[(8 * warp + (lane >> 2)) * uld + k];
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (j < nct) uform_dmma(c[j][0], c[j][1], a, Ws[k * wld + 8 * j + (lane >> 2)]);
    }
    const int r = 8 * warp + (lane >> 2);
    if (r < nr) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int col = 8 * j + 2 * (lane & 3);
            if (col < kout) out[(int64_t)r * kout + col] = c[j][0];
            if (col + 1 < kout) out[(int64_t)r * kout + col + 1] = c[j][1];
        }
    }
}

// uform_kernel for ranks up to KC (<= 32; the BASELINE configs' k = 10 .. 30):
// no shared memory, no barriers.  The part's slice of U_inner is held in
// registers as DMMA B fragments for the whole kernel; each warp streams 8-row
// sub-tiles of U_p (A fragments straight from HBM, four sub-tiles in flight)
// and writes its 8 x k_out output rows as 16-byte stores.  Memory-bound: reads
// U_p once, writes U_out once.
template <int KC>
__global__ void __launch_bounds__(256, KC <= 16 ? 3 : 2) uform_reg_kernel(const PartDesc* parts, const int64_t* rowoff,
                                                           const int32_t* offs, const double* uin, int64_t ldin,
                                                           const double* kout_ptr, double* uout) {
    ZSVD_PDL_WAIT();
    constexpr int NS = KC / 4, NT = KC / 8;
    const int p = blockIdx.y;
    const PartDesc d = parts[p];
    const int64_t rows = rowoff[p + 1] - rowoff[p];
    const int kout = (int)kout_ptr[0];
    if (kout == 0) return;
    const int kp = (int)d.k_from[0];
    double* out = uout + rowoff[p] * kout;
    const int lane = threadIdx.x & 31;
    if (kp == 0) {  // rank-0 part: zero rows (query.hpp:133-140)
        for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * kout;
             e += (int64_t)gridDim.x * blockDim.x)
            out[e] = 0.0;
        return;
    }
    const double* w = uin + (int64_t)offs[p] * ldin;
    double B[NS][NT];
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            const int k = 4 * s + (lane & 3), n = 8 * j + (lane >> 2);
            B[s][j] = (k < kp && n < kout) ? w[(int64_t)k * ldin + n] : 0.0;
        }
    const int64_t nsub = (rows + 7) / 8;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const bool even = (kout & 1) == 0;
    auto tile = [&](int64_t st, const double (&A)[NS]) {
        double C[NT][2];
#pragma unroll
        for (int j = 0; j < NT; ++j) C[j][0] = C[j][1] = 0.0;
#pragma unroll
        for (int s = 0; s < NS; ++s)
#pragma unroll
            for (int j = 0; j < NT; ++j) uform_dmma(C[j][0], C[j][1], A[s], B[s][j]);
        const int64_t r = st * 8 + (lane >> 2);
        if (r >= rows) return;
        double* o = out + r * kout;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            const int col = 8 * j + 2 * (lane & 3);
            if (even && col + 1 < kout) {
                *reinterpret_cast<double2*>(o + col) = make_double2(C[j][0], C[j][1]);
            } else {
                if (col < kout) o[col] = C[j][0];
                if (col + 1 < kout) o[col + 1] = C[j][1];
            }
        }
    };
    auto load = [&](int64_t st, double (&A)[NS]) {
        const int64_t r = st * 8 + (lane >> 2);
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            const int k = 4 * s + (lane & 3);
            A[s] = (r < rows && k < kp) ? __ldg(d.u + r * d.ldu + k) : 0.0;
        }
    };
    int64_t st = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (; st + 3 * nw < nsub; st += 4 * nw) {  // four sub-tiles in flight
        double A0[NS], A1[NS], A2[NS], A3[NS];
        load(st, A0);
        load(st + nw, A1);
        load(st + 2 * nw, A2);
        load(st + 3 * nw, A3);
        tile(st, A0);
        tile(st + nw, A1);
        tile(st + 2 * nw, A2);
        tile(st + 3 * nw, A3);
    }
    for (; st < nsub; st += nw) {
        double A0[NS];
        load(st, A0);
        tile(st, A0);
    }
}
template __global__ void uform_reg_kernel<8>(const PartDesc*, const int64_t*, const int32_t*, const double*, int64_t,
                                             const double*, double*);
template __global__ void uform_reg_kernel<16>(const PartDesc*, const int64_t*, const int32_t*, const double*, int64_t,
                                              const double*, double*);
template __global__ void uform_reg_kernel<24>(const PartDesc*, const int64_t*, const int32_t*, const double*, int64_t,
                                              const double*, double*);
template __global__ void uform_reg_kernel<32>(const PartDesc*, const int64_t*, const int32_t*, const double*, int64_t,
                                              const double*, double*);

// uform_kernel for ranks above 64 (energy policy on c > 64 stores): row tile
// blockIdx.x (64 rows) of part blockIdx.y, column tile
// blockIdx.z (64 of the k_out columns):
// U_out[rowoff[p] + r] = U_p[r] * U_inner[offs[p] .. offs[p] + k_p)   (query.hpp:129-141)
// Operands staged in shared memory 64 ranks at a time; each thread keeps 16
// outputs of the 64 x nc tile in registers (compact: thread-major over the
// nr x nc outputs); output rows are contiguous.
__global__ void __launch_bounds__(256) uform_wide_kernel(const PartDesc* parts, const int64_t* rowoff, int nparts,
                                                    const int32_t* offs, const double* uin, int64_t ldin,
                                                    const double* kout_ptr, double* uout, int64_t L, int kcap) {
    ZSVD_PDL_WAIT();
    extern __shared__ double ushm[];
    double* Ws = ushm;             // 64 ranks x 64 output columns
    double* Us = ushm + 64 * 64;   // 64 rows x 64 ranks (ld 65)
    const int p = blockIdx.y;
    const PartDesc d = parts[p];
    const int64_t rows = rowoff[p + 1] - rowoff[p];
    const int64_t r0 = (int64_t)blockIdx.x * 64;
    if (r0 >= rows) return;
    const int nr = (int)(rows - r0 < 64 ? rows - r0 : 64);
    const int kout = (int)kout_ptr[0];
    const int c0 = 64 * blockIdx.z;
    if (c0 >= kout) return;
    const int nc = kout - c0 < 64 ? kout - c0 : 64;
    const int kp = (int)d.k_from[0];
    double* out = uout + (rowoff[p] + r0) * kout + c0;
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.0;
    const double* w = uin + (int64_t)offs[p] * ldin + c0;
    for (int t0 = 0; t0 < kp; t0 += 64) {  // rank-0 parts keep zero rows (query.hpp:133-140)
        const int tk = kp - t0 < 64 ? kp - t0 : 64;
        for (int e = threadIdx.x; e < tk * 64; e += blockDim.x) {
            const int t = e / 64, c = e % 64;
            Ws[t * 64 + c] = c < nc ? w[(int64_t)(t0 + t) * ldin + c] : 0.0;
        }
        for (int e = threadIdx.x; e < nr * tk; e += blockDim.x) {
            const int r = e / tk, t = e % tk;
            Us[r * 65 + t] = d.u[(r0 + r) * d.ldu + t0 + t];
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int e = threadIdx.x + 256 * i, r = e / nc, c = e % nc;
            if (r < nr) {
                const double* ur = Us + r * 65;
                double a = acc[i];
                for (int t = 0; t < tk; ++t) a = fma(ur[t], Ws[t * 64 + c], a);
                acc[i] = a;
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int e = threadIdx.x + 256 * i, r = e / nc, c = e % nc;
        if (r < nr) out[(int64_t)r * kout + c] = acc[i];
    }
}

// Grid-stride over rows; each warp scans whole rows (coalesced), no divisions.
__global__ void validate_kernel(const double* rows, int64_t nrows, int c, int64_t ld,
                                int32_t* bad) {
    const int lane = threadIdx.x & 31;
    bool ok = true;
    if (ld == c && (reinterpret_cast<uintptr_t>(rows) & 15) == 0) {
        // compact rows: one flat stream of 16-byte loads, four per thread in
        // flight (a warp-per-row loop keeps too few bytes in flight for HBM)
        const int64_t total = nrows * c, n2 = total / 2;
        const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        const int64_t nth = (int64_t)gridDim.x * blockDim.x;
        const double2* p = reinterpret_cast<const double2*>(rows);
        int64_t i = tid;
        for (; i + 3 * nth < n2; i += 4 * nth) {
            const double2 a = p[i], b = p[i + nth], c2 = p[i + 2 * nth], d = p[i + 3 * nth];
            ok &= isfinite(a.x) & isfinite(a.y) & isfinite(b.x) & isfinite(b.y) & isfinite(c2.x) & isfinite(c2.y) &
                  isfinite(d.x) & isfinite(d.y);
        }
        for (; i < n2; i += nth) ok &= isfinite(p[i].x) & isfinite(p[i].y);
        if (tid == 0 && (total & 1)) ok &= isfinite(rows[total - 1]);
    } else {
        const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
        const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
        for (int64_t r = warp; r < nrows; r += nwarps) {
            const double* row = rows + r * ld;
            for (int j = lane; j < c; j += 32) ok &= isfinite(row[j]);
        }
    }
    if (!__all_sync(0xffffffffu, ok) && lane == 0) *bad = 1;
}

// Copies leading keep columns of (u, s, v) after computing keep exactly as
// truncate_rank does.  Single CTA.
__global__ void truncate_kernel(const double* u, const double* s, const double* v,
                                const double* k_in, int64_t m, int64_t n, int64_t ldu,
                                int64_t ldv, Trunc tr, double* uo, double* so, double* vo,
                                double* ko) {
    __shared__ int keep;
    const int r = (int)k_in[0];
    if (threadIdx.x == 0) {
        int kk = r;
        if (tr.kind == TRUNC_FIXED) {
            kk = tr.k < r ? tr.k : r;
        } else if (tr.kind == TRUNC_ENERGY) {
            double total = 0.0;
            for (int i = 0; i < r; ++i) total += s[i] * s[i];
            if (total == 0.0) {
                kk = 0;
            } else {
                double cum = 0.0;
                for (int i = 0; i < r; ++i) {
                    cum += s[i] * s[i];
                    if (cum / total >= tr.xi) {
                        kk = i + 1;
                        break;
                    }
                }
            }
        }
        keep = kk;
        *ko = (double)kk;
    }
    __syncthreads();
    const int k = keep;
    for (int64_t e = threadIdx.x; e < m * k; e += blockDim.x) uo[e] = u[(e / k) * ldu + e % k];
    for (int64_t e = threadIdx.x; e < n * k; e += blockDim.x) vo[e] = v[(e / k) * ldv + e % k];
    for (int e = threadIdx.x; e < k; e += blockDim.x) so[e] = s[e];
}

// canonical_sign on compact (ld = k) factors, in place.  One warp per column.
__global__ void sign_kernel(double* u, double* v, const double* k_in, int64_t m, int64_t n) {
    const int k = (int)k_in[0];
    const int lane = threadIdx.x & 31;
    const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (c >= k) return;
    double best = -1.0;
    int64_t idx = INT64_MAX;
    for (int64_t r = lane; r < n; r += 32) {
        double mag = fabs(v[r * k + c]);
        if (mag > best) { best = mag; idx = r; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double ob = __shfl_xor_sync(0xffffffffu, best, o);
        int64_t oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ob > best || (ob == best && oi < idx)) { best = ob; idx = oi; }
    }
    if (n > 0 && v[idx * k + c] < 0.0) {
        for (int64_t r = lane; r < n; r += 32) v[r * k + c] = -v[r * k + c];
        for (int64_t r = lane; r < m; r += 32) u[r * k + c] = -u[r * k + c];
    }
}

}  // namespace zsvd

namespace zsvd {

// ---------------------------------------------------------------------------
// Batched window queries for similar_range_search (analysis.hpp:78-148).
//
// stack_multi_kernel: the stack_kernel of many stitches at once.  Part p of
// the concatenated part list belongs to window part_win[p]; its band offset
// sums the ranks of the window's earlier parts; the window's stack starts at
// stack + win_stack_off[w] and its height goes to m_out[w].
__global__ void stack_multi_kernel(const PartDesc* parts, const int32_t* part_win, const int32_t* win_part0,
                                   const int32_t* win_nparts, const int64_t* win_stack_off, int c, double* stack,
                                   int32_t* offs, int32_t* m_out) {
    const int p = blockIdx.x;
    const int w = part_win[p], p0 = win_part0[w];
    __shared__ int off, kp;
    __shared__ int wsum[32];
    int acc = 0;
    for (int t = p0 + threadIdx.x; t < p; t += blockDim.x) acc += (int)parts[t].k_from[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int o = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) o += wsum[i];
        off = o;
        kp = (int)parts[p].k_from[0];
        offs[p] = o;
        if (p == p0 + win_nparts[w] - 1) m_out[w] = o + kp;
    }
    __syncthreads();
    const PartDesc d = parts[p];
    double* st = stack + win_stack_off[w];
    for (int idx = threadIdx.x; idx < kp * c; idx += blockDim.x) {
        const int i = idx / c, j = idx % c;
        st[(int64_t)(off + i) * c + j] = d.s[i] * d.v[(int64_t)j * d.ldv + i];
    }
}

// One item = a part of a stitched window (its rows of the window's leading
// left singular vector are U_p * U_inner[band p, 0]) or a single-block window
// (the column 0 of its trim's U).  Writes (u1 . base_u1, |u1|^2) over the
// item's rows, reduced in a fixed order (analysis.hpp:89-103).
__global__ void __launch_bounds__(256) similarity_kernel(const SimItem* items, const double* base_u1,
                                                         int64_t base_ld, double2* partial) {
    const SimItem it = items[blockIdx.x];
    const int kp = (int)it.k_from[0];
    __shared__ double wv[64];
    __shared__ double2 red[8];
    const double* wcol = it.w ? it.w + (int64_t)(it.band ? *it.band : 0) * it.ldw : nullptr;
    if (wcol && threadIdx.x < kp && threadIdx.x < 64) wv[threadIdx.x] = wcol[(int64_t)threadIdx.x * it.ldw];
    __syncthreads();
    double dot = 0.0, nrm = 0.0;
    if (kp > 0) {
        for (int64_t r = threadIdx.x; r < it.rows; r += blockDim.x) {
            const double* ur = it.u + r * it.ldu;
            double x;
            if (wcol) {
                x = 0.0;
                for (int t = 0; t < kp && t < 64; ++t) x = fma(ur[t], wv[t], x);
                for (int t = 64; t < kp; ++t) x = fma(ur[t], wcol[(int64_t)t * it.ldw], x);
            } else {
                x = ur[0];
            }
            dot = fma(x, base_u1[(it.row0 + r) * base_ld], dot);
            nrm = fma(x, x, nrm);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dot += __shfl_xor_sync(0xffffffffu, dot, o);
        nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = make_double2(dot, nrm);
    __syncthreads();
    if (threadIdx.x == 0) {
        double2 s = red[0];
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            s.x += red[i].x;
            s.y += red[i].y;
        }
        partial[blockIdx.x] = s;
    }
}

// out[i] = *src[i] (the windows' ranks, scattered through the batch buffers).
__global__ void gather_kernel(const double* const* src, int n, double* out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = *src[i];
}


// ---------------------------------------------------------------------------
// naive_range_svd / reconstruction_error (analysis.hpp:20-66).
//
// reconstruct_kernel: rows [tile * tr, +tr) of part blockIdx.y, i.e.
// out[rowoff[p] + r] = U_p[r] diag(sigma_p) V_p^T (the range's raw rows rebuilt
// from the stored factors; U_p already offset to the first kept row).
__global__ void __launch_bounds__(256) reconstruct_kernel(const PartDesc* parts, const int64_t* rowoff, int c,
                                                          double* out, int tr) {
    extern __shared__ double rsm[];  // tr x (k + 1): U rows scaled by sigma
    const PartDesc d = parts[blockIdx.y];
    const int64_t rows = rowoff[blockIdx.y + 1] - rowoff[blockIdx.y];
    const int64_t r0 = (int64_t)blockIdx.x * tr;
    if (r0 >= rows) return;
    const int nr = (int)(rows - r0 < tr ? rows - r0 : tr);
    const int k = (int)d.k_from[0];
    const int ld = k + 1;
    for (int e = threadIdx.x; e < nr * k; e += blockDim.x) {
        const int r = e / k, t = e % k;
        rsm[r * ld + t] = d.u[(r0 + r) * d.ldu + t] * d.s[t];
    }
    __syncthreads();
    double* o = out + (rowoff[blockIdx.y] + r0) * c;
    for (int e = threadIdx.x; e < nr * c; e += blockDim.x) {
        const int r = e / c, j = e % c;
        const double* vr = d.v + (int64_t)j * d.ldv;
        double acc = 0.0;
        for (int t = 0; t < k; ++t) acc = fma(rsm[r * ld + t], vr[t], acc);
        o[(int64_t)r * c + j] = acc;
    }
}

// Partial sums (|X - U S V^T|^2, |X|^2) of rows [blockIdx.x * tr, +tr): one
// double2 per CTA, summed on the host in CTA order (deterministic).
__global__ void __launch_bounds__(256) recon_error_kernel(const double* x, int64_t m, int n, const double* u,
                                                          int64_t ldu, const double* s, const double* v,
                                                          int64_t ldv, const double* k_ptr, double2* partial, int tr) {
    extern __shared__ double esm[];  // tr x (k + 1)
    __shared__ double2 red[8];
    const int k = (int)k_ptr[0];
    const int ld = k + 1;
    const int64_t r0 = (int64_t)blockIdx.x * tr;
    const int nr = (int)(m - r0 < tr ? m - r0 : tr);
    for (int e = threadIdx.x; e < nr * k; e += blockDim.x) {
        const int r = e / k, t = e % k;
        esm[r * ld + t] = u[(r0 + r) * ldu + t] * s[t];
    }
    __syncthreads();
    double num = 0.0, den = 0.0;
    for (int e = threadIdx.x; e < nr * n; e += blockDim.x) {
        const int r = e / n, j = e % n;
        const double* vr = v + (int64_t)j * ldv;
        double acc = 0.0;
        for (int t = 0; t < k; ++t) acc = fma(esm[r * ld + t], vr[t], acc);
        const double xv = x[(r0 + r) * n + j];
        num = fma(xv - acc, xv - acc, num);
        den = fma(xv, xv, den);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, o);
        den += __shfl_xor_sync(0xffffffffu, den, o);
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = make_double2(num, den);
    __syncthreads();
    if (threadIdx.x == 0) {
        double2 t = red[0];
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            t.x += red[i].x;
            t.y += red[i].y;
        }
        partial[blockIdx.x] = t;
    }
}


// ---------------------------------------------------------------------------
// orthonormality_defect (svd.hpp:48-58): max |M^T M - I|.
//
// defect_partial_kernel: CTA (x = 32 x 32 column-tile pair, y = row split)
// sums rows [y * rps, +rps) of tiles (ti, tj), ti <= tj, in row order, staging
// 32 rows of both column tiles in shared memory; thread (ty, tx) owns entries
// (4 ty + q, tx).  defect_reduce_kernel adds the splits in order (bitwise
// reproducible) and writes each tile pair's max |G - I|.
__global__ void __launch_bounds__(256) defect_partial_kernel(const double* __restrict__ m, int64_t rows, int cols,
                                                             int64_t ld, int64_t rps, double* __restrict__ partial) {
    __shared__ double a[32][33], b[32][33];
    const int nt = (cols + 31) / 32;
    int t = blockIdx.x, ti = 0;
    while (t >= nt - ti) {
        t -= nt - ti;
        ++ti;
    }
    const int tj = ti + t;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t r0 = (int64_t)blockIdx.y * rps;
    const int64_t r1 = r0 + rps < rows ? r0 + rps : rows;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t rr = r0; rr < r1; rr += 32) {
        for (int e = threadIdx.x; e < 32 * 32; e += 256) {
            const int r = e >> 5, cc = e & 31;
            const bool in = rr + r < r1;
            const int ca = ti * 32 + cc, cb = tj * 32 + cc;
            a[r][cc] = in && ca < cols ? m[(rr + r) * ld + ca] : 0.0;
            b[r][cc] = in && cb < cols ? m[(rr + r) * ld + cb] : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int r = 0; r < 32; ++r) {
            const double bv = b[r][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = fma(a[r][4 * ty + q], bv, acc[q]);
        }
        __syncthreads();
    }
    double* out = partial + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * 1024;
#pragma unroll
    for (int q = 0; q < 4; ++q) out[(4 * ty + q) * 32 + tx] = acc[q];
}

__global__ void __launch_bounds__(256) defect_reduce_kernel(const double* __restrict__ partial, int npairs, int nsplit,
                                                            int cols, double* __restrict__ tile_max) {
    __shared__ double red[8];
    const int nt = (cols + 31) / 32;
    int t = blockIdx.x, ti = 0;
    while (t >= nt - ti) {
        t -= nt - ti;
        ++ti;
    }
    const int tj = ti + t;
    double worst = 0.0;
    for (int e = threadIdx.x; e < 1024; e += 256) {
        const int i = ti * 32 + (e >> 5), j = tj * 32 + (e & 31);
        if (i >= cols || j >= cols) continue;
        double g = 0.0;
        for (int y = 0; y < nsplit; ++y) g += partial[((int64_t)y * npairs + blockIdx.x) * 1024 + e];
        const double d = fabs(g - (i == j ? 1.0 : 0.0));
        worst = d > worst || d != d ? d : worst;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double w = __shfl_xor_sync(0xffffffffu, worst, o);
        worst = w > worst || w != w ? w : worst;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = worst;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < 8; ++i) worst = red[i] > worst || red[i] != red[i] ? red[i] : worst;
        tile_max[blockIdx.x] = worst;
    }
}

}  // namespace zsvd
