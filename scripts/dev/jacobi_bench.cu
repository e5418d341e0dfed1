// Standalone timing of one-sided Jacobi variants on batches of 64 x 64
// matrices (one CTA of 256 threads per matrix, matrix in shared memory), to
// pick the mapping used by the engine's Mid-2 phase. Dev tool.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o jb jacobi_bench.cu
//   ./jb
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

constexpr int Q = 64, JLD = 66, T = 256;

__device__ __forceinline__ void rot_angle(double a, double b, double g, double& cth, double& sth, double& tt) {
    const double d = b - a;
    const double h2 = fma(d, d, 4.0 * g * g);
    double rh, rd;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rh) : "d"(h2));
    const double den = fma(h2, rh, fabs(d));
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rd) : "d"(den));
    rd = rd * fma(-den, rd, 2.0);
    tt = 2.0 * g * rd;
    if (d < 0.0) tt = -tt;
    cth = rsqrt(fma(tt, tt, 1.0));
    sth = cth * tt;
}

template <int NT>
__device__ __forceinline__ void bar() {
    if constexpr (NT == T) __syncthreads();
    else asm volatile("bar.sync 1, %0;" ::"n"(NT));
}

// LPP lanes per pair, 32 pairs -> 32*LPP active threads. TRACK: column norms
// tracked through rotations (recomputed at every sweep start).
template <int LPP, bool TRACK>
__device__ void jacobi(double* Y, int q, int* flags, double* nrm, int* sweeps_out) {
    constexpr int NT = 32 * LPP;
    constexpr int EPL2 = Q / (2 * LPP);
    const double tol = (double)q * DBL_EPSILON, tol2 = tol * tol;
    if (threadIdx.x == 0) flags[0] = flags[1] = 0;
    __syncthreads();
    if (threadIdx.x >= NT) {
        __syncthreads();
        return;
    }
    const int slot = threadIdx.x / LPP, li = threadIdx.x % LPP;
    int sweep = 0;
    for (; sweep < 40; ++sweep) {
        const int fcur = sweep & 1;
        if (threadIdx.x == 0) flags[fcur ^ 1] = 0;
        if constexpr (TRACK) {
            for (int cc = slot; cc < Q; cc += 32) {
                const double2* col = reinterpret_cast<const double2*>(Y + cc * JLD);
                double a = 0.0;
#pragma unroll
                for (int e = 0; e < EPL2; ++e) {
                    const double2 v = col[li + e * LPP];
                    a = fma(v.x, v.x, fma(v.y, v.y, a));
                }
#pragma unroll
                for (int o = 1; o < LPP; o <<= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                if (li == 0) nrm[cc] = a;
            }
            bar<NT>();
        }
        for (int G = 32; G >= 1; G >>= 1) {
            const int grp = slot / G, ls = slot % G;
            const int xi = grp * 2 * G + ls;
            const bool xlive = xi < q;
            double2 X[EPL2], Yc[EPL2];
            const double2* xcol = reinterpret_cast<const double2*>(Y + xi * JLD);
#pragma unroll
            for (int e = 0; e < EPL2; ++e) X[e] = xlive ? xcol[li + e * LPP] : make_double2(0.0, 0.0);
            double an = TRACK ? nrm[xi] : 0.0;
            for (int r = 0; r < G; ++r) {
                const int yi = grp * 2 * G + G + ((ls + r) & (G - 1));
                const bool act = xlive && yi < q;
                double2* ycol = reinterpret_cast<double2*>(Y + yi * JLD);
#pragma unroll
                for (int e = 0; e < EPL2; ++e) Yc[e] = act ? ycol[li + e * LPP] : make_double2(0.0, 0.0);
                double a, b, g;
                if constexpr (TRACK) {
                    double g0 = 0.0, g1 = 0.0;
#pragma unroll
                    for (int e = 0; e < EPL2; ++e) {
                        g0 = fma(X[e].x, Yc[e].x, g0);
                        g1 = fma(X[e].y, Yc[e].y, g1);
                    }
                    g = g0 + g1;
#pragma unroll
                    for (int o = 1; o < LPP; o <<= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
                    a = an;
                    b = nrm[yi];
                } else {
                    double a0 = 0, b0 = 0, g0 = 0, a1 = 0, b1 = 0, g1 = 0;
#pragma unroll
                    for (int e = 0; e < EPL2; ++e) {
                        a0 = fma(X[e].x, X[e].x, a0);
                        b0 = fma(Yc[e].x, Yc[e].x, b0);
                        g0 = fma(X[e].x, Yc[e].x, g0);
                        a1 = fma(X[e].y, X[e].y, a1);
                        b1 = fma(Yc[e].y, Yc[e].y, b1);
                        g1 = fma(X[e].y, Yc[e].y, g1);
                    }
                    a = a0 + a1;
                    b = b0 + b1;
                    g = g0 + g1;
#pragma unroll
                    for (int o = 1; o < LPP; o <<= 1) {
                        a += __shfl_xor_sync(0xffffffffu, a, o);
                        b += __shfl_xor_sync(0xffffffffu, b, o);
                        g += __shfl_xor_sync(0xffffffffu, g, o);
                    }
                }
                if (act && a > 0.0 && b > 0.0 && g * g > tol2 * a * b) {
                    double cth, sth, tt;
                    rot_angle(a, b, g, cth, sth, tt);
#pragma unroll
                    for (int e = 0; e < EPL2; ++e) {
                        const double2 x = X[e], y = Yc[e];
                        X[e] = make_double2(cth * x.x - sth * y.x, cth * x.y - sth * y.y);
                        ycol[li + e * LPP] = make_double2(sth * x.x + cth * y.x, sth * x.y + cth * y.y);
                    }
                    if constexpr (TRACK) {
                        an = fma(-tt, g, a);
                        if (li == 0) nrm[yi] = fma(tt, g, b);
                    }
                    flags[fcur] = 1;
                }
                bar<NT>();
            }
            if (xlive) {
                double2* xw = reinterpret_cast<double2*>(Y + xi * JLD);
#pragma unroll
                for (int e = 0; e < EPL2; ++e) xw[li + e * LPP] = X[e];
                if (TRACK && li == 0) nrm[xi] = an;
            }
            bar<NT>();
        }
        const bool done = flags[fcur] == 0;
        bar<NT>();
        if (done) break;
    }
    if (threadIdx.x == 0) *sweeps_out = sweep + 1;
    __syncthreads();
}

template <int LPP, bool TRACK>
__global__ void __launch_bounds__(T, 3) kern(const double* in, double* out, int* sweeps, int q) {
    __shared__ __align__(16) double Y[Q * JLD];
    __shared__ double nrm[Q];
    __shared__ int flags[2];
    const double* src = in + (size_t)blockIdx.x * Q * Q;
    for (int i = threadIdx.x; i < Q * Q; i += T) Y[(i / Q) * JLD + i % Q] = src[i];
    __syncthreads();
    jacobi<LPP, TRACK>(Y, q, flags, nrm, sweeps + blockIdx.x);
    // column norms out
    for (int c = threadIdx.x; c < Q; c += T) {
        double a = 0;
        for (int r = 0; r < Q; ++r) a = fma(Y[c * JLD + r], Y[c * JLD + r], a);
        out[(size_t)blockIdx.x * Q + c] = sqrt(a);
    }
}


// Central-angle variant: 8 lanes per pair compute partial dot products of the
// RAW columns (g only; true norms are tracked), warp 0 (lane = pair) sums the
// partials, computes the rotation and the scaled-rotation coefficients, all
// lanes apply u' = u - alpha v, v' = v + beta u. Column scales s (true = s *
// raw) and 1/s are tracked; columns are renormalised at each sweep start.
__device__ void jacobi_central(double* Y, int q, int* flags, double* nrm, double* sc, double* isc,
                               double* part, double4* coef, int* sweeps_out) {
    constexpr int LPP = 8, EPL2 = 4;
    const double tol = (double)q * DBL_EPSILON, tol2 = tol * tol;
    const int slot = threadIdx.x / LPP, li = threadIdx.x % LPP, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) flags[0] = flags[1] = 0;
    __syncthreads();
    int sweep = 0;
    for (; sweep < 40; ++sweep) {
        const int fcur = sweep & 1;
        if (threadIdx.x == 0) flags[fcur ^ 1] = 0;
        // renormalise + fresh true norms
        for (int cc = slot; cc < Q; cc += 32) {
            double2* col = reinterpret_cast<double2*>(Y + cc * JLD);
            const double f = sweep ? sc[cc] : 1.0;
            double a = 0.0;
#pragma unroll
            for (int e = 0; e < EPL2; ++e) {
                double2 v = col[li + e * LPP];
                v.x *= f;
                v.y *= f;
                col[li + e * LPP] = v;
                a = fma(v.x, v.x, fma(v.y, v.y, a));
            }
#pragma unroll
            for (int o = 1; o < LPP; o <<= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (li == 0) {
                nrm[cc] = a;
                sc[cc] = 1.0;
                isc[cc] = 1.0;
            }
        }
        __syncthreads();
        for (int G = 32; G >= 1; G >>= 1) {
            const int grp = slot / G, ls = slot % G;
            const int xi = grp * 2 * G + ls;
            const bool xlive = xi < q;
            double2 X[EPL2], Yc[EPL2];
            const double2* xcol = reinterpret_cast<const double2*>(Y + xi * JLD);
#pragma unroll
            for (int e = 0; e < EPL2; ++e) X[e] = xlive ? xcol[li + e * LPP] : make_double2(0.0, 0.0);
            for (int r = 0; r < G; ++r) {
                const int yi = grp * 2 * G + G + ((ls + r) & (G - 1));
                const bool act = xlive && yi < q;
                double2* ycol = reinterpret_cast<double2*>(Y + yi * JLD);
#pragma unroll
                for (int e = 0; e < EPL2; ++e) Yc[e] = act ? ycol[li + e * LPP] : make_double2(0.0, 0.0);
                double g0 = 0.0, g1 = 0.0;
#pragma unroll
                for (int e = 0; e < EPL2; ++e) {
                    g0 = fma(X[e].x, Yc[e].x, g0);
                    g1 = fma(X[e].y, Yc[e].y, g1);
                }
                part[slot * 9 + li] = g0 + g1;
                __syncthreads();
                if (warp == 0) {
                    // lane = pair
                    const int p = lane;
                    const int pg = p / G, pls = p % G;
                    const int pxi = pg * 2 * G + pls, pyi = pg * 2 * G + G + ((pls + r) & (G - 1));
                    double4 cf = make_double4(0.0, 0.0, 0.0, 0.0);
                    if (pxi < q && pyi < q) {
                        const double* pp = part + p * 9;
                        const double graw = ((pp[0] + pp[1]) + (pp[2] + pp[3])) + ((pp[4] + pp[5]) + (pp[6] + pp[7]));
                        const double sx = sc[pxi], sy = sc[pyi], ix = isc[pxi], iy = isc[pyi];
                        const double a = nrm[pxi], b = nrm[pyi];
                        const double g = graw * (sx * sy);
                        if (a > 0.0 && b > 0.0 && g * g > tol2 * a * b) {
                            double cth, sth, tt;
                            rot_angle(a, b, g, cth, sth, tt);
                            cf.x = tt * (sy * ix);   // alpha
                            cf.y = tt * (sx * iy);   // beta
                            cf.z = 1.0;
                            const double ic = fma(tt, tt, 1.0) * cth;  // 1 / c
                            sc[pxi] = sx * cth;
                            sc[pyi] = sy * cth;
                            isc[pxi] = ix * ic;
                            isc[pyi] = iy * ic;
                            nrm[pxi] = fma(-tt, g, a);
                            nrm[pyi] = fma(tt, g, b);
                            flags[fcur] = 1;
                        }
                    }
                    coef[p] = cf;
                }
                __syncthreads();
                const double4 cf = coef[slot];
                if (cf.z != 0.0) {
#pragma unroll
                    for (int e = 0; e < EPL2; ++e) {
                        const double2 x = X[e], y = Yc[e];
                        X[e] = make_double2(fma(-cf.x, y.x, x.x), fma(-cf.x, y.y, x.y));
                        ycol[li + e * LPP] = make_double2(fma(cf.y, x.x, y.x), fma(cf.y, x.y, y.y));
                    }
                }
                __syncthreads();
            }
            if (xlive) {
                double2* xw = reinterpret_cast<double2*>(Y + xi * JLD);
#pragma unroll
                for (int e = 0; e < EPL2; ++e) xw[li + e * LPP] = X[e];
            }
            __syncthreads();
        }
        const bool done = flags[fcur] == 0;
        __syncthreads();
        if (done) break;
    }
    // final renormalisation
    for (int cc = slot; cc < Q; cc += 32) {
        double2* col = reinterpret_cast<double2*>(Y + cc * JLD);
        const double f = sc[cc];
#pragma unroll
        for (int e = 0; e < EPL2; ++e) {
            double2 v = col[li + e * LPP];
            v.x *= f;
            v.y *= f;
            col[li + e * LPP] = v;
        }
    }
    if (threadIdx.x == 0) *sweeps_out = sweep + 1;
    __syncthreads();
}

__global__ void __launch_bounds__(T, 3) kern_central(const double* in, double* out, int* sweeps, int q) {
    __shared__ __align__(16) double Y[Q * JLD];
    __shared__ double nrm[Q], sc[Q], isc[Q], part[32 * 9];
    __shared__ double4 coef[32];
    __shared__ int flags[2];
    const double* src = in + (size_t)blockIdx.x * Q * Q;
    for (int i = threadIdx.x; i < Q * Q; i += T) Y[(i / Q) * JLD + i % Q] = src[i];
    __syncthreads();
    jacobi_central(Y, q, flags, nrm, sc, isc, part, coef, sweeps + blockIdx.x);
    for (int c = threadIdx.x; c < Q; c += T) {
        double a = 0;
        for (int r = 0; r < Q; ++r) a = fma(Y[c * JLD + r], Y[c * JLD + r], a);
        out[(size_t)blockIdx.x * Q + c] = sqrt(a);
    }
}


__device__ long long g_stage[8];
__global__ void __launch_bounds__(T, 3) kern_inst(const double* in, double* out, int* sweeps, int q) {
    __shared__ __align__(16) double Y[Q * JLD];
    __shared__ double nrm[Q];
    __shared__ int flags[2];
    const double* src = in + (size_t)blockIdx.x * Q * Q;
    for (int i = threadIdx.x; i < Q * Q; i += T) Y[(i / Q) * JLD + i % Q] = src[i];
    __syncthreads();
    constexpr int LPP = 8, EPL2 = 4;
    const double tol = (double)q * DBL_EPSILON, tol2 = tol * tol;
    long long st[6] = {0, 0, 0, 0, 0, 0};
    if (threadIdx.x == 0) flags[0] = flags[1] = 0;
    __syncthreads();
    const int slot = threadIdx.x / LPP, li = threadIdx.x % LPP;
    for (int sweep = 0; sweep < 40; ++sweep) {
        const int fcur = sweep & 1;
        if (threadIdx.x == 0) flags[fcur ^ 1] = 0;
        for (int cc = slot; cc < Q; cc += 32) {
            const double2* col = reinterpret_cast<const double2*>(Y + cc * JLD);
            double a = 0.0;
            for (int e = 0; e < EPL2; ++e) { const double2 v = col[li + e * LPP]; a = fma(v.x, v.x, fma(v.y, v.y, a)); }
            for (int o = 1; o < LPP; o <<= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (li == 0) nrm[cc] = a;
        }
        __syncthreads();
        for (int G = 32; G >= 1; G >>= 1) {
            const int grp = slot / G, ls = slot % G;
            const int xi = grp * 2 * G + ls;
            double2 X[EPL2], Yc[EPL2];
            const double2* xcol = reinterpret_cast<const double2*>(Y + xi * JLD);
            for (int e = 0; e < EPL2; ++e) X[e] = xcol[li + e * LPP];
            double an = nrm[xi];
            for (int r = 0; r < G; ++r) {
                long long t0 = clock64();
                const int yi = grp * 2 * G + G + ((ls + r) & (G - 1));
                double2* ycol = reinterpret_cast<double2*>(Y + yi * JLD);
#pragma unroll
                for (int e = 0; e < EPL2; ++e) Yc[e] = ycol[li + e * LPP];
                const double b = nrm[yi];
                double g0 = 0.0, g1 = 0.0;
#pragma unroll
                for (int e = 0; e < EPL2; ++e) { g0 = fma(X[e].x, Yc[e].x, g0); g1 = fma(X[e].y, Yc[e].y, g1); }
                double g = g0 + g1;
                long long t1 = clock64();
#pragma unroll
                for (int o = 1; o < LPP; o <<= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
                long long t2 = clock64();
                const double a = an;
                if (a > 0.0 && b > 0.0 && g * g > tol2 * a * b) {
                    double cth, sth, tt;
                    rot_angle(a, b, g, cth, sth, tt);
                    long long t3 = clock64();
#pragma unroll
                    for (int e = 0; e < EPL2; ++e) {
                        const double2 x = X[e], y = Yc[e];
                        X[e] = make_double2(cth * x.x - sth * y.x, cth * x.y - sth * y.y);
                        ycol[li + e * LPP] = make_double2(sth * x.x + cth * y.x, sth * x.y + cth * y.y);
                    }
                    an = fma(-tt, g, a);
                    if (li == 0) nrm[yi] = fma(tt, g, b);
                    flags[fcur] = 1;
                    long long t4 = clock64();
                    st[2] += t3 - t2; st[3] += t4 - t3;
                }
                long long t5 = clock64();
                __syncthreads();
                long long t6 = clock64();
                st[0] += t1 - t0; st[1] += t2 - t1; st[4] += t6 - t5; st[5] += t6 - t0;
            }
            for (int e = 0; e < EPL2; ++e) reinterpret_cast<double2*>(Y + xi * JLD)[li + e * LPP] = X[e];
            if (li == 0) nrm[xi] = an;
            __syncthreads();
        }
        const bool done = flags[fcur] == 0;
        __syncthreads();
        if (done) { if (threadIdx.x == 0) sweeps[blockIdx.x] = sweep + 1; break; }
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) for (int i = 0; i < 6; ++i) g_stage[i] = st[i];
    for (int c = threadIdx.x; c < Q; c += T) { double a = 0; for (int r = 0; r < Q; ++r) a = fma(Y[c * JLD + r], Y[c * JLD + r], a); out[(size_t)blockIdx.x * Q + c] = sqrt(a); }
}

template <class K>
void run_k(K kfn, const char* name, const double* d_in, double* d_out, int* d_sw, int nmat) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int ns[] = {1, 148, 296, 444, 500};
    std::printf("%-16s", name);
    for (int n : ns) {
        if (n > nmat) continue;
        kfn<<<n, T>>>(d_in, d_out, d_sw, Q);
        cudaEventRecord(e0);
        for (int it = 0; it < 5; ++it) kfn<<<n, T>>>(d_in, d_out, d_sw, Q);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        std::printf("  n=%d %.1fus", n, ms * 1e3 / 5);
    }
    std::vector<int> sw(nmat);
    std::vector<double> o((size_t)nmat * Q);
    cudaMemcpy(sw.data(), d_sw, 4 * nmat, cudaMemcpyDeviceToHost);
    cudaMemcpy(o.data(), d_out, 8 * o.size(), cudaMemcpyDeviceToHost);
    double sm = 0;
    for (int i = 0; i < nmat; ++i) sm += sw[i];
    // sum of sorted sigma of matrix 0 (checksum across variants)
    std::vector<double> s0(o.begin(), o.begin() + Q);
    std::sort(s0.begin(), s0.end());
    std::printf("  | sweeps avg %.2f  sigma0 max %.15e min %.15e\n", sm / nmat, s0.back(), s0.front());
}

#include <algorithm>
int main() {
    const int nmat = 500;
    std::mt19937_64 rng(1);
    std::normal_distribution<double> nd;
    std::vector<double> h((size_t)nmat * Q * Q);
    // R^T of (2000 x 64 gaussian with graded columns): emulate with a random
    // triangular-ish dense matrix with graded column scales
    for (int m = 0; m < nmat; ++m)
        for (int c = 0; c < Q; ++c)
            for (int r = 0; r < Q; ++r)
                h[(size_t)m * Q * Q + c * Q + r] = (r <= c ? nd(rng) : 0.0) * std::pow(10.0, -3.0 * r / Q) * 40.0;
    double *d_in, *d_out;
    int* d_sw;
    cudaMalloc(&d_in, 8 * h.size());
    cudaMalloc(&d_out, 8 * (size_t)nmat * Q);
    cudaMalloc(&d_sw, 4 * nmat);
    cudaMemcpy(d_in, h.data(), 8 * h.size(), cudaMemcpyHostToDevice);
    kern_inst<<<1, T>>>(d_in, d_out, d_sw, Q);
    cudaDeviceSynchronize();
    long long hs[8];
    cudaMemcpyFromSymbol(hs, g_stage, sizeof(hs));
    int sw; cudaMemcpy(&sw, d_sw, 4, cudaMemcpyDeviceToHost);
    double rounds = sw * 63.0;
    std::printf("inst single CTA: sweeps %d, cycles/round: load+dots %.0f shfl %.0f angle %.0f rot+store %.0f barrier %.0f total %.0f\n", sw,
                hs[0] / rounds, hs[1] / rounds, hs[2] / rounds, hs[3] / rounds, hs[4] / rounds, hs[5] / rounds);
    run_k(kern<8, false>, "lpp8", d_in, d_out, d_sw, nmat);
    run_k(kern<8, true>, "lpp8 track", d_in, d_out, d_sw, nmat);
    run_k(kern_central, "central", d_in, d_out, d_sw, nmat);
    cudaError_t e = cudaDeviceSynchronize();
    std::printf("%s\n", cudaGetErrorString(e));
    return 0;
}
