// sturm_probe.cu — dev tool: cycles per Sturm count (n = 64, the eigensolver's
// three-term recurrence) as a function of the number of warps counting at once
// and of how many independent counts each lane interleaves.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sturm_probe sturm_probe.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ double renorm_factor(double a, double b) {
    const int ea = (__double2hiint(a) >> 20) & 0x7ff, eb = (__double2hiint(b) >> 20) & 0x7ff;
    const int e = ea > eb ? ea : eb;
    return e == 0 ? 1.0 : __hiloint2double((2046 - e) << 20, 0);
}

template <int ILP>
__global__ void sturm(const double* dg, const double* eg, int n, int active_warps, int reps, long long* out, int* sink) {
    __shared__ double d[64], ee[64];
    const int tid = threadIdx.x;
    if (tid < 64) {
        d[tid] = dg[tid];
        ee[tid] = eg[tid] * eg[tid];
    }
    __syncthreads();
    if ((tid >> 5) >= active_warps) return;
    double x[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = 0.01 * (tid + 1) + 0.37 * k;
    int total = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        double pa[ILP], pb[ILP];
        int sg[ILP], cn[ILP];
#pragma unroll
        for (int k = 0; k < ILP; ++k) {
            pa[k] = 1.0;
            pb[k] = d[0] - x[k];
            sg[k] = __double2hiint(pb[k]) >> 31;
            cn[k] = sg[k];
        }
        for (int i = 1; i + 8 <= n; i += 8) {
            double dd[8], e2[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                dd[u] = d[i + u];
                e2[u] = ee[i + u - 1];
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
#pragma unroll
                for (int k = 0; k < ILP; ++k) {
                    const double q = fma(dd[u] - x[k], pb[k], -e2[u] * pa[k]);
                    const int s2 = __double2hiint(q) >> 31;
                    cn[k] += s2 ^ sg[k];
                    sg[k] = s2;
                    pa[k] = pb[k];
                    pb[k] = q;
                }
            }
#pragma unroll
            for (int k = 0; k < ILP; ++k) {
                const double f = renorm_factor(pa[k], pb[k]);
                pa[k] *= f;
                pb[k] *= f;
            }
        }
#pragma unroll
        for (int k = 0; k < ILP; ++k) {
            total += cn[k];
            x[k] += 1e-3 * cn[k];
        }
    }
    long long t1 = clock64();
    if (tid == 0) out[0] = (t1 - t0) / reps;
    sink[tid] = total;
}

// fp32 variant of the same recurrence (one count per lane)
__global__ void sturm32(const double* dg, const double* eg, int n, int active_warps, int reps, long long* out, int* sink) {
    __shared__ float d[64], ee[64];
    const int tid = threadIdx.x;
    if (tid < 64) {
        d[tid] = (float)dg[tid];
        ee[tid] = (float)(eg[tid] * eg[tid]);
    }
    __syncthreads();
    if ((tid >> 5) >= active_warps) return;
    float x = 0.01f * (tid + 1);
    int total = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        float q = d[0] - x;
        int cn = __float_as_int(q) >> 31;
        for (int i = 1; i < n; ++i) {
            q = (d[i] - x) - ee[i - 1] / q;  // divisions: the classic form
            cn += __float_as_int(q) >> 31;
        }
        total += cn;
        x += 1e-3f * cn;
    }
    long long t1 = clock64();
    if (tid == 0) out[0] = (t1 - t0) / reps;
    sink[tid] = total;
}

int main() {
    double hd[64], he[64];
    for (int i = 0; i < 64; ++i) {
        hd[i] = 1.0 + 0.3 * ((i * 37) % 11);
        he[i] = 0.2 + 0.01 * i;
    }
    double *dd, *de;
    long long* out;
    int* sink;
    cudaMalloc(&dd, 512);
    cudaMalloc(&de, 512);
    cudaMalloc(&out, 64);
    cudaMalloc(&sink, 1 << 16);
    cudaMemcpy(dd, hd, 512, cudaMemcpyHostToDevice);
    cudaMemcpy(de, he, 512, cudaMemcpyHostToDevice);
    long long h;
    for (int w : {1, 2, 4, 7, 8, 16}) {
        std::printf("warps %2d:", w);
        sturm<1><<<1, 512>>>(dd, de, 64, w, 20, out, sink);
        sturm<1><<<1, 512>>>(dd, de, 64, w, 20, out, sink);
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        std::printf("  ilp1 %5lld cyc/iter", h);
        sturm<2><<<1, 512>>>(dd, de, 64, w, 20, out, sink);
        sturm<2><<<1, 512>>>(dd, de, 64, w, 20, out, sink);
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        std::printf("  ilp2 %5lld", h);
        sturm<4><<<1, 512>>>(dd, de, 64, w, 20, out, sink);
        sturm<4><<<1, 512>>>(dd, de, 64, w, 20, out, sink);
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        std::printf("  ilp4 %5lld", h);
        sturm32<<<1, 512>>>(dd, de, 64, w, 20, out, sink);
        sturm32<<<1, 512>>>(dd, de, 64, w, 20, out, sink);
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        std::printf("  fp32div %5lld\n", h);
    }
    std::printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
