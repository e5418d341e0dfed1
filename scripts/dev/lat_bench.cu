// Dependent-chain latencies (cycles per op) of the fp64 operations on the
// Jacobi critical path, single warp. Dev tool.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double x0) {
    double x = x0 + threadIdx.x * 1e-9, y = 1.0000001;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) x = fma(x, y, 1e-300);
    t1 = clock64();
    cyc[0] = (t1 - t0);
    // DADD chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) x = x + 1e-300;
    t1 = clock64();
    cyc[1] = (t1 - t0);
    // shfl + dadd chain (64-bit shuffle)
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
    t1 = clock64();
    cyc[2] = (t1 - t0);
    // rsqrt.approx.f64 chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) {
        double r;
        asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
        x = r + 1.0;
    }
    t1 = clock64();
    cyc[3] = (t1 - t0);
    // full rsqrt chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) x = rsqrt(x) + 1.0;
    t1 = clock64();
    cyc[4] = (t1 - t0);
    // empty loop
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) asm volatile("");
    t1 = clock64();
    cyc[5] = (t1 - t0);
    // __syncthreads loop (256 threads)
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) __syncthreads();
    t1 = clock64();
    cyc[6] = (t1 - t0);
    // DFMA throughput: 8 independent chains, all warps
    double a0 = x, a1 = x + 1, a2 = x + 2, a3 = x + 3, a4 = x + 4, a5 = x + 5, a6 = x + 6, a7 = x + 7;
    __syncthreads();
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) {
        a0 = fma(a0, y, 1e-300); a1 = fma(a1, y, 1e-300); a2 = fma(a2, y, 1e-300); a3 = fma(a3, y, 1e-300);
        a4 = fma(a4, y, 1e-300); a5 = fma(a5, y, 1e-300); a6 = fma(a6, y, 1e-300); a7 = fma(a7, y, 1e-300);
    }
    __syncthreads();
    t1 = clock64();
    cyc[7] = (t1 - t0);
    out[threadIdx.x] = x + a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
int main() {
    double* o; long long* c;
    cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8 * 16);
    const char* nm[] = {"dfma", "dadd", "shfl64+dadd", "rsqrt.approx", "rsqrt full+add", "loop", "syncthreads(256)", "dfma thr (8 chains, 8 warps/SM) per iter"};
    for (int nt : {32, 256, 1024}) {
        k<<<1, nt>>>(o, c, 1.0);
        long long h[8];
        cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
        printf("threads %d\n", nt);
        for (int i = 0; i < 8; ++i) printf("  %-44s %.1f cycles\n", nm[i], h[i] / 1024.0);
    }
    return 0;
}
