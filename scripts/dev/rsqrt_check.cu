// Max relative error of the inline rsqrt variants against 1/sqrt(x) in fp64 (dev tool).
#include <cstdio>
#include <cmath>
__device__ __forceinline__ double seed(double x) { double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y; }
__device__ double nr2(double x) { double y = seed(x); const double h = 0.5 * x; y = y * fma(-h * y, y, 1.5); y = y * fma(-h * y, y, 1.5); return y; }
__device__ double cub(double x) { double y = seed(x); const double e = fma(-x * y, y, 1.0); return fma(y * e, fma(0.375, e, 0.5), y); }
__global__ void k(double* out, int n) {
    double m0 = 0, m1 = 0, m2 = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double x = (i % 3 == 0) ? 1.0 + (double)i / n : ldexp(1.0 + (double)(i * 7919 % n) / n, (i % 200) - 100);
        double r = 1.0 / sqrt(x);
        m0 = fmax(m0, fabs(seed(x) - r) / r);
        m1 = fmax(m1, fabs(nr2(x) - r) / r);
        m2 = fmax(m2, fabs(cub(x) - r) / r);
    }
    atomicMax((unsigned long long*)&out[0], __double_as_longlong(m0));
    atomicMax((unsigned long long*)&out[1], __double_as_longlong(m1));
    atomicMax((unsigned long long*)&out[2], __double_as_longlong(m2));
}
int main() {
    double* d; cudaMalloc(&d, 24); cudaMemset(d, 0, 24);
    k<<<1184, 256>>>(d, 1 << 26);
    double h[3]; cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("seed rel err %.3e (2^%.1f), two Newton %.3e, cubic %.3e (eps %.3e)\n", h[0], log2(h[0]), h[1], h[2], 2.2204e-16);
}
