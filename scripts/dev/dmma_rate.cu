// fp64 MMA throughput per SM for the m8n8k4 and m16n8k{4,8,16} shapes. Dev tool.
#include <cstdio>
template <int SHAPE>
__global__ void k(double* out, long long* cyc, int iters) {
    double a[8], b[4], c[8][4];
    for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (threadIdx.x + i);
    for (int i = 0; i < 4; ++i) b[i] = 1e-3 * (threadIdx.x - i);
    for (int j = 0; j < 8; ++j) for (int i = 0; i < 4; ++i) c[j][i] = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (SHAPE == 0)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a[0]), "d"(b[0]));
            else if (SHAPE == 1)
                asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                             : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
            else if (SHAPE == 2)
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
            else
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                             : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    double s = 0;
    for (int j = 0; j < 8; ++j) for (int i = 0; i < 4; ++i) s += c[j][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    double* o; long long* c;
    cudaMalloc(&o, 8 << 20); cudaMalloc(&c, 8 * 4096);
    const int fmas[] = {8 * 8 * 4, 16 * 8 * 4, 16 * 8 * 8, 16 * 8 * 16};
    const char* nm[] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
    for (int sh = 0; sh < 4; ++sh)
        for (int warps : {4, 8, 16, 32}) {
            const int iters = 2000;
            auto launch = [&]() {
                if (sh == 0) k<0><<<148, 32 * warps>>>(o, c, iters);
                if (sh == 1) k<1><<<148, 32 * warps>>>(o, c, iters);
                if (sh == 2) k<2><<<148, 32 * warps>>>(o, c, iters);
                if (sh == 3) k<3><<<148, 32 * warps>>>(o, c, iters);
            };
            launch();
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
            double f = (double)fmas[sh] * 8 * iters * warps;
            printf("%-9s warps/SM %2d: %.1f FMA/clk/SM (clock64), %.1f TFLOP/s (events)\n", nm[sh], warps, f / cy,
                   2.0 * f * 148 / (ms * 1e-3) / 1e12);
        }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
