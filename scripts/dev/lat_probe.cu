// lat_probe.cu — dev tool: latency of the operations the eigensolver's
// sequential chains are made of (dependent DFMA, DADD, MUFU rcp f64, double
// shuffle, shared load, CTA barrier at 128/256/512 threads), in SM cycles.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_probe lat_probe.cu
#include <cstdio>
#include <cstdint>

__global__ void chains(double x0, long long* out, double* sink) {
    __shared__ double sm[1024];
    const int tid = threadIdx.x;
    sm[tid] = x0 + tid;
    __syncthreads();
    double x = x0;
    long long t0, t1;
    constexpr int N = 256;
    // dependent DFMA
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = fma(x, 0.999999, 1e-9);
    t1 = clock64();
    if (tid == 0) out[0] = (t1 - t0) / N;
    // dependent DADD
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = x + 1e-9;
    t1 = clock64();
    if (tid == 0) out[1] = (t1 - t0) / N;
    // dependent rcp.approx f64
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) {
        double y;
        asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
        x = y;
    }
    t1 = clock64();
    if (tid == 0) out[2] = (t1 - t0) / N;
    // dependent double shuffle
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1);
    t1 = clock64();
    if (tid == 0) out[3] = (t1 - t0) / N;
    // dependent shared load (pointer chase through an index)
    int idx = tid & 7;
    for (int i = 0; i < 8; ++i) ((int*)(sm + 512))[i] = (i + 1) & 7;
    __syncthreads();
    const int* nx = (const int*)(sm + 512);
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) idx = nx[idx];
    t1 = clock64();
    if (tid == 0) out[4] = (t1 - t0) / N;
    // CTA barrier
    __syncthreads();
    t0 = clock64();
    for (int i = 0; i < N; ++i) __syncthreads();
    t1 = clock64();
    if (tid == 0) out[5] = (t1 - t0) / N;
    // barrier + shared write/read round trip (the handoff between warps)
    t0 = clock64();
    double v = x;
    for (int i = 0; i < N; ++i) {
        if (tid == (i & 31)) sm[0] = v;
        __syncthreads();
        v = sm[0] * 1.0000001;
        __syncthreads();
    }
    t1 = clock64();
    if (tid == 0) out[6] = (t1 - t0) / N;
    // throughput: independent DFMA, 8 chains per thread
    double a[8];
    for (int u = 0; u < 8; ++u) a[u] = x + u;
    t0 = clock64();
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] = fma(a[u], 0.999999, 1e-9);
    t1 = clock64();
    if (tid == 0) out[7] = (t1 - t0);  // cycles for N*8 DFMA per thread
    double s = 0;
    for (int u = 0; u < 8; ++u) s += a[u];
    sink[blockIdx.x * blockDim.x + tid] = x + s + idx + v;
}

int main() {
    long long* d;
    double* sink;
    cudaMalloc(&d, 64);
    cudaMalloc(&sink, 1 << 20);
    for (int th : {32, 128, 256, 512, 1024}) {
        chains<<<1, th>>>(1.0, d, sink);
        chains<<<1, th>>>(1.0, d, sink);
        long long h[8];
        cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
        std::printf("threads %4d: dfma %lld dadd %lld rcp64 %lld shfl64 %lld lds %lld bar %lld bar+handoff %lld | dfma tput %.2f warp-instr/clk/SM\n",
                    th, h[0], h[1], h[2], h[3], h[4], h[5], h[6], (double)(th / 32) * 256 * 8 / (double)h[7]);
    }
    cudaError_t e = cudaDeviceSynchronize();
    std::printf("%s\n", cudaGetErrorString(e));
    return 0;
}
