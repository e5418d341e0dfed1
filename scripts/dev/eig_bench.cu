// Dev harness: times eig::jacobi_eig (sym_eig.cuh) on Gram matrices from files
// (scripts/dev/eig_data/*.bin: int32 n, then n*n doubles) and writes the
// eigenvalues / vectors for scripts/dev/eig_check.py.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <string>
#include <cuda_runtime.h>
#include "../../paper_1805_00754_b200/csrc/sym_eig.cuh"
using namespace zsvd;

template <int N>
__global__ void __launch_bounds__(eig::Shared<N>::NT) kern(const double* A, int n, double scale, double tol, double tabs,
                                                           double* lam, double* V, long long* clk, int* sweeps) {
    extern __shared__ __align__(16) char buf[];
    auto& S = *reinterpret_cast<eig::Shared<N>*>(buf);
    long long t0 = clock64();
    eig::jacobi_eig<N>(A, n, n, scale, S, tol, tabs, 40);
    long long t1 = clock64();
    for (int i = threadIdx.x; i < n; i += blockDim.x) lam[i] = S.lam[i] / scale;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) V[e] = S.V[(e / n) * N + e % n];
    if (threadIdx.x == 0) { clk[0] = t1 - t0; sweeps[0] = S.sweeps; }
}

template <int N>
void run(const std::vector<double>& A, int n, const char* out, double tol, double tabs) {
    double *dA, *dl, *dV; long long* dc; int* ds;
    cudaMalloc(&dA, n * n * 8); cudaMalloc(&dl, n * 8); cudaMalloc(&dV, n * n * 8);
    cudaMalloc(&dc, 8); cudaMalloc(&ds, 4);
    cudaMemcpy(dA, A.data(), n * n * 8, cudaMemcpyHostToDevice);
    double dmax = 0; for (int i = 0; i < n; ++i) dmax = std::max(dmax, A[i * n + i]);
    int e2; std::frexp(dmax, &e2); double scale = std::ldexp(1.0, -e2);
    size_t smem = sizeof(eig::Shared<N>);
    cudaFuncSetAttribute(kern<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e9; long long clk = 0; int sw = 0;
    for (int it = 0; it < 5; ++it) {
        cudaEventRecord(a);
        kern<N><<<1, eig::Shared<N>::NT, smem>>>(dA, n, scale, tol, tabs, dl, dV, dc, ds);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { std::printf("CUDA error %s\n", cudaGetErrorString(e)); std::exit(1); }
    cudaMemcpy(&clk, dc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&sw, ds, 4, cudaMemcpyDeviceToHost);
    std::vector<double> lam(n), V(n * n);
    cudaMemcpy(lam.data(), dl, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(V.data(), dV, n * n * 8, cudaMemcpyDeviceToHost);
    FILE* f = std::fopen(out, "wb"); std::fwrite(&n, 4, 1, f); std::fwrite(lam.data(), 8, n, f);
    std::fwrite(V.data(), 8, n * n, f); std::fclose(f);
    std::printf("%s n=%d N=%d sweeps=%d cycles=%lld (%.0f per round) kernel %.1f us smem %zu\n", out, n, N, sw, clk,
                (double)clk / std::max(1, sw * (N - 1)), best * 1e3, smem);
}

int main(int argc, char** argv) {
    double tol = argc > 3 ? std::atof(argv[3]) : 1e-15, tabs = argc > 4 ? std::atof(argv[4]) : 8 * 2.220446049250313e-16;
    FILE* f = std::fopen(argv[1], "rb");
    int n; std::fread(&n, 4, 1, f);
    std::vector<double> A(n * n); std::fread(A.data(), 8, n * n, f); std::fclose(f);
    if (n <= 16) run<16>(A, n, argv[2], tol, tabs);
    else if (n <= 32) run<32>(A, n, argv[2], tol, tabs);
    else run<64>(A, n, argv[2], tol, tabs);
    return 0;
}
