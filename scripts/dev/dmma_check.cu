// Verifies the mma.m8n8k4 f64 fragment layout assumed by svd_engine.cu.
#include <cstdio>
#include <cmath>
__global__ void k(const double* A, const double* B, double* C) {
    int lane = threadIdx.x;
    double a = A[(lane >> 2) * 4 + (lane & 3)];      // A 8x4 row-major
    double b = B[(lane & 3) * 8 + (lane >> 2)];      // B 4x8 row-major storage, frag (k=lane&3, n=lane>>2)
    double c0 = 0, c1 = 0;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    C[(lane >> 2) * 8 + (lane & 3) * 2] = c0;
    C[(lane >> 2) * 8 + (lane & 3) * 2 + 1] = c1;
}
int main() {
    double hA[32], hB[32], hC[64], ref[64];
    for (int i = 0; i < 32; ++i) { hA[i] = i * 0.5 - 3; hB[i] = (i * 7 % 11) - 4.0; }
    for (int m = 0; m < 8; ++m) for (int n = 0; n < 8; ++n) { double s = 0; for (int kk = 0; kk < 4; ++kk) s += hA[m*4+kk] * hB[kk*8+n]; ref[m*8+n] = s; }
    double *A, *B, *C; cudaMalloc(&A, 256); cudaMalloc(&B, 256); cudaMalloc(&C, 512);
    cudaMemcpy(A, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(A, B, C); cudaMemcpy(hC, C, 512, cudaMemcpyDeviceToHost);
    double err = 0; for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hC[i] - ref[i]));
    printf("dmma layout max err %g %s\n", err, err < 1e-12 ? "OK" : "MISMATCH");
    return err < 1e-12 ? 0 : 1;
}
