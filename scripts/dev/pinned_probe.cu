// Dev: pinned host allocations on this platform: host writes (main and other
// threads) and H2D copies, by size and allocation call.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <thread>
int main() {
    double* d = nullptr;
    cudaMalloc(&d, 64 << 20);
    const size_t sizes[] = {1 << 20, 1024000, 4 << 20, 32 << 20};
    for (size_t sz : sizes) {
        for (int how = 0; how < 3; ++how) {
            void* h = nullptr;
            cudaError_t e = how == 0 ? cudaMallocHost(&h, sz) : how == 1 ? cudaHostAlloc(&h, sz, cudaHostAllocPortable)
                                                                         : cudaHostAlloc(&h, sz, cudaHostAllocDefault);
            std::printf("size %zu how %d alloc %d ptr %p\n", sz, how, (int)e, h);
            std::fflush(stdout);
            std::memset(h, 1, sz);
            std::printf("  main memset ok\n");
            std::fflush(stdout);
            std::thread t([&] { std::memset(h, 2, sz); });
            t.join();
            std::printf("  thread memset ok\n");
            std::fflush(stdout);
            e = cudaMemcpy(d, h, sz, cudaMemcpyHostToDevice);
            std::printf("  h2d %d\n", (int)e);
            std::fflush(stdout);
            cudaFreeHost(h);
        }
    }
}
