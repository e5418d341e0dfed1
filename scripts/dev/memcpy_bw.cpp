// Dev: host memcpy bandwidth with the copy pool (host_pool.h), pageable -> pageable.
#include "../../paper_1805_00754_b200/csrc/host_pool.h"
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>
int main() {
    const size_t n = 64 << 20;  // doubles: 512 MB
    std::vector<double> src(n, 1.0), dst(n, 0.0);
    auto& pool = zsvd::CopyPool::get();
    for (int parts : {1, 2, 4, 8, 12, 16, 24}) {
        double best = 0;
        for (int rep = 0; rep < 3; ++rep) {
            auto t0 = std::chrono::steady_clock::now();
            for (size_t off = 0; off < n; off += (4 << 20)) {  // 32 MB chunks
                const size_t m = std::min<size_t>(4 << 20, n - off);
                pool.run(parts, [&](int p) {
                    size_t a = m * p / parts, e = m * (p + 1) / parts;
                    std::memcpy(dst.data() + off + a, src.data() + off + a, (e - a) * 8);
                });
            }
            double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            best = std::max(best, n * 8 / s / 1e9);
        }
        std::printf("parts %2d: %.1f GB/s\n", parts, best);
    }
}
