// Dev micro-benchmark: ways to get file bytes (page cache) into HBM.
// (a) pread with T threads into pinned memory, then H2D; (b) mmap + cudaHostRegister(ReadOnly) + H2D.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main(int argc, char** argv) {
  const char* path = argv[1];
  int fd = open(path, O_RDONLY); struct stat st; fstat(fd, &st); size_t size = st.st_size;
  const size_t CH = 32ull << 20;
  char* pin; cudaHostAlloc((void**)&pin, CH, 0);
  void* dbuf; cudaMalloc(&dbuf, CH);
  cudaStream_t s; cudaStreamCreate(&s);
  for (int T : {1, 4, 8, 12, 16}) {
    double t0 = now();
    for (size_t off = 0; off < size; off += CH) {
      size_t len = std::min(CH, size - off);
      std::vector<std::thread> th;
      size_t part = (len + T - 1) / T;
      for (int i = 0; i < T; ++i) { size_t b = i * part, e = std::min(len, b + part); if (b >= e) break;
        th.emplace_back([&, b, e] { size_t g = 0; while (g < e - b) { ssize_t r = pread(fd, pin + b + g, e - b - g, off + b + g); if (r <= 0) break; g += r; } }); }
      for (auto& t : th) t.join();
    }
    double t1 = now();
    printf("pread T=%2d: %.2f GB/s\n", T, size / (t1 - t0) / 1e9);
  }
  { double t0 = now();
    for (size_t off = 0; off < size; off += CH) { size_t len = std::min(CH, size - off); cudaMemcpyAsync(dbuf, pin, len, cudaMemcpyHostToDevice, s); }
    cudaStreamSynchronize(s); double t1 = now(); printf("H2D pinned: %.2f GB/s\n", size / (t1 - t0) / 1e9); }
  char* map = (char*)mmap(nullptr, size, PROT_READ, MAP_SHARED, fd, 0);
  if (map == MAP_FAILED) { printf("mmap failed\n"); return 0; }
  for (int rep = 0; rep < 2; ++rep) {
    double treg = 0, t0 = now();
    for (size_t off = 0; off < size; off += CH) {
      size_t len = std::min(CH, size - off);
      double a = now();
      cudaError_t e = cudaHostRegister(map + off, len, cudaHostRegisterReadOnly);
      treg += now() - a;
      if (e != cudaSuccess) { printf("register failed: %s\n", cudaGetErrorString(e)); return 0; }
      cudaMemcpyAsync(dbuf, map + off, len, cudaMemcpyHostToDevice, s);
      cudaStreamSynchronize(s);
      cudaHostUnregister(map + off);
    }
    double t1 = now();
    printf("mmap+register+H2D (serial): %.2f GB/s (register %.1f ms of %.1f ms)\n", size / (t1 - t0) / 1e9, treg * 1e3, (t1 - t0) * 1e3);
  }
  { double t0 = now(); cudaError_t e = cudaHostRegister(map, size, cudaHostRegisterReadOnly); double t1 = now();
    printf("register whole file: %s %.1f ms\n", cudaGetErrorString(e), (t1 - t0) * 1e3);
    double t2 = now();
    for (size_t off = 0; off < size; off += CH) { size_t len = std::min(CH, size - off); cudaMemcpyAsync(dbuf, map + off, len, cudaMemcpyHostToDevice, s); }
    cudaStreamSynchronize(s); double t3 = now(); printf("H2D from registered mmap: %.2f GB/s\n", size / (t3 - t2) / 1e9);
    cudaHostUnregister(map); }
  // memcpy from mmap with threads (page cache -> pinned) for comparison
  for (int T : {8, 16}) {
    double t0 = now();
    for (size_t off = 0; off < size; off += CH) {
      size_t len = std::min(CH, size - off); size_t part = (len + T - 1) / T; std::vector<std::thread> th;
      for (int i = 0; i < T; ++i) { size_t b = i * part, e = std::min(len, b + part); if (b >= e) break; th.emplace_back([&, b, e] { memcpy(pin + b, map + off + b, e - b); }); }
      for (auto& t : th) t.join();
    }
    double t1 = now(); printf("memcpy from mmap T=%d: %.2f GB/s\n", T, size / (t1 - t0) / 1e9);
  }
  return 0;
}
