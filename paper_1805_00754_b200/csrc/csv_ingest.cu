// csv_ingest.cu — CSV ingestion on the device.
//
// The reference reads CSV text row by row on the host (CsvReader::next,
// csv.hpp:79-132: std::getline, split on ',', trim, std::from_chars per cell)
// and appends each row to the store (cmd_ingest, commands.hpp:106-139).  Here
// the host only moves bytes: the file is read in chunks that end at a line
// break (parallel pread into a ring of pinned buffers) and copied to HBM on a
// copy stream while the previous chunk is processed.  Everything that looks
// at a byte runs on the device, per chunk:
//   csv_count_kernel     newlines per 32 KB tile (4-byte SIMD compares)
//   csv_lines_kernel     line ends (block scan, prefix over earlier tiles)
//   csv_classify_kernel  blank lines (csv.hpp:83-85)
//   csv_rowidx_kernel    data-row index per line (only when a chunk skips lines)
//   csv_parse_kernel     one warp per line: commas by 16-byte vector loads and a
//                        warp scan, each cell converted by the lane that owns its
//                        first byte (csv_number.cuh, bit-exact with from_chars),
//                        written to the row-major output; per-line errors
//   csv_line_info_kernel the header test, the first data row and the error
//                        line's details (one line, one thread; a few per file)
// The result is a device matrix the store appends without another copy.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/zsvd.h"
#include "csv_number.cuh"
#include "zsvd_internal.h"

namespace zsvd {
namespace {
#include "pow5_table.inc"
constexpr int kPow5N = ZSVD_POW5_QMAX - ZSVD_POW5_QMIN + 1;
}  // namespace

__device__ unsigned long long g_csv_pow5[2 * kPow5N];
__device__ short g_csv_pow5e[kPow5N];

namespace {

constexpr int kTileBytes = 32768;  // 256 threads x 128 bytes
constexpr long long kNone = 0x7FFFFFFFFFFFFFFFll;

struct CsvSummary {
    long long nl;              // lines in the chunk
    unsigned long long nonblank;  // non-blank lines
    long long first_nonblank;  // smallest non-blank line index
    long long err_line;        // smallest line index with an error
};

struct LineInfo {
    long long ncells;
    long long bad_idx;  // first failing cell at index >= drop, or -1
    long long bad_b, bad_e;  // its trimmed byte range in the chunk
    long long ls, le;
    int none_numeric;
    int bad_kind;
};

__device__ __forceinline__ const uint64_t* pow5_ptr() { return (const uint64_t*)g_csv_pow5; }

// Bit i set when byte i of the 16 bytes equals the pattern byte (replicated x4).
__device__ __forceinline__ unsigned match16(uint4 v, unsigned pat) {
    unsigned m = 0;
    const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const unsigned e = __vcmpeq4(w[i], pat) & 0x80808080u;
        m |= (((e >> 7) & 1u) | ((e >> 14) & 2u) | ((e >> 21) & 4u) | ((e >> 28) & 8u)) << (4 * i);
    }
    return m;
}

// Bits of the 16 bytes at [off, off + 16) that lie in [lo, hi).
__device__ __forceinline__ unsigned range16(long long off, long long lo, long long hi) {
    long long a = lo - off, b = hi - off;
    a = a < 0 ? 0 : (a > 16 ? 16 : a);
    b = b < 0 ? 0 : (b > 16 ? 16 : b);
    if (b <= a) return 0;
    const unsigned full = (b >= 16) ? 0xFFFFu : ((1u << b) - 1u);
    return full & ~((1u << a) - 1u);
}

__device__ __forceinline__ int warp_incl_scan(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Exclusive block scan of one int per thread (blockDim.x == 256); returns the
// thread's exclusive prefix and writes the block total to *total.
__device__ __forceinline__ int block_excl_scan(int v, int* total) {
    __shared__ int s_w[8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int inc = warp_incl_scan(v);
    if (lane == 31) s_w[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        const int x = lane < 8 ? s_w[lane] : 0;
        const int y = warp_incl_scan(x);
        if (lane < 8) s_w[lane] = y - x;
        if (lane == 7) *total = y;
    }
    __syncthreads();
    const int r = s_w[wid] + inc - v;
    __syncthreads();
    return r;
}

__global__ void csv_reset_kernel(CsvSummary* s) {
    s->nl = 0;
    s->nonblank = 0;
    s->first_nonblank = kNone;
    s->err_line = kNone;
}

__global__ void __launch_bounds__(256) csv_count_kernel(const uint8_t* __restrict__ text, long long n,
                                                        int* __restrict__ tile_cnt) {
    const long long base = (long long)blockIdx.x * kTileBytes + threadIdx.x * 128;
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const long long off = base + 16 * k;
        if (off < n) {
            const uint4 v = *reinterpret_cast<const uint4*>(text + off);
            cnt += __popc(match16(v, 0x0a0a0a0au) & range16(off, 0, n));
        }
    }
    __shared__ int tot;
    block_excl_scan(cnt, &tot);
    if (threadIdx.x == 0) tile_cnt[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(256) csv_lines_kernel(const uint8_t* __restrict__ text, long long n,
                                                        const int* __restrict__ tile_cnt, int ntiles,
                                                        int* __restrict__ line_end, CsvSummary* sum) {
    // lines before this tile
    int pre = 0;
    for (int t = threadIdx.x; t < (int)blockIdx.x; t += 256) pre += tile_cnt[t];
    __shared__ int s_pre;
    block_excl_scan(pre, &s_pre);
    const int ptot = s_pre;
    const long long base = (long long)blockIdx.x * kTileBytes + threadIdx.x * 128;
    unsigned masks[8];
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const long long off = base + 16 * k;
        masks[k] = 0;
        if (off < n) {
            const uint4 v = *reinterpret_cast<const uint4*>(text + off);
            masks[k] = match16(v, 0x0a0a0a0au) & range16(off, 0, n);
        }
        cnt += __popc(masks[k]);
    }
    __shared__ int tot;
    int idx = ptot + block_excl_scan(cnt, &tot);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        unsigned m = masks[k];
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            line_end[idx++] = (int)(base + 16 * k + b);
        }
    }
    if (blockIdx.x == ntiles - 1 && threadIdx.x == 0) sum->nl = ptot + tot;
}

__global__ void __launch_bounds__(256) csv_classify_kernel(const uint8_t* __restrict__ text,
                                                           const int* __restrict__ line_end, CsvSummary* sum,
                                                           uint8_t* __restrict__ flag) {
    const long long nl = sum->nl;
    const int lane = threadIdx.x & 31;
    for (long long L0 = (long long)blockIdx.x * blockDim.x; L0 < nl; L0 += (long long)gridDim.x * blockDim.x) {
        const long long L = L0 + threadIdx.x;
        bool nonblank = false;
        if (L < nl) {
            const long long ls = L ? (long long)line_end[L - 1] + 1 : 0, le = line_end[L];
            for (long long p = ls; p < le; ++p)
                if (!zcsv::is_ws(text[p])) {
                    nonblank = true;
                    break;
                }
            flag[L] = nonblank ? 1 : 0;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, nonblank);
        if (bal && lane == 0) {
            atomicAdd(&sum->nonblank, (unsigned long long)__popc(bal));
            atomicMin(&sum->first_nonblank, L0 + threadIdx.x + (__ffs(bal) - 1));
        }
    }
}

__global__ void csv_line_info_kernel(const uint8_t* __restrict__ text, const int* __restrict__ line_end,
                                     long long L, int drop, const short* __restrict__ pexp, LineInfo* out) {
    const long long ls = L ? (long long)line_end[L - 1] + 1 : 0, le = line_end[L];
    LineInfo r;
    r.ls = ls;
    r.le = le;
    r.none_numeric = 1;
    r.bad_idx = -1;
    r.bad_kind = 0;
    r.bad_b = r.bad_e = 0;
    long long idx = 0, p = ls;
    while (true) {
        long long e = p;
        while (e < le && text[e] != ',') ++e;
        double v;
        const int kind = zcsv::parse_raw_cell(text + p, text + e, pow5_ptr(), pexp, &v);
        if (kind != zcsv::kNotNumeric) r.none_numeric = 0;
        if (idx >= drop && kind != zcsv::kOk && r.bad_idx < 0) {
            r.bad_idx = idx;
            r.bad_kind = kind;
            long long b = p, ee = e;
            while (b < ee && zcsv::is_ws(text[b])) ++b;
            while (ee > b && zcsv::is_ws(text[ee - 1])) --ee;
            r.bad_b = b;
            r.bad_e = ee;
        }
        ++idx;
        if (e >= le) break;
        p = e + 1;
    }
    r.ncells = idx;
    *out = r;
}

// First line >= from with flag set (or nl).
__global__ void csv_find_kernel(const uint8_t* __restrict__ flag, const CsvSummary* sum, long long from,
                                long long* out) {
    long long L = from;
    while (L < sum->nl && !flag[L]) ++L;
    *out = L;
}

// rowidx[L] = number of data lines before L (one CTA of 1024 threads).
__global__ void __launch_bounds__(1024) csv_rowidx_kernel(const uint8_t* __restrict__ flag, const CsvSummary* sum,
                                                          int* __restrict__ rowidx) {
    __shared__ int s_w[32];
    __shared__ int s_carry;
    const long long nl = sum->nl;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (long long b = 0; b < nl; b += 1024) {
        const long long L = b + threadIdx.x;
        const int f = (L < nl) ? flag[L] : 0;
        const int inc = warp_incl_scan(f);
        if (lane == 31) s_w[wid] = inc;
        __syncthreads();
        if (wid == 0) {
            const int x = s_w[lane];
            s_w[lane] = warp_incl_scan(x) - x;
        }
        __syncthreads();
        const int carry = s_carry;
        if (L < nl) rowidx[L] = carry + s_w[wid] + inc - f;
        __syncthreads();
        if (threadIdx.x == 1023) s_carry = carry + s_w[wid] + inc;
        __syncthreads();
    }
}

// One warp per line.  Lines with flag 0 (blank, header) are skipped; a data
// line's values go to out[(row_base + rowidx) * C + cell - drop].
__global__ void __launch_bounds__(256) csv_parse_kernel(const uint8_t* __restrict__ text,
                                                        const int* __restrict__ line_end,
                                                        const uint8_t* __restrict__ flag,
                                                        const int* __restrict__ rowidx, CsvSummary* sum,
                                                        long long row_base, int C, int drop,
                                                        const short* __restrict__ pexp,
                                                        double* __restrict__ out) {
    const long long nl = sum->nl;
    const int lane = threadIdx.x & 31;
    const long long warp0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    const uint64_t* pow5 = pow5_ptr();
    for (long long L = warp0; L < nl; L += nwarps) {
        if (!flag[L]) continue;
        const long long ls = L ? (long long)line_end[L - 1] + 1 : 0, le = line_end[L];
        const long long row = row_base + (rowidx ? rowidx[L] : L);
        double* orow = out + row * C;
        long long bad = kNone;
        long long before = 0;  // commas before the current window
        auto cell = [&](long long idx, long long start) {
            long long e = start;
            while (e < le && text[e] != ',') ++e;
            if (idx < drop) return;
            double v;
            const int kind = zcsv::parse_raw_cell(text + start, text + e, pow5, pexp, &v);
            if (kind != zcsv::kOk) {
                if (idx < bad) bad = idx;
            } else if (idx - drop < C) {
                orow[idx - drop] = v;
            }
        };
        for (long long wb = ls & ~15ll; wb < le; wb += 512) {
            const long long seg = wb + 16 * lane;
            unsigned m = 0;
            if (seg < le) {
                const uint4 v = *reinterpret_cast<const uint4*>(text + seg);
                m = match16(v, 0x2c2c2c2cu) & range16(seg, ls, le);
            }
            const int cnt = __popc(m);
            const int inc = warp_incl_scan(cnt);
            const int tot = __shfl_sync(0xffffffffu, inc, 31);
            if (seg <= ls && ls < seg + 16) cell(0, ls);
            long long k = before + inc - cnt;
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                cell(++k, seg + b + 1);
            }
            before += tot;
        }
        // the first failing cell of the line
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const long long t = __shfl_xor_sync(0xffffffffu, bad, o);
            bad = t < bad ? t : bad;
        }
        const long long ncells = before + 1;
        const bool err = (drop && ncells < 2) || bad != kNone || ncells - drop != C;
        if (err && lane == 0) atomicMin(&sum->err_line, L);
    }
}

// ---- host ----------------------------------------------------------------------
#define CSV_CUDA(expr)                                                                               \
    do {                                                                                             \
        cudaError_t e_ = (expr);                                                                     \
        if (e_ != cudaSuccess)                                                                       \
            return set_error(e_ == cudaErrorMemoryAllocation ? ZSVD_ERR_NO_MEMORY : ZSVD_ERR_CUDA,   \
                             std::string(#expr) + ": " + cudaGetErrorString(e_));                    \
    } while (0)
#define CSV_TRY(expr)                   \
    do {                                \
        int st_ = (expr);               \
        if (st_ != ZSVD_OK) return st_; \
    } while (0)

std::mutex g_csv_mu;
bool g_csv_tables[64];

int csv_init_device(int dev) {
    std::lock_guard<std::mutex> lk(g_csv_mu);
    if (g_csv_tables[dev]) return ZSVD_OK;
    CSV_CUDA(cudaMemcpyToSymbol(g_csv_pow5, kPow5Mant, sizeof(kPow5Mant)));
    CSV_CUDA(cudaMemcpyToSymbol(g_csv_pow5e, kPow5Exp, sizeof(kPow5Exp)));
    g_csv_tables[dev] = true;
    return ZSVD_OK;
}

// Pinned chunk buffers are kept for the process (allocating 100+ MB of pinned
// memory costs tens of milliseconds; a reader reuses them).
struct PinnedPool {
    std::mutex mu;
    std::vector<std::pair<char*, size_t>> free_list;
    char* get(size_t bytes, size_t* cap) {
        {
            std::lock_guard<std::mutex> lk(mu);
            for (size_t i = 0; i < free_list.size(); ++i)
                if (free_list[i].second >= bytes) {
                    char* p = free_list[i].first;
                    *cap = free_list[i].second;
                    free_list.erase(free_list.begin() + (long)i);
                    return p;
                }
        }
        void* p = nullptr;
        if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) return nullptr;
        *cap = bytes;
        return (char*)p;
    }
    void put(char* p, size_t cap) {
        if (!p) return;
        std::lock_guard<std::mutex> lk(mu);
        free_list.emplace_back(p, cap);
    }
};
PinnedPool g_pinned;

constexpr int kRing = 4;

// Chunk size: 64 MB; ZSVD_CSV_CHUNK_BYTES overrides it (tests use tiny chunks
// to put chunk boundaries, carries and buffer growth everywhere).
size_t chunk_bytes() {
    static const size_t v = [] {
        const char* e = std::getenv("ZSVD_CSV_CHUNK_BYTES");
        const long long x = e ? std::atoll(e) : 0;
        return x >= 64 ? (size_t)x : (size_t)(64ull << 20);
    }();
    return v;
}

size_t pread_all(int fd, char* d, size_t n, size_t o) {
    size_t got = 0;
    while (got < n) {
        const ssize_t r = pread(fd, d + got, n - got, (off_t)(o + got));
        if (r <= 0) break;
        got += (size_t)r;
    }
    return got;
}

// Persistent pread workers: one chunk is read as P slices in parallel (page
// cache -> pinned memory runs at ~8 GB/s per thread; 12 threads exceed the
// ~50 GB/s host-to-device copy that follows).
struct ReadPool {
    int fd, P;
    std::vector<std::thread> th;
    std::mutex mu;
    std::condition_variable cv, done_cv;
    uint64_t gen = 0;
    int pending = 0;
    bool quit = false;
    char* dst = nullptr;
    size_t len = 0, off = 0, part = 0;
    std::vector<size_t> got;

    ReadPool(int f, int p) : fd(f), P(p), got(p, 0) {
        for (int i = 0; i < P; ++i) th.emplace_back([this, i] { loop(i); });
    }
    ~ReadPool() {
        {
            std::lock_guard<std::mutex> lk(mu);
            quit = true;
        }
        cv.notify_all();
        for (auto& t : th) t.join();
    }
    void loop(int i) {
        uint64_t seen = 0;
        std::unique_lock<std::mutex> lk(mu);
        while (true) {
            cv.wait(lk, [&] { return quit || gen != seen; });
            if (quit) return;
            seen = gen;
            const size_t b = i * part, e = std::min(len, b + part);
            char* d = dst;
            const size_t o = off;
            lk.unlock();
            const size_t g = b < e ? pread_all(fd, d + b, e - b, o + b) : 0;
            lk.lock();
            got[i] = g;
            if (--pending == 0) done_cv.notify_all();
        }
    }
    // Reads n bytes at o into d; returns the bytes read (short at end of file).
    size_t read(char* d, size_t n, size_t o) {
        if (n < (8u << 20) || P == 1) return pread_all(fd, d, n, o);
        {
            std::unique_lock<std::mutex> lk(mu);
            dst = d;
            len = n;
            off = o;
            part = (n + P - 1) / P;
            pending = P;
            ++gen;
        }
        cv.notify_all();
        std::unique_lock<std::mutex> lk(mu);
        done_cv.wait(lk, [&] { return pending == 0; });
        size_t total = 0;
        for (int i = 0; i < P; ++i) {
            const size_t b = i * part, e = std::min(n, b + part);
            if (b >= e) break;
            total += got[i];
            if (got[i] < e - b) break;  // end of file inside this slice
        }
        return total;
    }
};

struct HostChunk {
    char* buf = nullptr;
    size_t cap = 0;
    size_t len = 0;
    bool eof = false;
    bool ready = false;
    bool busy = false;  // handed to the consumer
};

// Background reader: fills the pinned ring with chunks that end at '\n'.
struct Reader {
    int fd;
    std::mutex mu;
    std::condition_variable cv;
    HostChunk ring[kRing];
    bool stop = false;
    bool failed = false;
    std::thread th;

    ReadPool pool;
    explicit Reader(int f)
        : fd(f), pool(f, (int)std::max(2u, std::min(12u, std::thread::hardware_concurrency() > 2
                                                              ? std::thread::hardware_concurrency() - 2
                                                              : 2u))) {}
    ~Reader() {
        {
            std::lock_guard<std::mutex> lk(mu);
            stop = true;
        }
        cv.notify_all();
        if (th.joinable()) th.join();
        for (auto& c : ring) g_pinned.put(c.buf, c.cap);
    }

    void run() {
        std::vector<char> carry;
        size_t pos = 0;
        for (int k = 0;; k = (k + 1) % kRing) {
            HostChunk* c = &ring[k];
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return stop || (!c->ready && !c->busy); });
                if (stop) return;
            }
            size_t want_cap = std::max(chunk_bytes(), carry.size() * 2 + 1);
            if (c->cap < want_cap) {
                g_pinned.put(c->buf, c->cap);
                c->buf = g_pinned.get(want_cap, &c->cap);
                if (!c->buf) return fail_now();
            }
            std::memcpy(c->buf, carry.data(), carry.size());
            size_t len = carry.size();
            bool eof = false;
            while (true) {
                const size_t want = c->cap - 1 - len;
                const size_t got = pool.read(c->buf + len, want, pos);
                pos += got;
                len += got;
                if (got < want) {
                    eof = true;
                    break;
                }
                if (memrchr(c->buf, '\n', len)) break;
                // one line longer than the buffer: grow it
                size_t ncap = 0;
                char* nb = g_pinned.get(c->cap * 2, &ncap);
                if (!nb) return fail_now();
                std::memcpy(nb, c->buf, len);
                g_pinned.put(c->buf, c->cap);
                c->buf = nb;
                c->cap = ncap;
            }
            size_t clen;
            if (eof) {
                clen = len;
                if (len > 0 && c->buf[len - 1] != '\n') c->buf[clen++] = '\n';
                carry.clear();
            } else {
                const char* p = (const char*)memrchr(c->buf, '\n', len);
                clen = (size_t)(p - c->buf) + 1;
                carry.assign(c->buf + clen, c->buf + len);
            }
            {
                std::lock_guard<std::mutex> lk(mu);
                c->len = clen;
                c->eof = eof;
                c->ready = true;
            }
            cv.notify_all();
            if (eof) return;
        }
    }
    void fail_now() {
        std::lock_guard<std::mutex> lk(mu);
        failed = true;
        cv.notify_all();
    }
    // Blocks for chunk k; null if the reader failed.
    HostChunk* take(int k) {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return ring[k].ready || failed; });
        if (!ring[k].ready) return nullptr;
        ring[k].ready = false;
        ring[k].busy = true;
        return &ring[k];
    }
    void give_back(HostChunk* c) {
        {
            std::lock_guard<std::mutex> lk(mu);
            c->busy = false;
        }
        cv.notify_all();
    }
};

}  // namespace
}  // namespace zsvd

using namespace zsvd;

struct zsvd_csv {
    int device = 0;
    long long rows = 0, cols = 0;
    int status = ZSVD_OK;
    size_t err_line = 0;
    std::string msg;
    double* d_rows = nullptr;
    long long cap = 0;
};

namespace {

struct DevGuard {
    int prev = -1;
    explicit DevGuard(int d) {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != d) cudaSetDevice(d);
    }
    ~DevGuard() {
        int cur;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

// Device buffers, streams and pinned scalars of one reader; the last one used
// on a device is cached, so a steady stream of files allocates nothing.
struct CsvWorkspace {
    cudaStream_t cs = nullptr, xs = nullptr;  // compute, copy
    cudaEvent_t copied[2] = {nullptr, nullptr}, consumed[2] = {nullptr, nullptr};
    uint8_t* dtext[2] = {nullptr, nullptr};
    size_t dtext_cap[2] = {0, 0};
    size_t scratch_cap = 0;  // lines
    int* d_tile = nullptr;
    int* d_line_end = nullptr;
    uint8_t* d_flag = nullptr;
    int* d_rowidx = nullptr;
    CsvSummary* d_sum = nullptr;
    LineInfo* d_info = nullptr;
    long long* d_find = nullptr;
    CsvSummary* h_sum = nullptr;  // pinned
    LineInfo* h_info = nullptr;
    long long* h_find = nullptr;

    CsvWorkspace() = default;
    CsvWorkspace(const CsvWorkspace&) = delete;
    CsvWorkspace& operator=(const CsvWorkspace&) = delete;
    void swap(CsvWorkspace& o) {
        std::swap(cs, o.cs);
        std::swap(xs, o.xs);
        for (int i = 0; i < 2; ++i) {
            std::swap(copied[i], o.copied[i]);
            std::swap(consumed[i], o.consumed[i]);
            std::swap(dtext[i], o.dtext[i]);
            std::swap(dtext_cap[i], o.dtext_cap[i]);
        }
        std::swap(scratch_cap, o.scratch_cap);
        std::swap(d_tile, o.d_tile);
        std::swap(d_line_end, o.d_line_end);
        std::swap(d_flag, o.d_flag);
        std::swap(d_rowidx, o.d_rowidx);
        std::swap(d_sum, o.d_sum);
        std::swap(d_info, o.d_info);
        std::swap(d_find, o.d_find);
        std::swap(h_sum, o.h_sum);
        std::swap(h_info, o.h_info);
        std::swap(h_find, o.h_find);
    }
    ~CsvWorkspace() {
        if (cs) cudaStreamSynchronize(cs);
        if (xs) cudaStreamSynchronize(xs);
        for (int i = 0; i < 2; ++i) {
            if (dtext[i]) cudaFree(dtext[i]);
            if (copied[i]) cudaEventDestroy(copied[i]);
            if (consumed[i]) cudaEventDestroy(consumed[i]);
        }
        cudaFree(d_tile);
        cudaFree(d_line_end);
        cudaFree(d_flag);
        cudaFree(d_rowidx);
        cudaFree(d_sum);
        cudaFree(d_info);
        cudaFree(d_find);
        cudaFreeHost(h_sum);
        cudaFreeHost(h_info);
        cudaFreeHost(h_find);
        if (cs) cudaStreamDestroy(cs);
        if (xs) cudaStreamDestroy(xs);
    }
};

std::mutex g_ws_mu;
CsvWorkspace* g_ws_cache[64];

struct Ingest : CsvWorkspace {
    zsvd_csv* h;
    zsvd_csv_options opt;
    int fd;
    int device;
    size_t file_size;
    short* pexp = nullptr;
    // parse state
    bool seen_content = false;
    long long C = 0;
    long long row_base = 0, line_base = 0;
    bool done = false;

    // borrow the device's cached workspace (if no other reader holds it)
    void borrow() {
        std::lock_guard<std::mutex> lk(g_ws_mu);
        if (g_ws_cache[device]) {
            swap(*g_ws_cache[device]);
            delete g_ws_cache[device];
            g_ws_cache[device] = nullptr;
        }
    }
    void give_back_ws() {
        if (cs) cudaStreamSynchronize(cs);
        if (xs) cudaStreamSynchronize(xs);
        std::lock_guard<std::mutex> lk(g_ws_mu);
        if (!g_ws_cache[device]) {
            g_ws_cache[device] = new CsvWorkspace();
            g_ws_cache[device]->swap(*this);
        }
    }

    int setup() {
        borrow();
        if (!cs) CSV_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        if (!xs) CSV_CUDA(cudaStreamCreateWithFlags(&xs, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            if (!copied[i]) CSV_CUDA(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming));
            if (!consumed[i]) CSV_CUDA(cudaEventCreateWithFlags(&consumed[i], cudaEventDisableTiming));
        }
        if (!d_sum) CSV_CUDA(cudaMalloc(&d_sum, sizeof(CsvSummary)));
        if (!d_info) CSV_CUDA(cudaMalloc(&d_info, sizeof(LineInfo)));
        if (!d_find) CSV_CUDA(cudaMalloc(&d_find, sizeof(long long)));
        if (!h_sum) CSV_CUDA(cudaMallocHost(&h_sum, sizeof(CsvSummary)));
        if (!h_info) CSV_CUDA(cudaMallocHost(&h_info, sizeof(LineInfo)));
        if (!h_find) CSV_CUDA(cudaMallocHost(&h_find, sizeof(long long)));
        CSV_CUDA(cudaGetSymbolAddress((void**)&pexp, g_csv_pow5e));
        // a cached workspace's events may still carry an earlier file's state
        for (int i = 0; i < 2; ++i) CSV_CUDA(cudaEventRecord(consumed[i], cs));
        return ZSVD_OK;
    }

    int ensure_text(int s, size_t n) {
        if (dtext_cap[s] >= n + 64) return ZSVD_OK;
        if (dtext[s]) {
            CSV_CUDA(cudaStreamSynchronize(cs));
            CSV_CUDA(cudaStreamSynchronize(xs));
            cudaFree(dtext[s]);
        }
        dtext_cap[s] = std::max(n + 64, chunk_bytes() + 64);
        CSV_CUDA(cudaMalloc(&dtext[s], dtext_cap[s]));
        return ZSVD_OK;
    }

    int ensure_scratch(size_t n) {
        if (scratch_cap >= n + 1) return ZSVD_OK;
        CSV_CUDA(cudaStreamSynchronize(cs));
        cudaFree(d_tile);
        cudaFree(d_line_end);
        cudaFree(d_flag);
        cudaFree(d_rowidx);
        scratch_cap = std::max(n + 1, chunk_bytes() + 1);
        CSV_CUDA(cudaMalloc(&d_tile, (scratch_cap / kTileBytes + 2) * sizeof(int)));
        CSV_CUDA(cudaMalloc(&d_line_end, scratch_cap * sizeof(int)));
        CSV_CUDA(cudaMalloc(&d_flag, scratch_cap));
        CSV_CUDA(cudaMalloc(&d_rowidx, scratch_cap * sizeof(int)));
        return ZSVD_OK;
    }

    int ensure_rows(long long need, long long line_bytes) {
        if (need <= h->cap) return ZSVD_OK;
        long long cap = h->cap * 2;
        if (h->cap == 0) {
            const long long per = std::max(2ll, line_bytes + 1);
            cap = (long long)(file_size / (size_t)per) * 5 / 4 + 1024;
        }
        cap = std::max(cap, need);
        double* nb = nullptr;
        CSV_CUDA(cudaMallocAsync((void**)&nb, (size_t)cap * (size_t)C * 8, cs));
        if (h->d_rows) {
            CSV_CUDA(cudaMemcpyAsync(nb, h->d_rows, (size_t)row_base * (size_t)C * 8, cudaMemcpyDeviceToDevice, cs));
            CSV_CUDA(cudaFreeAsync(h->d_rows, cs));
        }
        h->d_rows = nb;
        h->cap = cap;
        return ZSVD_OK;
    }

    int line_info(int s, long long L, int drop) {
        csv_line_info_kernel<<<1, 1, 0, cs>>>(dtext[s], d_line_end, L, drop, pexp, d_info);
        count_launches(1);
        CSV_CUDA(cudaGetLastError());
        CSV_CUDA(cudaMemcpyAsync(h_info, d_info, sizeof(LineInfo), cudaMemcpyDeviceToHost, cs));
        CSV_CUDA(cudaStreamSynchronize(cs));
        return ZSVD_OK;
    }

    // Records the reader's pending error after `rows_before` rows and stops.
    void parse_error(long long line_no, const std::string& what, long long rows_before) {
        h->status = ZSVD_ERR_PARSE;
        h->err_line = (size_t)line_no;
        h->msg = "line " + std::to_string(line_no) + ": " + what;
        h->rows = rows_before;
        done = true;
    }

    std::string cell_error(const HostChunk* c, const LineInfo& in) {
        if (in.bad_kind == zcsv::kNonFinite) return "cell value is not finite";
        return "cell '" + std::string(c->buf + in.bad_b, c->buf + in.bad_e) + "' is not numeric";
    }

    // The first data row fixes the column count (csv.hpp:115-125).
    int first_data_row(int s, const HostChunk* c, long long L) {
        const int drop = opt.drop_timestamp ? 1 : 0;
        CSV_TRY(line_info(s, L, drop));
        const LineInfo in = *h_info;
        const long long line_no = line_base + L + 1;
        if (drop && in.ncells < 2) {
            parse_error(line_no, "row has no value columns after the timestamp", row_base);
            return ZSVD_OK;
        }
        if (in.bad_idx >= 0) {
            parse_error(line_no, cell_error(c, in), row_base);
            return ZSVD_OK;
        }
        const long long cols = in.ncells - drop;
        if (opt.expected_cols >= 0 && cols != opt.expected_cols) {
            h->status = ZSVD_ERR_SCHEMA;
            h->err_line = 0;
            h->msg = "expected " + std::to_string(opt.expected_cols) + " columns, file has " + std::to_string(cols);
            h->rows = row_base;
            done = true;
            return ZSVD_OK;
        }
        C = cols;
        h->cols = cols;
        return ensure_rows(1, in.le - in.ls);
    }

    int process(int s, const HostChunk* c) {
        const long long n = (long long)c->len;
        const int ntiles = (int)((n + kTileBytes - 1) / kTileBytes);
        CSV_TRY(ensure_scratch((size_t)n));
        CSV_CUDA(cudaStreamWaitEvent(cs, copied[s], 0));
        csv_reset_kernel<<<1, 1, 0, cs>>>(d_sum);
        csv_count_kernel<<<ntiles, 256, 0, cs>>>(dtext[s], n, d_tile);
        csv_lines_kernel<<<ntiles, 256, 0, cs>>>(dtext[s], n, d_tile, ntiles, d_line_end, d_sum);
        const int cgrid = (int)std::min<long long>(148 * 8, std::max<long long>(1, n / (256 * 16)));
        csv_classify_kernel<<<cgrid, 256, 0, cs>>>(dtext[s], d_line_end, d_sum, d_flag);
        count_launches(4);
        CSV_CUDA(cudaGetLastError());
        CSV_CUDA(cudaMemcpyAsync(h_sum, d_sum, sizeof(CsvSummary), cudaMemcpyDeviceToHost, cs));
        CSV_CUDA(cudaStreamSynchronize(cs));
        const CsvSummary sm = *h_sum;
        long long ndata = (long long)sm.nonblank;
        long long first_data = sm.nonblank ? sm.first_nonblank : -1;
        if (!seen_content && sm.nonblank > 0) {
            seen_content = true;
            // a leading line with no numeric cell is a header (csv.hpp:89-94)
            CSV_TRY(line_info(s, sm.first_nonblank, 0));
            if (h_info->none_numeric) {
                CSV_CUDA(cudaMemsetAsync(d_flag + sm.first_nonblank, 0, 1, cs));
                --ndata;
                first_data = -1;
                if (ndata > 0) {
                    csv_find_kernel<<<1, 1, 0, cs>>>(d_flag, d_sum, sm.first_nonblank + 1, d_find);
                    count_launches(1);
                    CSV_CUDA(cudaMemcpyAsync(h_find, d_find, sizeof(long long), cudaMemcpyDeviceToHost, cs));
                    CSV_CUDA(cudaStreamSynchronize(cs));
                    first_data = *h_find;
                }
            }
        }
        if (ndata > 0 && C == 0) {
            CSV_TRY(first_data_row(s, c, first_data));
            if (done) return ZSVD_OK;
        }
        if (ndata > 0) {
            const bool skips = ndata != sm.nl;
            if (skips) {
                csv_rowidx_kernel<<<1, 1024, 0, cs>>>(d_flag, d_sum, d_rowidx);
                count_launches(1);
            }
            CSV_TRY(ensure_rows(row_base + ndata, 0));
            const int pgrid = (int)std::min<long long>(148 * 16, (sm.nl + 7) / 8);
            csv_parse_kernel<<<pgrid, 256, 0, cs>>>(dtext[s], d_line_end, d_flag, skips ? d_rowidx : nullptr, d_sum,
                                                    row_base, (int)C, opt.drop_timestamp ? 1 : 0, pexp, h->d_rows);
            count_launches(1);
            CSV_CUDA(cudaGetLastError());
            CSV_CUDA(cudaMemcpyAsync(h_sum, d_sum, sizeof(CsvSummary), cudaMemcpyDeviceToHost, cs));
            CSV_CUDA(cudaStreamSynchronize(cs));
            const long long err = h_sum->err_line;
            if (err != kNone) {
                long long before = err;
                if (skips) {
                    int r = 0;
                    CSV_CUDA(cudaMemcpy(&r, d_rowidx + err, sizeof(int), cudaMemcpyDeviceToHost));
                    before = r;
                }
                const int drop = opt.drop_timestamp ? 1 : 0;
                CSV_TRY(line_info(s, err, drop));
                const LineInfo in = *h_info;
                std::string what;
                if (drop && in.ncells < 2) what = "row has no value columns after the timestamp";
                else if (in.bad_idx >= 0) what = cell_error(c, in);
                else what = "expected " + std::to_string(C) + " columns, got " + std::to_string(in.ncells - drop);
                parse_error(line_base + err + 1, what, row_base + before);
                return ZSVD_OK;
            }
        }
        CSV_CUDA(cudaEventRecord(consumed[s], cs));
        row_base += std::max(0ll, ndata);
        line_base += sm.nl;
        return ZSVD_OK;
    }

    int issue_copy(int s, const HostChunk* c) {
        CSV_TRY(ensure_text(s, c->len));
        CSV_CUDA(cudaStreamWaitEvent(xs, consumed[s], 0));
        CSV_CUDA(cudaMemcpyAsync(dtext[s], c->buf, c->len, cudaMemcpyHostToDevice, xs));
        CSV_CUDA(cudaEventRecord(copied[s], xs));
        return ZSVD_OK;
    }

    double t_wait = 0, t_proc = 0;
    int nchunks = 0;
    static double now_s() {
        return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
    }

    int run() {
        CSV_TRY(setup());
        Reader rd(fd);
        rd.th = std::thread([&rd] { rd.run(); });
        int k = 0;
        HostChunk* cur = rd.take(k);
        if (!cur) return set_error(ZSVD_ERR_IO, "read failed");
        if (cur->len == 0) {
            rd.give_back(cur);
            h->rows = 0;
            return ZSVD_OK;
        }
        int st = issue_copy(0, cur);
        for (int j = 0; st == ZSVD_OK; ++j) {
            HostChunk* next = nullptr;
            if (!cur->eof) {
                const double tw = now_s();
                next = rd.take((k + 1) % kRing);
                t_wait += now_s() - tw;
                if (!next) {
                    st = set_error(ZSVD_ERR_IO, "read failed");
                    break;
                }
                if (next->len > 0) st = issue_copy((j + 1) & 1, next);
                if (st != ZSVD_OK) break;
            }
            const double tp = now_s();
            st = process(j & 1, cur);
            t_proc += now_s() - tp;
            ++nchunks;
            rd.give_back(cur);
            cur = nullptr;
            if (st != ZSVD_OK || done || !next || next->len == 0) {
                if (next) rd.give_back(next);
                break;
            }
            cur = next;
            k = (k + 1) % kRing;
        }
        if (cur) rd.give_back(cur);
        if (st != ZSVD_OK) return st;
        if (!done) h->rows = row_base;
        if (std::getenv("ZSVD_CSV_TRACE"))
            std::fprintf(stderr, "[csv] %d chunks, waiting for the reader %.1f ms, processing %.1f ms\n", nchunks,
                         t_wait * 1e3, t_proc * 1e3);
        CSV_CUDA(cudaStreamSynchronize(cs));
        return ZSVD_OK;
    }
};

}  // namespace

extern "C" {

int zsvd_csv_read(const char* path, zsvd_csv_options opt, int device, zsvd_csv** out) {
    if (!out || !path) return set_error(ZSVD_ERR_INVALID_PARAMETER, "null argument");
    *out = nullptr;
    const int fd = open(path, O_RDONLY);
    if (fd < 0) return set_error(ZSVD_ERR_IO, std::string("cannot open '") + path + "' for reading");
    struct stat stt;
    if (fstat(fd, &stt) != 0 || S_ISDIR(stt.st_mode)) {
        close(fd);
        return set_error(ZSVD_ERR_IO, std::string("cannot open '") + path + "' for reading");
    }
    int st = ensure_device(device);
    if (st != ZSVD_OK) {
        close(fd);
        return st;
    }
    DevGuard g(device);
    st = csv_init_device(device);
    if (st != ZSVD_OK) {
        close(fd);
        return st;
    }
    auto* h = new zsvd_csv();
    h->device = device;
    {
        Ingest ing;
        ing.h = h;
        ing.opt = opt;
        ing.fd = fd;
        ing.file_size = (size_t)stt.st_size;
        ing.device = device;
        st = ing.run();
        if (st == ZSVD_OK) ing.give_back_ws();
    }
    close(fd);
    if (st != ZSVD_OK) {
        zsvd_csv_release(h);
        return st;
    }
    *out = h;
    return ZSVD_OK;
}

int zsvd_csv_info(zsvd_csv* h, size_t* rows, size_t* cols, int* error, size_t* error_line) {
    if (!h) return set_error(ZSVD_ERR_INVALID_PARAMETER, "null csv");
    if (rows) *rows = (size_t)h->rows;
    if (cols) *cols = (size_t)h->cols;
    if (error) *error = h->status;
    if (error_line) *error_line = h->err_line;
    return ZSVD_OK;
}

int zsvd_csv_error_message(zsvd_csv* h, char* buf, size_t len) {
    if (!h) return set_error(ZSVD_ERR_INVALID_PARAMETER, "null csv");
    if (buf && len) std::snprintf(buf, len, "%s", h->msg.c_str());
    return ZSVD_OK;
}

int zsvd_csv_rows_device(zsvd_csv* h, const double** rows) {
    if (!h || !rows) return set_error(ZSVD_ERR_INVALID_PARAMETER, "null argument");
    *rows = h->d_rows;
    return ZSVD_OK;
}

int zsvd_csv_rows_copy(zsvd_csv* h, size_t first, size_t count, double* out) {
    if (!h) return set_error(ZSVD_ERR_INVALID_PARAMETER, "null csv");
    if (first + count > (size_t)h->rows) return set_error(ZSVD_ERR_RANGE, "rows out of range");
    if (count == 0) return ZSVD_OK;
    if (!out) return set_error(ZSVD_ERR_INVALID_PARAMETER, "null output");
    DevGuard g(h->device);
    CSV_CUDA(cudaMemcpy(out, h->d_rows + first * (size_t)h->cols, count * (size_t)h->cols * 8,
                        cudaMemcpyDeviceToHost));
    return ZSVD_OK;
}

int zsvd_csv_release(zsvd_csv* h) {
    if (!h) return ZSVD_OK;
    if (h->d_rows) {
        DevGuard g(h->device);
        cudaFreeAsync(h->d_rows, 0);
    }
    delete h;
    return ZSVD_OK;
}

int zsvd_store_append_csv(zsvd_store* s, zsvd_csv* h, size_t* appended) {
    if (appended) *appended = 0;
    if (!s || !h) return set_error(ZSVD_ERR_INVALID_PARAMETER, "null argument");
    if (h->status != ZSVD_OK) return set_error(h->status, h->msg, h->err_line);
    if (h->rows == 0) return ZSVD_OK;
    zsvd_store_info info;
    CSV_TRY(zsvd_store_info_get(s, &info));
    if ((long long)info.num_columns != h->cols)
        return set_error(ZSVD_ERR_INVALID_INPUT, "row has wrong number of columns");
    CSV_TRY(zsvd_store_append(s, h->d_rows, (size_t)h->rows, (size_t)h->cols, ZSVD_MEM_DEVICE));
    if (appended) *appended = (size_t)h->rows;
    return ZSVD_OK;
}

}  // extern "C"
