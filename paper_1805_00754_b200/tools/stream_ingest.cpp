// stream_ingest — cfg4's streaming ingest (BASELINE configs[3]) as a C++ caller
// of the C ABI sees it: rows arrive in small chunks (zsvd_store_append per
// chunk, host memory), a block's SVD fires on fill, and a range query runs
// every `query_every` rows (L ~ U[1e4, 3.2e5] clamped to the rows so far).
//
//   stream_ingest <rows.f64> <rows> <c> <b> <k> <chunk> <query_every> <seed>
//
// Prints one JSON object: wall-clock ingest rows/s (queries included, as in
// cmd_ingest + cmd_query interleaved), the queries' device p50, call counts.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../../include/zsvd.h"

static void ck(int rc, const char* what) {
    if (rc == ZSVD_OK) return;
    char buf[512];
    zsvd_last_error(buf, sizeof buf);
    std::fprintf(stderr, "%s failed (%d): %s\n", what, rc, buf);
    std::exit(2);
}

int main(int argc, char** argv) {
    if (argc < 9) {
        std::fprintf(stderr, "usage: %s rows.f64 rows c b k chunk query_every seed\n", argv[0]);
        return 1;
    }
    const size_t rows = std::strtoull(argv[2], nullptr, 10), c = std::strtoull(argv[3], nullptr, 10);
    const size_t b = std::strtoull(argv[4], nullptr, 10), k = std::strtoull(argv[5], nullptr, 10);
    const size_t chunk = std::strtoull(argv[6], nullptr, 10), every = std::strtoull(argv[7], nullptr, 10);
    std::mt19937_64 rng(std::strtoull(argv[8], nullptr, 10));
    std::vector<double> raw(rows * c);
    FILE* f = std::fopen(argv[1], "rb");
    if (!f || std::fread(raw.data(), sizeof(double), raw.size(), f) != raw.size()) {
        std::fprintf(stderr, "cannot read %s\n", argv[1]);
        return 1;
    }
    std::fclose(f);
    zsvd_store* s = nullptr;
    const zsvd_truncation tr{ZSVD_POLICY_FIXED_RANK, 1.0, (uint64_t)k};
    ck(zsvd_store_create_ex(b, c, tr, 0, &s), "create");
    void *e0 = nullptr, *e1 = nullptr;
    ck(zsvd_event_create(&e0), "event");
    ck(zsvd_event_create(&e1), "event");
    // warm: one block through the whole path (first-use allocations)
    ck(zsvd_store_append(s, raw.data(), b, c, ZSVD_MEM_HOST), "warm append");
    ck(zsvd_store_sync(s), "sync");
    ck(zsvd_store_reset(s), "reset");
    std::vector<float> qms;
    size_t calls = 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (size_t i = 0; i < rows; i += chunk) {
        const size_t n = std::min(chunk, rows - i);
        ck(zsvd_store_append(s, raw.data() + i * c, n, c, ZSVD_MEM_HOST), "append");
        ++calls;
        const size_t total = i + n;
        if (every && total % every == 0) {
            const size_t L = std::min<size_t>(total, std::uniform_int_distribution<size_t>(10000, 320000)(rng));
            const size_t first = std::uniform_int_distribution<size_t>(0, total - L)(rng);
            zsvd_snapshot* sn = nullptr;
            ck(zsvd_snapshot_create(s, &sn), "snapshot");
            void* qs = nullptr;
            ck(zsvd_snapshot_stream(sn, &qs), "stream");
            zsvd_factors* res = nullptr;
            ck(zsvd_event_record(e0, qs), "record");
            ck(zsvd_range_query(sn, first, first + L - 1, tr, &res), "query");
            ck(zsvd_event_record(e1, qs), "record");
            float ms = 0.f;
            ck(zsvd_event_elapsed_ms(e0, e1, &ms), "elapsed");
            qms.push_back(ms);
            zsvd_factors_release(res);
            zsvd_snapshot_release(sn);
        }
    }
    ck(zsvd_store_sync(s), "sync");
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::sort(qms.begin(), qms.end());
    const double p50 = qms.empty() ? 0.0 : qms[qms.size() / 2];
    std::printf("{\"ingest_rows_s\": %.6g, \"seconds\": %.6g, \"append_calls\": %zu, \"queries\": %zu, "
                "\"query_p50_ms\": %.6g, \"us_per_call\": %.6g}\n",
                rows / el, el, calls, qms.size(), p50, 1e6 * el / (double)calls);
    zsvd_store_destroy(s);
    return 0;
}
