// Dev: pageable host append through the C ABI, with a SIGSEGV backtrace.
#include <execinfo.h>
#include <signal.h>
#include <unistd.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../include/zsvd.h"
static void on_segv(int) {
    void* bt[64];
    int n = backtrace(bt, 64);
    backtrace_symbols_fd(bt, n, 2);
    _exit(3);
}
int main(int argc, char** argv) {
    signal(SIGSEGV, on_segv);
    const size_t b = 1000, c = 16, rows = 100000;
    std::vector<double> raw(rows * c);
    for (size_t i = 0; i < raw.size(); ++i) raw[i] = (double)((i * 2654435761u) % 1000) / 1000.0 - 0.5;
    zsvd_store* s = nullptr;
    zsvd_truncation t{ZSVD_POLICY_FIXED_RANK, 1.0, 10};
    if (zsvd_store_create_ex(b, c, t, 0, &s)) { std::printf("create failed\n"); return 1; }
    for (int rep = 0; rep < 3; ++rep) {
        int rc = zsvd_store_append(s, raw.data(), rows, c, ZSVD_MEM_HOST);
        char buf[512];
        zsvd_last_error(buf, sizeof buf);
        std::printf("append rc %d %s\n", rc, rc ? buf : "");
        zsvd_store_sync(s);
        zsvd_store_reset(s);
    }
    zsvd_store_destroy(s);
    std::printf("done\n");
}
