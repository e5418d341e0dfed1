// Runs the reference's own CsvReader (csv.hpp, compiled in place from
// /root/reference by oracle/Makefile) over one file and prints what it yields:
// one line per row ("R" + hex bit patterns), then "OK", or the exception
// ("E <type> <line> <what>").  Test tooling only: tests/golden/csv_cases.json is
// generated from this by scripts/gen_csv_golden.py; bench.py --impl reference
// times it ("T" mode) as the reference's CPU parse rate.
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include <rangesvd/csv.hpp>

using namespace rangesvd;

int main(int argc, char** argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: csv_ref <path> <expected_cols|-1> <drop_timestamp 0|1> [T]\n");
        return 2;
    }
    CsvOptions opt;
    const long ec = std::atol(argv[2]);
    if (ec >= 0) opt.expected_cols = (std::size_t)ec;
    opt.drop_timestamp = std::atoi(argv[3]) != 0;
    const bool timing = argc > 4 && argv[4][0] == 'T';
    std::size_t nrows = 0;
    double checksum = 0.0;
    const auto t0 = std::chrono::steady_clock::now();
    try {
        CsvReader reader(argv[1], opt);
        while (auto row = reader.next()) {
            ++nrows;
            if (timing) {
                for (double v : *row) checksum += v;
                continue;
            }
            std::printf("R");
            for (double v : *row) {
                uint64_t b;
                std::memcpy(&b, &v, 8);
                std::printf(" %016" PRIx64, b);
            }
            std::printf("\n");
        }
    } catch (const ParseError& e) {
        std::printf("E ParseError %zu %s\n", e.line(), e.what());
        return 0;
    } catch (const SchemaError& e) {
        std::printf("E SchemaError 0 %s\n", e.what());
        return 0;
    } catch (const IoError& e) {
        std::printf("E IoError 0 %s\n", e.what());
        return 0;
    }
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (timing) std::printf("T %zu %.6f %.17g\n", nrows, s, checksum);
    else std::printf("OK\n");
    return 0;
}
