// Reference-style C++ test of the drop-in header (include/zsvd.hpp): the same
// calls and assertions as proj/tests/{svd,store,query}_test.cpp, on the GPU.
// Built and run by tests/test_cpp_dropin.py (gpu marker).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "zsvd.hpp"

using namespace rangesvd;

static int failures = 0;
#define EXPECT(cond)                                                        \
    do {                                                                    \
        if (!(cond)) {                                                      \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
            ++failures;                                                     \
        }                                                                   \
    } while (0)
#define EXPECT_THROW(stmt, T)            \
    do {                                 \
        bool thrown = false;             \
        try {                            \
            stmt;                        \
        } catch (const T&) {             \
            thrown = true;               \
        }                                \
        EXPECT(thrown);                  \
    } while (0)

static DenseMatrix random_matrix(std::size_t r, std::size_t c, std::mt19937& rng) {
    std::uniform_real_distribution<double> d(-1.0, 1.0);
    DenseMatrix m(r, c);
    for (std::size_t i = 0; i < r; ++i)
        for (std::size_t j = 0; j < c; ++j) m(i, j) = d(rng);
    return m;
}

static double rel_fro(const DenseMatrix& a, const SvdFactors& f) {
    double num = 0, den = 0;
    for (std::size_t i = 0; i < a.rows(); ++i)
        for (std::size_t j = 0; j < a.cols(); ++j) {
            double x = 0;
            for (std::size_t t = 0; t < f.rank(); ++t) x += f.u(i, t) * f.sigma[t] * f.v(j, t);
            num += (a(i, j) - x) * (a(i, j) - x);
            den += a(i, j) * a(i, j);
        }
    return std::sqrt(num / den);
}

int main() {
    // svd_test.cpp:26-47
    auto f = thin_svd(DenseMatrix::from_rows({{1, 2}, {2, 4}}));
    EXPECT(f.rank() == 1 && std::fabs(f.sigma[0] - 5.0) < 1e-12);
    f = thin_svd(DenseMatrix::from_rows({{3, 0}, {0, 2}}));
    EXPECT(std::fabs(f.sigma[0] - 3.0) < 1e-12 && std::fabs(f.sigma[1] - 2.0) < 1e-12);
    EXPECT_THROW(BlockStore(0, 5, 0.98), InvalidParameterError);
    EXPECT_THROW(BlockStore(5, 5, 1.5), InvalidParameterError);
    // store_test.cpp:85-94
    {
        BlockStore store(4, 3, 0.98);
        std::vector<double> row{1, 2, 2};
        store.append(row);
        store.append(row);
        auto open = store.block(0);
        EXPECT(open.rank() == 1 && std::fabs(open.sigma[0] - 4.242640687119285) <= 1e-12);
        std::vector<double> bad{1, 2, NAN};
        EXPECT_THROW(store.append(bad), InvalidInputError);
        EXPECT(store.total_rows() == 2);
    }
    // query_test.cpp:195-216 (exhaustive over a 14 x 3 stream, b = 4, open tail)
    {
        std::mt19937 rng(149);
        const auto raw = random_matrix(14, 3, rng);
        BlockStore store(4, 3, 1.0);
        for (std::size_t i = 0; i < raw.rows(); ++i) store.append(raw.row(i));
        const auto snap = store.snapshot();
        const auto r = TimeRange::resolve(5, 13, snap);
        EXPECT(r.start_block == 1 && r.end_block == 3 && r.skip_front == 1 && r.keep_back == 2 && r.skip_back == 0);
        for (std::size_t s = 0; s < 14; ++s)
            for (std::size_t e = s; e < 14; ++e) {
                const auto ans = range_query(snap, s, e, 1.0);
                EXPECT(ans.rows() == e - s + 1);
                EXPECT(rel_fro(raw.middle_rows(s, e - s + 1), ans.factors) <= 1e-6);
            }
        EXPECT_THROW(range_query(snap, 0, 14, 1.0), RangeError);
        EXPECT_THROW(range_query(snap, 0, 3, 0.0), InvalidParameterError);
    }
    // fixed-rank policy (BASELINE configs)
    {
        std::mt19937 rng(7);
        const auto raw = random_matrix(300, 16, rng);
        BlockStore store(100, 16, Truncation::fixed_rank(4));
        store.append_rows(raw.data(), raw.rows(), raw.cols());
        const auto ans = range_query(store, 50, 249);
        EXPECT(ans.rank() == 4 && ans.rows() == 200);
    }
    // analysis_test.cpp SimilarRangeSearch: identical copy scores one, errors
    {
        std::mt19937 rng(367);
        std::normal_distribution<double> noise(0.0, 0.3);
        DenseMatrix raw(600, 3);
        for (std::size_t i = 0; i < raw.rows(); ++i)
            for (std::size_t j = 0; j < raw.cols(); ++j) raw(i, j) = noise(rng);
        for (std::size_t t = 0; t < 100; ++t)
            for (std::size_t j = 0; j < raw.cols(); ++j) raw(500 + t, j) = raw(t, j);
        BlockStore store(100, 3, 1.0);
        store.append_rows(raw.data(), raw.rows(), raw.cols());
        const auto hits = similar_range_search(store, 500, 599, 100, 1, 1.0);
        EXPECT(hits.size() == 1 && hits[0].window_start == 0 && std::fabs(hits[0].similarity - 1.0) <= 1e-10);
        EXPECT(similar_range_search(store, 20, 119, 5, 0, 1.0).empty());
        EXPECT_THROW(similar_range_search(store, 7, 7, 5, 2, 1.0), InvalidParameterError);
        EXPECT_THROW(similar_range_search(store, 10, 20, 0, 2, 1.0), InvalidParameterError);
    }
    // io_test.cpp SaveLoad: round trip, byte-identical re-save, bad magic
    {
        std::mt19937 rng(211);
        const auto raw = random_matrix(22, 4, rng);
        BlockStore store(5, 4, 0.95);
        store.append_rows(raw.data(), raw.rows(), raw.cols());
        const std::string path = "/tmp/zsvd_dropin_roundtrip.zsvd";
        save_store(store, path);
        auto loaded = load_store(path);
        EXPECT(loaded.total_rows() == 22 && loaded.sealed_count() == 4 && loaded.energy_threshold() == 0.95);
        const auto a = range_query(store, 3, 20).factors, b = range_query(loaded, 3, 20).factors;
        EXPECT(a.rank() == b.rank() && a.sigma == b.sigma);
        std::FILE* f = std::fopen(path.c_str(), "r+b");
        std::fputc('X', f);
        std::fclose(f);
        EXPECT_THROW(load_store(path), FormatError);
        std::remove(path.c_str());
    }
    // analysis_test.cpp ReconstructionError / NaiveRangeSvd
    {
        std::mt19937 rng(307);
        const auto raw = random_matrix(18, 4, rng);
        EXPECT(reconstruction_error(raw, thin_svd(raw)) <= 1e-12);
        const double inv = 1.0 / std::sqrt(2.0);
        const auto two = DenseMatrix::from_rows({{3 * inv, inv}, {3 * inv, -inv}});
        const auto t = truncate_rank(thin_svd(two), 0.9);
        EXPECT(t.rank() == 1 && std::fabs(reconstruction_error(two, t) - 0.1) <= 1e-12);
        EXPECT_THROW(reconstruction_error(DenseMatrix(5, 4), thin_svd(raw)), InvalidInputError);
        BlockStore store(5, 4, 1.0);
        store.append_rows(raw.data(), raw.rows(), raw.cols());
        const auto naive = naive_range_svd(store.snapshot(), 3, 12);
        EXPECT(naive.rank() == 4 && rel_fro(raw.middle_rows(3, 10), naive) <= 1e-8);
        EXPECT_THROW(naive_range_svd(store.snapshot(), 5, 18), RangeError);
    }
    // io_test.cpp CsvReader cases (:52-135), parsed on the GPU
    {
        auto write = [](const std::string& path, const std::string& text) {
            std::FILE* f = std::fopen(path.c_str(), "wb");
            std::fwrite(text.data(), 1, text.size(), f);
            std::fclose(f);
        };
        const std::string p = "/tmp/zsvd_dropin_csv.csv";
        write(p, "1,2\n3,4\n5,6\n");
        auto rows = read_csv_rows(p);
        EXPECT(rows.size() == 3 && rows[0] == (std::vector<double>{1, 2}) && rows[2] == (std::vector<double>{5, 6}));
        write(p, "a,b\n1,2\n");
        rows = read_csv_rows(p);
        EXPECT(rows.size() == 1 && rows[0] == (std::vector<double>{1, 2}));
        write(p, "1,x\n");
        try {
            read_csv_rows(p);
            EXPECT(false);
        } catch (const ParseError& e) {
            EXPECT(e.line() == 1);
        }
        write(p, "1,2\n3,4,5\n");
        try {
            read_csv_rows(p);
            EXPECT(false);
        } catch (const ParseError& e) {
            EXPECT(e.line() == 2 && std::string(e.what()) == "line 2: expected 2 columns, got 3");
        }
        write(p, "1,2,3\n");
        EXPECT_THROW(read_csv_rows(p, CsvOptions{2, false}), SchemaError);
        write(p, "time,s1,s2\n100,1.5,2.5\n200,3.5,4.5\n");
        rows = read_csv_rows(p, CsvOptions{std::nullopt, true});
        EXPECT(rows.size() == 2 && rows[1] == (std::vector<double>{3.5, 4.5}));
        write(p, "  1.5e2 , -3E-1 \n 2 , 0.25 \n");
        rows = read_csv_rows(p);
        EXPECT(rows.size() == 2 && rows[0][0] == 150.0 && rows[0][1] == -0.3);
        write(p, "1,2\n3,inf\n");
        CsvReader reader(p);
        EXPECT(reader.cols() == 0);
        auto first = reader.next();
        EXPECT(first && (*first)[1] == 2.0 && reader.cols() == 2);
        try {
            reader.next();
            EXPECT(false);
        } catch (const ParseError& e) {
            EXPECT(e.line() == 2);
        }
        EXPECT_THROW(CsvReader("/nonexistent/really_not_here.csv"), IoError);
        write(p, "");
        EXPECT_THROW(read_csv_matrix(p), InvalidInputError);
        // ingest: the CSV rows land in the store like the same rows appended directly
        std::mt19937 rng(401);
        const auto raw = random_matrix(300, 4, rng);
        std::string text;
        char buf[64];
        for (std::size_t i = 0; i < raw.rows(); ++i)
            for (std::size_t j = 0; j < raw.cols(); ++j) {
                std::snprintf(buf, sizeof buf, "%.17g%c", raw(i, j), j + 1 < raw.cols() ? ',' : '\n');
                text += buf;
            }
        write(p, text);
        {
            const auto m = read_csv_matrix(p);
            EXPECT(std::equal(m.values().begin(), m.values().end(), raw.values().begin(), raw.values().end()));
        }
        BlockStore a(100, 4, 0.98), b(100, 4, 0.98);
        EXPECT(append_csv(a, p) == 300);
        b.append_rows(raw.data(), raw.rows(), raw.cols());
        EXPECT(a.block(2).sigma == b.block(2).sigma);
        std::remove(p.c_str());
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
