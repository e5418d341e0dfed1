// zsvd_commands.hpp — the two command entry points of the reference's
// commands.hpp that drive the hot path directly, over the drop-in API
// (zsvd.hpp): cmd_bench (commands.hpp:231-275, the query-latency protocol)
// and cmd_search (commands.hpp:209-229).  The rest of the CLI (ingest, query,
// verify, argument parsing) is out of scope.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <fstream>
#include <optional>
#include <ostream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "zsvd.hpp"

namespace rangesvd {
namespace detail {
/// 17 significant digits (commands.hpp:33-37).
inline std::string format_value(double v) {
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    return buf;
}
template <typename Fn>
double timed_ms(Fn&& fn) {
    const auto begin = std::chrono::steady_clock::now();
    fn();
    const auto end = std::chrono::steady_clock::now();
    return std::chrono::duration<double, std::milli>(end - begin).count();
}
/// Exit codes (commands.hpp:79-93): 1 bad parameter, 2 any other error.
template <typename Fn>
int run_command(std::ostream& err, Fn&& fn) {
    try {
        return fn();
    } catch (const InvalidParameterError& e) {
        err << "error: " << e.what() << "\n";
        return 1;
    } catch (const Error& e) {
        err << "error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        err << "error: " << e.what() << "\n";
        return 2;
    }
}
}  // namespace detail

struct SearchOptions {
    std::string store;
    std::size_t start = 0;
    std::size_t end = 0;
    std::size_t stride = 500;
    std::size_t top_n = 2;
    std::optional<double> xi;
};

/// "window_start,similarity" per hit (commands.hpp:219-229).
inline int cmd_search(const SearchOptions& opt, std::ostream& out, std::ostream& err) {
    return detail::run_command(err, [&]() -> int {
        const BlockStore store = load_store(opt.store);
        const double xi = opt.xi.value_or(store.energy_threshold());
        const auto hits = similar_range_search(store, opt.start, opt.end, opt.stride, opt.top_n, xi);
        for (const SearchHit& hit : hits) out << hit.window_start << "," << detail::format_value(hit.similarity) << "\n";
        return 0;
    });
}

struct BenchOptions {
    std::string store;
    std::vector<std::size_t> lengths;
    std::size_t reps = 5;
    std::uint64_t seed = 42;
    std::optional<double> xi;
};

/// "length,median_ms" per length (commands.hpp:241-275): range_query at
/// offsets drawn from one seeded sequence per length, answer on the host.
inline int cmd_bench(const BenchOptions& opt, std::ostream& out, std::ostream& err) {
    return detail::run_command(err, [&]() -> int {
        if (opt.reps < 1) throw InvalidParameterError("--reps must be at least 1");
        if (opt.lengths.empty()) throw InvalidParameterError("--lengths must name at least one query length");
        const BlockStore store = load_store(opt.store);
        const StoreSnapshot snap = store.snapshot();
        const double xi = opt.xi.value_or(store.energy_threshold());
        for (std::size_t length : opt.lengths) {
            if (length < 1 || length > snap.total_rows)
                throw RangeError("query length " + std::to_string(length) + " exceeds the stored stream");
            std::mt19937_64 rng(opt.seed);
            std::uniform_int_distribution<std::size_t> offsets(0, snap.total_rows - length);
            std::vector<double> times;
            times.reserve(opt.reps);
            for (std::size_t rep = 0; rep < opt.reps; ++rep) {
                const std::size_t first = offsets(rng);
                times.push_back(detail::timed_ms([&] { (void)range_query(snap, first, first + length - 1, xi); }));
            }
            std::sort(times.begin(), times.end());
            const std::size_t mid = times.size() / 2;
            const double median = times.size() % 2 == 1 ? times[mid] : 0.5 * (times[mid - 1] + times[mid]);
            out << length << "," << detail::format_value(median) << "\n";
        }
        return 0;
    });
}
}  // namespace rangesvd
