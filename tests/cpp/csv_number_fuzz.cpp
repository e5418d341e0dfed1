// Host-side fuzz of the CSV cell parser (csrc/csv_number.cuh, the code the
// GPU kernels run) against the reference's own rule: std::from_chars over the
// trimmed cell, whole cell consumed, std::isfinite (csv.hpp:42-50, :106-112).
// Usage: csv_number_fuzz [iterations] [seed]; exits non-zero on a mismatch.
#include <charconv>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../paper_1805_00754_b200/csrc/csv_number.cuh"
#include "../../paper_1805_00754_b200/csrc/pow5_table.inc"

static int reference_kind(const std::string& cell, double& v) {
    const char* b = cell.data();
    const char* e = b + cell.size();
    while (b < e && zcsv::is_ws((unsigned char)*b)) ++b;
    while (e > b && zcsv::is_ws((unsigned char)e[-1])) --e;
    if (b == e) return zcsv::kNotNumeric;
    auto [p, ec] = std::from_chars(b, e, v);
    if (ec != std::errc() || p != e) return zcsv::kNotNumeric;
    return std::isfinite(v) ? zcsv::kOk : zcsv::kNonFinite;
}

static int mine(const std::string& cell, double& v) {
    const auto* b = (const unsigned char*)cell.data();
    return zcsv::parse_raw_cell(b, b + cell.size(), (const uint64_t*)kPow5Mant, kPow5Exp, &v);
}

static std::mt19937_64 rng;
static uint64_t r64() { return rng(); }
static int rint_(int lo, int hi) { return lo + (int)(r64() % (uint64_t)(hi - lo + 1)); }

static std::string digits(int n) {
    std::string s;
    for (int i = 0; i < n; ++i) s += char('0' + rint_(0, 9));
    return s;
}

static std::string fmt(const char* f, double x) {
    char buf[64];
    std::snprintf(buf, sizeof buf, f, x);
    return buf;
}

// exact decimal expansion of a double's halfway point to its successor, as text
static std::string halfway_text(double x, int cut) {
    // x = m * 2^e2; halfway = (2m + 1) * 2^(e2 - 1), written exactly in decimal
    int e2;
    double fr = std::frexp(std::fabs(x), &e2);
    uint64_t m = (uint64_t)std::ldexp(fr, 53);
    e2 -= 53;
    if (m < (1ull << 52)) return "1";
    uint64_t H = 2 * m + 1;
    int t = e2 - 1;
    // decimal digits of H * 2^t: if t >= 0 integer; else H * 5^-t / 10^-t
    std::vector<int> big;  // little-endian base-10 digits
    for (uint64_t h = H; h; h /= 10) big.push_back((int)(h % 10));
    auto mul = [&](int f) {
        int carry = 0;
        for (auto& d : big) {
            int v = d * f + carry;
            d = v % 10;
            carry = v / 10;
        }
        while (carry) {
            big.push_back(carry % 10);
            carry /= 10;
        }
    };
    int frac = 0;
    if (t >= 0) {
        for (int i = 0; i < t; ++i) mul(2);
    } else {
        for (int i = 0; i < -t; ++i) mul(5);
        frac = -t;
    }
    std::string s;
    for (int i = (int)big.size() - 1; i >= 0; --i) s += char('0' + big[i]);
    std::string out;
    if (frac >= (int)s.size()) out = "0." + std::string(frac - s.size(), '0') + s;
    else if (frac == 0) out = s;
    else out = s.substr(0, s.size() - frac) + "." + s.substr(s.size() - frac);
    if (cut > 0 && (int)out.size() > cut) {
        out.resize(cut);  // slightly below the halfway point
    } else if (cut < 0) {
        out += "0000000000001";  // slightly above
    }
    return (x < 0 ? "-" : "") + out;
}

static std::string random_cell() {
    const int kind = rint_(0, 19);
    double x;
    uint64_t b;
    switch (kind) {
    case 0: {  // random bits, %.17g
        do {
            b = r64();
            std::memcpy(&x, &b, 8);
        } while (!std::isfinite(x));
        return fmt("%.17g", x);
    }
    case 1: return fmt("%.17g", std::ldexp((double)(r64() >> 11), -53) * 2 - 1);  // uniform(-1, 1)
    case 2: return fmt(rint_(0, 1) ? "%.15e" : "%.6g", (double)(int64_t)r64() * std::pow(10.0, rint_(-30, 30)));
    case 3: return digits(rint_(1, 30)) + (rint_(0, 1) ? "." + digits(rint_(0, 30)) : "");
    case 4: return digits(rint_(1, 25)) + "e" + std::to_string(rint_(-360, 330));
    case 5: return "0." + std::string(rint_(0, 40), '0') + digits(rint_(1, 25)) + "e-" + std::to_string(rint_(250, 330));
    case 6: {  // halfway points, exact / just below / just above
        b = r64() & 0x7FFFFFFFFFFFFFFFull;
        std::memcpy(&x, &b, 8);
        if (!std::isfinite(x)) x = 1.5;
        const int mode = rint_(0, 2);
        return halfway_text(x, mode == 0 ? 0 : mode == 1 ? rint_(20, 60) : -1);
    }
    case 7: {  // subnormal / underflow neighbourhood
        return digits(rint_(1, 20)) + "e-" + std::to_string(rint_(300, 345));
    }
    case 8: return digits(rint_(1, 20)) + "e" + std::to_string(rint_(280, 310));
    case 9: {  // integers around 2^53 .. 2^64
        uint64_t v = (1ull << rint_(52, 63)) + (r64() % 5000) - 2500;
        return std::to_string(v);
    }
    case 10: {  // syntax noise
        static const char* pieces[] = {"-", "+", ".", "e", "E", "1", "0", "9", "inf", "nan", "(", ")",
                                       "x", "_", " ", "\t", "infinity", "NaN", "INF", "e+", "e-", "a"};
        std::string s;
        int n = rint_(1, 6);
        for (int i = 0; i < n; ++i) s += pieces[rint_(0, 21)];
        return s;
    }
    case 11: {
        static const char* fixed[] = {"inf", "-inf", "Infinity", "-INFINITY", "nan", "-nan", "nan()", "nan(abc_1)",
                                      "nan(a-b)", "nan(", "infx", "infinit", "1e", "1e+", ".5", "5.", ".", "-.",
                                      "-0", "0e99999999999999999999", "1e99999999999999999999", "1e-400", "+1",
                                      "1.7976931348623157e308", "1.7976931348623158e308", "1.7976931348623159e308",
                                      "2.4703282292062327e-324", "2.4703282292062328e-324", "4.9406564584124654e-324",
                                      "2.2250738585072011e-308", "2.2250738585072014e-308", "9007199254740993",
                                      "  7 ", "\t-3.5e2\r", "1 2", "", "  ", "0x10", "1_0", "-.5e-2", "00012"};
        return fixed[rint_(0, 40)];
    }
    case 12: return std::string(rint_(0, 2), ' ') + fmt("%.17g", std::ldexp((double)(r64() >> 11), rint_(-1100, 1000))) +
                    std::string(rint_(0, 2), '\t');
    case 13: return "-" + digits(rint_(0, 3)) + "." + digits(rint_(0, 400));
    case 14: return digits(rint_(700, 900)) + "e-" + std::to_string(rint_(700, 1200));
    case 15: {  // exactly representable values written with many digits
        b = r64() & 0x7FFFFFFFFFFFFFFFull;
        std::memcpy(&x, &b, 8);
        if (!std::isfinite(x)) x = 3.0;
        return fmt("%.40e", x);
    }
    case 16: return fmt("%.16g", std::ldexp((double)(r64() >> 11), rint_(-60, 60)));
    case 17: return fmt("%.17g", std::ldexp((double)(r64() >> 11), rint_(-1074 - 53, -1000)));
    case 18: return digits(19) + "." + digits(rint_(1, 5)) + "e" + std::to_string(rint_(-30, 30));
    default: return fmt("%.20g", (double)r64() / (double)(r64() | 1));
    }
}

int main(int argc, char** argv) {
    const long iters = argc > 1 ? std::atol(argv[1]) : 2000000;
    rng.seed(argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 12345);
    long bad = 0, counts[3] = {0, 0, 0};
    for (long it = 0; it < iters; ++it) {
        const std::string cell = random_cell();
        double a = -7.0, b = -7.0;
        const int ka = reference_kind(cell, a), kb = mine(cell, b);
        counts[ka]++;
        bool ok = ka == kb;
        if (ok && ka == zcsv::kOk) ok = std::memcmp(&a, &b, 8) == 0;
        if (!ok && bad++ < 20) {
            uint64_t ba, bb;
            std::memcpy(&ba, &a, 8);
            std::memcpy(&bb, &b, 8);
            std::printf("MISMATCH '%s': ref kind %d bits %016" PRIx64 ", mine kind %d bits %016" PRIx64 "\n",
                        cell.substr(0, 120).c_str(), ka, ba, kb, bb);
        }
    }
    std::printf("%ld cells (ok %ld, non-finite %ld, not numeric %ld): %ld mismatches\n", iters, counts[0], counts[1],
                counts[2], bad);
    return bad ? 1 : 0;
}
