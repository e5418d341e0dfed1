// Decimal text -> double exactly as the reference's CSV cell parser decides it
// (csv.hpp:42-50: trimmed cell, std::from_chars with chars_format::general,
// the whole cell consumed, then std::isfinite at :110-112).  Compiles for the
// device (csv_ingest.cu) and for the host (tests/cpp/csv_number_fuzz.cpp, which
// checks it against std::from_chars on millions of strings).
//
// Grammar accepted by from_chars (libstdc++ 13, measured here):
//   '-'? ( digits ('.' digits?)? | '.' digits ) ([eE] [+-]? digits)?
//   '-'? ( inf | infinity | nan | nan '(' [A-Za-z0-9_]* ')' )   (case-insensitive)
// A result that overflows, or a non-zero value that rounds to zero, is
// errc::result_out_of_range, which the reference reports as "not numeric".
//
// Conversion: Clinger's exact fast path (w <= 2^53, |q| <= 22); otherwise the
// 19 leading significant digits times a 128-bit normalised power of five
// (pow5_table.inc) gives the value within a proven error bound; when a
// rounding boundary lies inside that bound, an exact big-integer comparison
// with the halfway point decides (slow path, up to 800 significant digits,
// which suffices because a double's halfway point has at most 767).
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define ZCSV_HD __host__ __device__ __forceinline__
#define ZCSV_HD_NOINLINE __host__ __device__ __noinline__
#else
#define ZCSV_HD inline
#define ZCSV_HD_NOINLINE inline
#endif

namespace zcsv {

enum CellKind : int { kOk = 0, kNonFinite = 1, kNotNumeric = 2 };

ZCSV_HD bool is_ws(unsigned c) { return c == ' ' || c == '\t' || c == '\r' || c == '\f' || c == '\v'; }
ZCSV_HD bool is_digit(unsigned c) { return c - '0' < 10u; }

ZCSV_HD uint64_t mulhi(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

ZCSV_HD int clz64(uint64_t x) {
#ifdef __CUDA_ARCH__
    return __clzll((long long)x);
#else
    return __builtin_clzll(x);
#endif
}

ZCSV_HD double bits_to_double(uint64_t b) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)b);
#else
    double d;
    __builtin_memcpy(&d, &b, 8);
    return d;
#endif
}

// ---- exact slow path ---------------------------------------------------------
struct Big {
    static constexpr int kLimbs = 64;  // 4096 bits; the comparisons below need < 2800
    uint64_t d[kLimbs];
    int n;
};

ZCSV_HD void big_set(Big& a, uint64_t v) {
    a.n = v ? 1 : 0;
    a.d[0] = v;
}

ZCSV_HD void big_mul_add(Big& a, uint64_t m, uint64_t add) {
    uint64_t carry = add;
    for (int i = 0; i < a.n; ++i) {
        const uint64_t lo = a.d[i] * m;
        const uint64_t hi = mulhi(a.d[i], m);
        const uint64_t s = lo + carry;
        carry = hi + (s < lo);
        a.d[i] = s;
    }
    if (carry && a.n < Big::kLimbs) a.d[a.n++] = carry;
}

ZCSV_HD void big_mul_pow5(Big& a, int64_t e) {
    const uint64_t p27 = 7450580596923828125ull;  // 5^27
    while (e >= 27) {
        big_mul_add(a, p27, 0);
        e -= 27;
    }
    uint64_t p = 1;
    while (e-- > 0) p *= 5;
    if (p != 1) big_mul_add(a, p, 0);
}

ZCSV_HD void big_shl(Big& a, int64_t bits) {
    if (a.n == 0 || bits <= 0) return;
    const int limbs = (int)(bits >> 6), sh = (int)(bits & 63);
    int n = a.n + limbs + 1;
    if (n > Big::kLimbs) n = Big::kLimbs;
    for (int i = n - 1; i >= 0; --i) {
        const int src = i - limbs;
        uint64_t v = 0;
        if (src >= 0 && src < a.n) v = a.d[src] << sh;
        if (sh && src - 1 >= 0 && src - 1 < a.n) v |= a.d[src - 1] >> (64 - sh);
        a.d[i] = v;
    }
    a.n = n;
    while (a.n > 0 && a.d[a.n - 1] == 0) --a.n;
}

ZCSV_HD int big_cmp(const Big& a, const Big& b) {
    if (a.n != b.n) return a.n < b.n ? -1 : 1;
    for (int i = a.n - 1; i >= 0; --i)
        if (a.d[i] != b.d[i]) return a.d[i] < b.d[i] ? -1 : 1;
    return 0;
}

// Rounds the decimal in s[0, n) (grammar already checked) between the doubles
// m * 2^lsb and (m + 1) * 2^lsb: returns m or m + 1 (ties to even).
ZCSV_HD_NOINLINE uint64_t slow_round(const unsigned char* s, int64_t n, uint64_t m, int64_t lsb) {
    Big A, B;
    big_set(A, 0);
    int64_t i = (s[0] == '-') ? 1 : 0;
    int nsig = 0;
    int64_t qd = 0;
    bool tail = false;
    uint64_t chunk = 0, scale = 1;
    auto digit = [&](unsigned d, bool frac) {
        if (nsig == 0 && d == 0) {
            if (frac) --qd;
            return;
        }
        if (nsig < 800) {
            chunk = chunk * 10 + d;
            scale *= 10;
            if (scale == 10000000000000000000ull) {
                big_mul_add(A, scale, chunk);
                if (A.n == 0 && chunk) big_set(A, chunk);
                chunk = 0;
                scale = 1;
            }
            ++nsig;
            if (frac) --qd;
        } else {
            if (d) tail = true;
            if (!frac) ++qd;
        }
    };
    while (i < n && is_digit(s[i])) digit(s[i++] - '0', false);
    if (i < n && s[i] == '.') {
        ++i;
        while (i < n && is_digit(s[i])) digit(s[i++] - '0', true);
    }
    if (scale != 1) {
        if (A.n == 0) big_set(A, chunk);
        else big_mul_add(A, scale, chunk);
    }
    if (i < n && (s[i] | 0x20) == 'e') {
        ++i;
        bool eneg = false;
        if (s[i] == '+' || s[i] == '-') eneg = s[i++] == '-';
        int64_t ev = 0;
        while (i < n && is_digit(s[i])) {
            if (ev < 1000000000000000ll) ev = ev * 10 + (s[i] - '0');
            ++i;
        }
        qd += eneg ? -ev : ev;
    }
    // compare D * 10^qd with (2m + 1) * 2^(lsb - 1)
    big_set(B, 2 * m + 1);
    int64_t a2 = qd, b2 = lsb - 1;
    if (qd >= 0) big_mul_pow5(A, qd);
    else big_mul_pow5(B, -qd);
    const int64_t mn = a2 < b2 ? a2 : b2;
    big_shl(A, a2 - mn);
    big_shl(B, b2 - mn);
    int c = big_cmp(A, B);
    if (c == 0 && tail) c = 1;
    if (c > 0) return m + 1;
    if (c < 0) return m;
    return m + (m & 1);
}

// ---- the cell parser -----------------------------------------------------------
// s[0, n) is the trimmed cell.  pow5 = kPow5Mant (hi, lo pairs), pexp = kPow5Exp,
// both indexed by q - ZSVD_POW5_QMIN.
ZCSV_HD int parse_cell(const unsigned char* s, int64_t n, const uint64_t* pow5, const short* pexp, double* out) {
    if (n <= 0) return kNotNumeric;
    int64_t i = 0;
    const bool neg = s[0] == '-';
    if (neg) i = 1;
    if (i >= n) return kNotNumeric;
    const unsigned c0 = s[i] | 0x20;
    if (c0 == 'i' || c0 == 'n') {
        auto match = [&](const char* w, int len) {
            if (i + len > n) return false;
            for (int k = 0; k < len; ++k)
                if ((unsigned)(s[i + k] | 0x20) != (unsigned)w[k]) return false;
            return true;
        };
        if (c0 == 'i') {
            if (match("infinity", 8) && i + 8 == n) return kNonFinite;
            if (match("inf", 3) && i + 3 == n) return kNonFinite;
            return kNotNumeric;
        }
        if (!match("nan", 3)) return kNotNumeric;
        if (i + 3 == n) return kNonFinite;
        if (s[i + 3] != '(') return kNotNumeric;
        int64_t j = i + 4;
        while (j < n) {
            const unsigned c = s[j];
            if (!(is_digit(c) || ((c | 0x20) - 'a' < 26u) || c == '_')) break;
            ++j;
        }
        return (j == n - 1 && s[j] == ')') ? kNonFinite : kNotNumeric;
    }
    // mantissa
    uint64_t w = 0;
    int nsig = 0;
    int64_t q = 0;
    bool any = false, trunc = false;
    while (i < n && is_digit(s[i])) {
        const unsigned d = s[i++] - '0';
        any = true;
        if (nsig == 0 && d == 0) continue;
        if (nsig < 19) {
            w = w * 10 + d;
            ++nsig;
        } else {
            ++q;
            if (d) trunc = true;
        }
    }
    if (i < n && s[i] == '.') {
        ++i;
        while (i < n && is_digit(s[i])) {
            const unsigned d = s[i++] - '0';
            any = true;
            if (nsig == 0 && d == 0) {
                --q;
                continue;
            }
            if (nsig < 19) {
                w = w * 10 + d;
                ++nsig;
                --q;
            } else if (d) {
                trunc = true;
            }
        }
    }
    if (!any) return kNotNumeric;
    if (i < n && (s[i] | 0x20) == 'e') {
        int64_t j = i + 1;
        bool eneg = false;
        if (j < n && (s[j] == '+' || s[j] == '-')) eneg = s[j++] == '-';
        if (j >= n || !is_digit(s[j])) return kNotNumeric;  // from_chars stops before the 'e'
        int64_t ev = 0;
        while (j < n && is_digit(s[j])) {
            if (ev < 1000000000000000ll) ev = ev * 10 + (s[j] - '0');
            ++j;
        }
        q += eneg ? -ev : ev;
        i = j;
    }
    if (i != n) return kNotNumeric;
    const uint64_t sign = neg ? (1ull << 63) : 0;
    if (w == 0) {  // every digit zero
        *out = bits_to_double(sign);
        return kOk;
    }
    if (!trunc && w <= (1ull << 53) && q >= -22 && q <= 22) {
        // 10^|q| by squaring: every partial power <= 10^22 is an exact double
        double p = 1.0, b = 10.0;
        for (int e = (int)(q < 0 ? -q : q); e; e >>= 1, b *= b)
            if (e & 1) p *= b;
        double v = (double)w;
        v = q < 0 ? v / p : v * p;
        *out = neg ? -v : v;
        return kOk;
    }
    if (q < -342 || q > 308) return kNotNumeric;  // |value| < 1e-324 rounds to 0; >= 1e309 overflows
    const int lz = clz64(w);
    const uint64_t wn = w << lz;
    const int qi = (int)(q + 342);
    const uint64_t thi = pow5[2 * qi], tlo = pow5[2 * qi + 1];
    const uint64_t l1 = wn * tlo, h1 = mulhi(wn, tlo);
    const uint64_t l2 = wn * thi, h2 = mulhi(wn, thi);
    const uint64_t mid = l2 + h1;
    const uint64_t top = h2 + (mid < l2);
    uint64_t phi, plo;
    int64_t e;
    if (top >> 63) {
        phi = top;
        plo = mid;
        e = 191 + pexp[qi] + q - lz;
    } else {
        phi = (top << 1) | (mid >> 63);
        plo = (mid << 1) | (l1 >> 63);
        e = 190 + pexp[qi] + q - lz;
    }
    // exact value in [P, P + delta) units of P's last bit; delta = 4 or 2^70
    if (e > 1023) return kNotNumeric;
    const int nm = e >= -1022 ? 53 : (int)(e + 1075);
    if (nm < 0) return kNotNumeric;  // below 2^-1075: rounds to zero
    const int sb = 128 - nm;  // bits below the mantissa, 75 .. 128
    uint64_t m = sb >= 128 ? 0 : phi >> (sb - 64);
    const uint64_t low_hi = sb >= 128 ? phi : phi & ((1ull << (sb - 64)) - 1), low_lo = plo;
    const uint64_t half_hi = 1ull << (sb - 65);
    const bool above = low_hi > half_hi || (low_hi == half_hi && low_lo > 0);
    bool ambiguous = false;
    if (!above) {
        // diff = half - low (128-bit), ambiguous when diff < delta
        const uint64_t dlo = 0 - low_lo;
        const uint64_t dhi = half_hi - low_hi - (low_lo != 0);
        ambiguous = trunc ? (dhi < (1ull << 6)) : (dhi == 0 && dlo < 4);
    }
    if (ambiguous) m = slow_round(s, n, m, e - 127 + sb);
    else if (above) m += 1;
    uint64_t bits = e >= -1022 ? ((uint64_t)(e + 1023) << 52) + (m - (1ull << 52)) : m;
    if (bits == 0 || bits >= 0x7FF0000000000000ull) return kNotNumeric;
    *out = bits_to_double(bits | sign);
    return kOk;
}

// Trims " \t\r\f\v" (csv.hpp:31-39) and parses.
ZCSV_HD int parse_raw_cell(const unsigned char* b, const unsigned char* e, const uint64_t* pow5, const short* pexp,
                           double* out) {
    while (b < e && is_ws(*b)) ++b;
    while (e > b && is_ws(e[-1])) --e;
    return parse_cell(b, e - b, pow5, pexp, out);
}

}  // namespace zcsv
