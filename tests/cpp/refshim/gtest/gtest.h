// Minimal GoogleTest stand-in (test infrastructure): enough of the gtest API
// to compile the reference's own suites (/root/reference/proj/tests/*.cpp)
// unmodified against include/zsvd.hpp — GoogleTest is absent from this image.
// TEST, EXPECT_/ASSERT_ {EQ,NE,LT,LE,GT,GE,TRUE,FALSE,NEAR,DOUBLE_EQ,THROW,
// NO_THROW}, `<< message`, ::testing::Test::HasFailure(), --gtest_filter.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace testing {
namespace internal {
struct TestInfo {
    std::string suite, name;
    std::function<void()> body;
};
inline std::vector<TestInfo>& registry() {
    static std::vector<TestInfo> r;
    return r;
}
inline bool& current_failed() {
    static bool f = false;
    return f;
}
struct Registrar {
    Registrar(const char* suite, const char* name, std::function<void()> body) {
        registry().push_back({suite, name, std::move(body)});
    }
};
template <class T>
std::string show(const T& v) {
    if constexpr (requires(std::ostream& o, const T& x) { o << x; }) {
        std::ostringstream o;
        o.precision(17);
        o << v;
        return o.str();
    } else {
        return "<value>";
    }
}
struct Result {
    bool ok;
    std::string text;
};
#define ZSVD_GT_CMP(NAME, OP)                                                                          \
    template <class A, class B>                                                                        \
    Result NAME(const char* ea, const char* eb, const A& a, const B& b) {                              \
        if (a OP b) return {true, {}};                                                                 \
        return {false, std::string("expected ") + ea + " " #OP " " + eb + ", got " + show(a) + " vs " + show(b)}; \
    }
ZSVD_GT_CMP(cmp_eq, ==)
ZSVD_GT_CMP(cmp_ne, !=)
ZSVD_GT_CMP(cmp_lt, <)
ZSVD_GT_CMP(cmp_le, <=)
ZSVD_GT_CMP(cmp_gt, >)
ZSVD_GT_CMP(cmp_ge, >=)
#undef ZSVD_GT_CMP
inline Result cmp_near(const char* ea, const char* eb, double a, double b, double tol) {
    if (std::fabs(a - b) <= tol) return {true, {}};
    return {false, std::string("|") + ea + " - " + eb + "| <= " + show(tol) + " failed: " + show(a) + " vs " + show(b)};
}
inline Result cmp_double_eq(const char* ea, const char* eb, double a, double b) {
    auto key = [](double x) {
        int64_t i;
        std::memcpy(&i, &x, 8);
        return i < 0 ? INT64_MIN - i : i;
    };
    const int64_t d = key(a) - key(b);
    if (a == b || (d <= 4 && d >= -4)) return {true, {}};
    return {false, std::string(ea) + " == " + eb + " (4 ulps) failed: " + show(a) + " vs " + show(b)};
}
struct Message {
    std::ostringstream s;
    template <class T>
    Message& operator<<(const T& v) {
        s << v;
        return *this;
    }
};
struct Reporter {
    const char* file;
    int line;
    std::string text;
    void operator=(const Message& m) const {
        current_failed() = true;
        std::cout << file << ":" << line << ": Failure\n" << text;
        const std::string extra = m.s.str();
        if (!extra.empty()) std::cout << "\n" << extra;
        std::cout << std::endl;
    }
};
inline bool glob(const char* p, const char* s) {
    if (*p == 0) return *s == 0;
    if (*p == '*') return glob(p + 1, s) || (*s && glob(p, s + 1));
    return *s && (*p == '?' || *p == *s) && glob(p + 1, s + 1);
}
inline bool selected(const std::string& filter, const std::string& full) {
    if (filter.empty()) return true;
    const size_t dash = filter.find('-');
    const std::string pos = filter.substr(0, dash), neg = dash == std::string::npos ? "" : filter.substr(dash + 1);
    auto any = [&](const std::string& list) {
        size_t b = 0;
        while (b <= list.size()) {
            size_t e = list.find(':', b);
            if (e == std::string::npos) e = list.size();
            const std::string pat = list.substr(b, e - b);
            if (!pat.empty() && glob(pat.c_str(), full.c_str())) return true;
            b = e + 1;
        }
        return false;
    };
    return (pos.empty() || any(pos)) && !any(neg);
}
}  // namespace internal

class Test {
public:
    static bool HasFailure() { return internal::current_failed(); }
};

inline int RunAllTests(int argc, char** argv) {
    std::string filter;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "--gtest_filter=", 15) == 0) filter = argv[i] + 15;
    int run = 0;
    std::vector<std::string> failed;
    for (auto& t : internal::registry()) {
        const std::string full = t.suite + "." + t.name;
        if (!internal::selected(filter, full)) continue;
        std::cout << "[ RUN      ] " << full << std::endl;
        internal::current_failed() = false;
        try {
            t.body();
        } catch (const std::exception& e) {
            internal::current_failed() = true;
            std::cout << "uncaught exception: " << e.what() << std::endl;
        } catch (...) {
            internal::current_failed() = true;
            std::cout << "uncaught non-standard exception" << std::endl;
        }
        ++run;
        if (internal::current_failed()) failed.push_back(full);
        std::cout << (internal::current_failed() ? "[  FAILED  ] " : "[       OK ] ") << full << std::endl;
    }
    std::cout << "[==========] " << run << " tests ran.\n[  PASSED  ] " << run - failed.size() << " tests."
              << std::endl;
    for (auto& f : failed) std::cout << "[  FAILED  ] " << f << std::endl;
    return failed.empty() && run > 0 ? 0 : 1;
}
}  // namespace testing

#define ZSVD_GT_REPORT(res, fatal)                                                                      \
    if (const ::testing::internal::Result zsvd_gt_r_ = (res); zsvd_gt_r_.ok)                            \
        ;                                                                                               \
    else                                                                                                \
        fatal ::testing::internal::Reporter{__FILE__, __LINE__, zsvd_gt_r_.text} = ::testing::internal::Message()

#define ZSVD_GT_FATAL return
#define ZSVD_GT_NONFATAL

#define EXPECT_EQ(a, b) ZSVD_GT_REPORT(::testing::internal::cmp_eq(#a, #b, a, b), ZSVD_GT_NONFATAL)
#define EXPECT_NE(a, b) ZSVD_GT_REPORT(::testing::internal::cmp_ne(#a, #b, a, b), ZSVD_GT_NONFATAL)
#define EXPECT_LT(a, b) ZSVD_GT_REPORT(::testing::internal::cmp_lt(#a, #b, a, b), ZSVD_GT_NONFATAL)
#define EXPECT_LE(a, b) ZSVD_GT_REPORT(::testing::internal::cmp_le(#a, #b, a, b), ZSVD_GT_NONFATAL)
#define EXPECT_GT(a, b) ZSVD_GT_REPORT(::testing::internal::cmp_gt(#a, #b, a, b), ZSVD_GT_NONFATAL)
#define EXPECT_GE(a, b) ZSVD_GT_REPORT(::testing::internal::cmp_ge(#a, #b, a, b), ZSVD_GT_NONFATAL)
#define ASSERT_EQ(a, b) ZSVD_GT_REPORT(::testing::internal::cmp_eq(#a, #b, a, b), ZSVD_GT_FATAL)
#define ASSERT_NE(a, b) ZSVD_GT_REPORT(::testing::internal::cmp_ne(#a, #b, a, b), ZSVD_GT_FATAL)
#define ASSERT_LT(a, b) ZSVD_GT_REPORT(::testing::internal::cmp_lt(#a, #b, a, b), ZSVD_GT_FATAL)
#define ASSERT_LE(a, b) ZSVD_GT_REPORT(::testing::internal::cmp_le(#a, #b, a, b), ZSVD_GT_FATAL)
#define ASSERT_GT(a, b) ZSVD_GT_REPORT(::testing::internal::cmp_gt(#a, #b, a, b), ZSVD_GT_FATAL)
#define ASSERT_GE(a, b) ZSVD_GT_REPORT(::testing::internal::cmp_ge(#a, #b, a, b), ZSVD_GT_FATAL)
#define EXPECT_TRUE(c) ZSVD_GT_REPORT((::testing::internal::Result{bool(c), "expected true: " #c}), ZSVD_GT_NONFATAL)
#define EXPECT_FALSE(c) ZSVD_GT_REPORT((::testing::internal::Result{!bool(c), "expected false: " #c}), ZSVD_GT_NONFATAL)
#define ASSERT_TRUE(c) ZSVD_GT_REPORT((::testing::internal::Result{bool(c), "expected true: " #c}), ZSVD_GT_FATAL)
#define ASSERT_FALSE(c) ZSVD_GT_REPORT((::testing::internal::Result{!bool(c), "expected false: " #c}), ZSVD_GT_FATAL)
#define EXPECT_NEAR(a, b, t) ZSVD_GT_REPORT(::testing::internal::cmp_near(#a, #b, a, b, t), ZSVD_GT_NONFATAL)
#define ASSERT_NEAR(a, b, t) ZSVD_GT_REPORT(::testing::internal::cmp_near(#a, #b, a, b, t), ZSVD_GT_FATAL)
#define EXPECT_DOUBLE_EQ(a, b) ZSVD_GT_REPORT(::testing::internal::cmp_double_eq(#a, #b, a, b), ZSVD_GT_NONFATAL)
#define ASSERT_DOUBLE_EQ(a, b) ZSVD_GT_REPORT(::testing::internal::cmp_double_eq(#a, #b, a, b), ZSVD_GT_FATAL)

#define ZSVD_GT_THROW(stmt, type, fatal)                                                                \
    ZSVD_GT_REPORT(([&]() -> ::testing::internal::Result {                                              \
                       try {                                                                            \
                           stmt;                                                                        \
                       } catch (const type&) {                                                          \
                           return {true, {}};                                                           \
                       } catch (const std::exception& e) {                                              \
                           return {false, std::string(#stmt " threw another type: ") + e.what()};       \
                       } catch (...) {                                                                  \
                           return {false, #stmt " threw another type"};                                 \
                       }                                                                                \
                       return {false, #stmt " did not throw " #type};                                   \
                   }()),                                                                                \
                   fatal)
#define EXPECT_THROW(stmt, type) ZSVD_GT_THROW(stmt, type, ZSVD_GT_NONFATAL)
#define ASSERT_THROW(stmt, type) ZSVD_GT_THROW(stmt, type, ZSVD_GT_FATAL)
#define ZSVD_GT_NO_THROW(stmt, fatal)                                                                   \
    ZSVD_GT_REPORT(([&]() -> ::testing::internal::Result {                                              \
                       try {                                                                            \
                           stmt;                                                                        \
                       } catch (const std::exception& e) {                                              \
                           return {false, std::string(#stmt " threw: ") + e.what()};                    \
                       } catch (...) {                                                                  \
                           return {false, #stmt " threw"};                                              \
                       }                                                                                \
                       return {true, {}};                                                               \
                   }()),                                                                                \
                   fatal)
#define EXPECT_NO_THROW(stmt) ZSVD_GT_NO_THROW(stmt, ZSVD_GT_NONFATAL)
#define ASSERT_NO_THROW(stmt) ZSVD_GT_NO_THROW(stmt, ZSVD_GT_FATAL)

#define FAIL() return ::testing::internal::Reporter{__FILE__, __LINE__, "Failed"} = ::testing::internal::Message()
#define ADD_FAILURE() ::testing::internal::Reporter{__FILE__, __LINE__, "Failed"} = ::testing::internal::Message()

#define TEST(suite, name)                                                                               \
    static void zsvd_gt_##suite##_##name();                                                             \
    static ::testing::internal::Registrar zsvd_gt_reg_##suite##_##name(#suite, #name,                   \
                                                                       zsvd_gt_##suite##_##name);       \
    static void zsvd_gt_##suite##_##name()
