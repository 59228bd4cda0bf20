// integration/doctest.h -- a minimal doctest-compatible shim (TEST_CASE, CHECK, CHECK_FALSE,
// REQUIRE, CHECK_THROWS, CHECK_THROWS_AS, doctest::Approx) so the reference's own unit suites
// (proj/tests/test_*.cpp) build without the vendored doctest (absent from this image,
// proj/README.md:226).  Not the doctest library: it implements only the
// subset those suites use, with doctest's meaning (a failed REQUIRE ends the test case, CHECKs
// continue).  Define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN in exactly one translation unit.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) { eps = e; return *this; }
    double value, eps = 1.19209290e-05 * 100;  // doctest's default: float epsilon * 100
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.value) < b.eps * (1.0 + std::fmax(std::fabs(a), std::fabs(b.value)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
};
namespace detail {
struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Reg {
    Reg(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct RequireFailed {};
inline int& failures() {
    static int n = 0;
    return n;
}
inline void fail(const char* kind, const char* expr, const char* file, int line) {
    ++failures();
    std::printf("  %s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC(fn, name)                                                                           \
    static void fn();                                                                                  \
    static doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);                  \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define CHECK(...) \
    do { if (!(__VA_ARGS__)) doctest::detail::fail("CHECK", #__VA_ARGS__, __FILE__, __LINE__); } while (0)
#define CHECK_FALSE(...) \
    do { if ((__VA_ARGS__)) doctest::detail::fail("CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__); } while (0)
#define REQUIRE(...)                                                                                   \
    do {                                                                                               \
        if (!(__VA_ARGS__)) {                                                                          \
            doctest::detail::fail("REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                        \
            throw doctest::detail::RequireFailed{};                                                    \
        }                                                                                              \
    } while (0)
#define CHECK_THROWS(...)                                                                              \
    do {                                                                                               \
        bool thrown_ = false;                                                                          \
        try { (void)(__VA_ARGS__); } catch (...) { thrown_ = true; }                                   \
        if (!thrown_) doctest::detail::fail("CHECK_THROWS", #__VA_ARGS__, __FILE__, __LINE__);         \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                     \
    do {                                                                                               \
        bool ok_ = false;                                                                              \
        try { (void)(expr); } catch (const __VA_ARGS__&) { ok_ = true; } catch (...) {}                \
        if (!ok_) doctest::detail::fail("CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0, n = 0;
    for (const auto& tc : doctest::detail::registry()) {
        const int before = doctest::detail::failures();
        bool threw = false;
        std::string what;
        try {
            tc.fn();
        } catch (const doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            threw = true;
            what = e.what();
        } catch (...) {
            threw = true;
            what = "unknown exception";
        }
        ++n;
        const bool ok = !threw && doctest::detail::failures() == before;
        if (threw) std::printf("  unexpected exception: %s\n", what.c_str());
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", tc.name);
        if (!ok) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", n, n - failed_cases, failed_cases);
    return failed_cases ? 1 : 0;
}
#endif
