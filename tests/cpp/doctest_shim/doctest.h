// doctest.h — a from-scratch subset of the doctest API (TEST_CASE, CHECK, CHECK_FALSE,
// REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, doctest::Approx) so the reference's own unit
// tests (/root/reference/proj/tests/test_{renderer,crowd,lod,metrics}.cpp, unmodified)
// compile against this repo's drop-in headers and run on the B200 (tests/test_ref_api.py).
// The reference vendors the real doctest under proj/vendor, which is absent here.
// TEST INFRASTRUCTURE ONLY.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    Approx& scale(double s) {
        scl = s;
        return *this;
    }
    double value;
    double eps = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
    double scl = 1.0;
    bool matches(double lhs) const {  // doctest's rule: |lhs - v| < eps * (scale + max(|lhs|, |v|))
        return std::fabs(lhs - value) < eps * (scl + std::max(std::fabs(lhs), std::fabs(value)));
    }
};
template <typename T> bool operator==(const T& lhs, const Approx& rhs) { return rhs.matches(static_cast<double>(lhs)); }
template <typename T> bool operator==(const Approx& lhs, const T& rhs) { return lhs.matches(static_cast<double>(rhs)); }
template <typename T> bool operator!=(const T& lhs, const Approx& rhs) { return !rhs.matches(static_cast<double>(lhs)); }
template <typename T> bool operator!=(const Approx& lhs, const T& rhs) { return !lhs.matches(static_cast<double>(rhs)); }
template <typename T> bool operator<=(const T& lhs, const Approx& rhs) { return lhs < rhs.value || rhs.matches(lhs); }
template <typename T> bool operator>=(const T& lhs, const Approx& rhs) { return lhs > rhs.value || rhs.matches(lhs); }

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

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct RequireFailed {};

inline int& failures() {
    static int f = 0;
    return f;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    if (ok) return;
    ++failures();
    std::fprintf(stdout, "  FAILED %s( %s ) at %s:%d\n", kind, expr, file, line);
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_(name, fn)                                                            \
    static void fn();                                                                           \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);   \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_(name, DOCTEST_CAT(doctest_case_, __COUNTER__))

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                            \
    do {                                                                                        \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                \
        ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);    \
        if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                             \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                             \
    do {                                                                                        \
        bool doctest_ok_ = false;                                                               \
        try {                                                                                   \
            static_cast<void>(expr);                                                            \
        } catch (const type&) {                                                                 \
            doctest_ok_ = true;                                                                 \
        } catch (...) {                                                                         \
        }                                                                                       \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #type, __FILE__, __LINE__); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                     \
    do {                                                                                        \
        bool doctest_ok_ = true;                                                                \
        try {                                                                                   \
            static_cast<void>(expr);                                                            \
        } catch (...) {                                                                         \
            doctest_ok_ = false;                                                                \
        }                                                                                       \
        ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__);     \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <exception>
// Runs every registered case (or those whose name contains argv[1]); one line per case,
// "ok" or "FAIL", then a summary; exit status 1 on any failed assertion or exception.
int main(int argc, char** argv) {
    const char* filter = argc > 1 ? argv[1] : nullptr;
    int cases = 0, failed_cases = 0;
    for (const auto& tc : ::doctest::detail::registry()) {
        if (filter && !std::strstr(tc.name, filter)) continue;
        ++cases;
        const int before = ::doctest::detail::failures();
        bool threw = false;
        std::string what;
        try {
            tc.fn();
        } catch (const ::doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            threw = true;
            what = e.what();
        } catch (...) {
            threw = true;
            what = "unknown exception";
        }
        const bool ok = !threw && ::doctest::detail::failures() == before;
        if (threw) ++::doctest::detail::failures();
        if (!ok) ++failed_cases;
        std::fprintf(stdout, "%s  %s  (%s:%d)%s%s\n", ok ? "ok  " : "FAIL", tc.name, tc.file, tc.line,
                     threw ? "  exception: " : "", what.c_str());
    }
    std::fprintf(stdout, "[doctest-shim] test cases: %d | passed: %d | failed: %d\n", cases, cases - failed_cases,
                 failed_cases);
    return failed_cases ? 1 : 0;
}
#endif
