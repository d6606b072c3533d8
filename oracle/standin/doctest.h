// ORACLE TEST INFRASTRUCTURE — minimal stand-in for the doctest macros the
// reference's own unit tests use (proj/tests/test_*.cpp). The vendored
// doctest (proj/vendor/, git-ignored upstream) is absent from the image;
// this lets the reference's tests run against the stand-in-built reference
// as a self-check of the oracle harness. Written from the macro names only.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) { eps = e; return *this; }
    Approx& scale(double s) { scl = s; return *this; }
    double value;
    double eps = 1.1920928955078125e-05 * 100;
    double scl = 1.0;
};
inline bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value) < a.eps * (a.scl + std::max(std::fabs(lhs), std::fabs(a.value)));
}
inline bool operator==(const Approx& a, double rhs) { return rhs == a; }
inline bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

struct Contains {
    explicit Contains(const char* s) : needle(s) {}
    bool matches(const std::string& what) const { return what.find(needle) != std::string::npos; }
    std::string needle;
};

namespace detail {
struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};
struct State {
    long checks = 0, failures = 0;
    int sub_target = 0, sub_seen = 0;
    const char* current = "";
};
inline State& state() {
    static State s;
    return s;
}
inline void record(bool ok, const char* expr, const char* file, int line) {
    auto& s = state();
    ++s.checks;
    if (!ok) {
        ++s.failures;
        if (s.failures <= 50) std::fprintf(stderr, "%s:%d: CHECK failed in '%s': %s\n", file, line, s.current, expr);
    }
}
// Each top-level run executes exactly one leaf SUBCASE (by encounter order).
inline bool enter_subcase() { auto& s = state(); return s.sub_seen++ == s.sub_target; }
struct FailNow {};
}  // namespace detail

inline int run_all() {
    auto& s = detail::state();
    int failed_cases = 0;
    for (const auto& c : detail::registry()) {
        long before = s.failures;
        s.current = c.name;
        s.sub_target = 0;
        for (;;) {
            s.sub_seen = 0;
            try {
                c.fn();
            } catch (const detail::FailNow&) {
            } catch (const std::exception& e) {
                detail::record(false, e.what(), c.file, c.line);
            }
            if (s.sub_seen > s.sub_target + 1) { ++s.sub_target; continue; }
            break;
        }
        if (s.failures != before) ++failed_cases;
    }
    std::printf("[doctest-standin] test cases: %zu | %d failed | checks: %ld | %ld failed\n",
                detail::registry().size(), failed_cases, s.checks, s.failures);
    return s.failures == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                     \
    static void fn();                                                                 \
    static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __LINE__), name)
#define SUBCASE(name) if (doctest::detail::enter_subcase())
#define CHECK(...) doctest::detail::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                      \
    do {                                                                  \
        bool ok_ = static_cast<bool>(__VA_ARGS__);                        \
        doctest::detail::record(ok_, #__VA_ARGS__, __FILE__, __LINE__);   \
        if (!ok_) throw doctest::detail::FailNow{};                       \
    } while (0)
#define FAIL(msg)                                                         \
    do {                                                                  \
        doctest::detail::record(false, msg, __FILE__, __LINE__);          \
        throw doctest::detail::FailNow{};                                 \
    } while (0)
#define CHECK_NOTHROW(...)                                                \
    do {                                                                  \
        bool ok_ = true;                                                  \
        try { (void)(__VA_ARGS__); } catch (...) { ok_ = false; }         \
        doctest::detail::record(ok_, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                        \
    do {                                                                  \
        bool ok_ = false;                                                 \
        try { (void)(expr); } catch (const __VA_ARGS__&) { ok_ = true; } catch (...) {} \
        doctest::detail::record(ok_, "throws: " #expr, __FILE__, __LINE__); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                          \
    do {                                                                  \
        bool ok_ = false;                                                 \
        try { (void)(expr); } catch (const __VA_ARGS__& e_) { ok_ = (matcher).matches(e_.what()); } catch (...) {} \
        doctest::detail::record(ok_, "throws-with: " #expr, __FILE__, __LINE__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::run_all(); }
#endif
