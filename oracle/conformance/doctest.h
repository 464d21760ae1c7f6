// Minimal doctest stand-in for running the reference's unit suites
// (/root/reference/proj/tests/test_*.cpp, which include <doctest.h>; the real
// header is not vendored there) against this framework's library.
// TEST INFRASTRUCTURE ONLY. Supports exactly the macros those suites use:
// TEST_CASE, SUBCASE (one nesting level), CHECK, CHECK_FALSE, REQUIRE,
// CAPTURE, CHECK_THROWS, CHECK_THROWS_AS, doctest::Approx(..).epsilon(..),
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace doctest_shim {

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
    int target = 0;    // index of the subcase to run in this pass
    int seen = 0;      // subcases met in this pass
    long checks = 0;
    long failures = 0;
    bool case_failed = false;
};

inline State& state() {
    static State s;
    return s;
}

inline bool enter_subcase() {
    State& s = state();
    return s.seen++ == s.target;
}

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    State& s = state();
    ++s.checks;
    if (ok)
        return;
    ++s.failures;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, require ? "REQUIRE" : "CHECK", expr);
    if (require)
        throw RequireFailed{};
}

inline int run_all() {
    int failed_cases = 0, cases = 0;
    for (const Case& c : registry()) {
        ++cases;
        State& s = state();
        s.case_failed = false;
        for (s.target = 0;; ++s.target) {
            s.seen = 0;
            try {
                c.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                std::fprintf(stderr, "%s:%d: TEST_CASE( %s ) threw: %s\n", c.file, c.line, c.name,
                             e.what());
                s.case_failed = true;
                ++s.failures;
            }
            if (s.seen <= s.target + 1)
                break; // no further subcase to visit
        }
        if (s.case_failed)
            ++failed_cases;
    }
    const State& s = state();
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %ld | %ld failed\n",
                cases, cases - failed_cases, failed_cases, s.checks, s.failures);
    return failed_cases ? 1 : 0;
}

} // namespace doctest_shim

namespace doctest {
class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) <
               a.eps_ * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

private:
    double value_;
    double eps_ = 1.1920928955078125e-07 * 100;
};
} // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_TEST(fn, name)                                                          \
    static void fn();                                                                        \
    static doctest_shim::Registrar DOCTEST_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TEST(DOCTEST_SHIM_CAT(doctest_shim_case_, __COUNTER__), name)
#define SUBCASE(name) if (doctest_shim::enter_subcase())
#define CHECK(...) doctest_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest_shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CAPTURE(x) ((void)0)
#define CHECK_THROWS(...)                                                                      \
    do {                                                                                       \
        bool threw_ = false;                                                                   \
        try {                                                                                  \
            (void)(__VA_ARGS__);                                                               \
        } catch (...) {                                                                        \
            threw_ = true;                                                                     \
        }                                                                                      \
        doctest_shim::report(threw_, "throws: " #__VA_ARGS__, __FILE__, __LINE__, false);     \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                            \
    do {                                                                                       \
        bool threw_ = false;                                                                   \
        try {                                                                                  \
            (void)(expr);                                                                      \
        } catch (const type&) {                                                                \
            threw_ = true;                                                                     \
        } catch (...) {                                                                        \
        }                                                                                      \
        doctest_shim::report(threw_, "throws " #type ": " #expr, __FILE__, __LINE__, false);  \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest_shim::run_all(); }
#endif
