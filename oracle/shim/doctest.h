// oracle/shim/doctest.h — TEST INFRASTRUCTURE ONLY.
//
// doctest is a third-party, header-only test framework the reference's suites use
// (`proj/tests/*.cpp`, expected in the git-ignored `proj/vendor/`, absent here).
// This is a minimal restatement of the subset the reference tests use: TEST_CASE,
// CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, CAPTURE, FAIL and
// doctest::Approx(..).epsilon(..) with doctest's published comparison rule
//   |lhs - v| < eps * (scale + max(|lhs|, |v|)),  scale = 1, default eps = 100 * FLT_EPSILON.
// It lets the unmodified reference suites run against the oracle build (pinning the
// shimmed FFT) and against this repo's C++ facade.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) <
               a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

private:
    double value_;
    double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
    double scale_ = 1.0;
};

namespace detail {

struct TestCase {
    const char* name;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct State {
    int checks = 0;
    int failed_checks = 0;
    bool case_failed = false;
    std::vector<std::string> captures;
};

inline State& state() {
    static State s;
    return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    State& s = state();
    ++s.checks;
    if (ok) return;
    ++s.failed_checks;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, require ? "REQUIRE" : "CHECK",
                 expr);
    for (const auto& c : s.captures) std::fprintf(stderr, "  with %s\n", c.c_str());
    if (require) throw RequireFailed{};
}

struct CaptureGuard {
    template <typename T>
    CaptureGuard(const char* name, const T& v) {
        std::ostringstream os;
        os << name << " := " << v;
        state().captures.push_back(os.str());
    }
    ~CaptureGuard() { state().captures.pop_back(); }
};

inline int run_all() {
    int failed_cases = 0;
    for (const auto& tc : registry()) {
        State& s = state();
        s.case_failed = false;
        s.captures.clear();
        try {
            tc.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "TEST CASE \"%s\" threw: %s\n", tc.name, e.what());
            s.case_failed = true;
        }
        if (s.case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "FAILED test case: %s\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks: %d | %d failed\n",
                registry().size(), registry().size() - static_cast<std::size_t>(failed_cases),
                failed_cases, state().checks, state().failed_checks);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __COUNTER__)

#define DOCTEST_TEST_CASE_IMPL(fn, name)                                    \
    static void fn();                                                       \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);   \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_ANON(doctest_tc_), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(msg) ::doctest::detail::report(false, "FAIL", __FILE__, __LINE__, true)
#define CAPTURE(x) ::doctest::detail::CaptureGuard DOCTEST_ANON(doctest_cap_)(#x, x)

#define CHECK_THROWS_AS(expr, ...)                                                   \
    do {                                                                             \
        bool doctest_ok_ = false;                                                    \
        try {                                                                        \
            (void)(expr);                                                            \
        } catch (const __VA_ARGS__&) {                                               \
            doctest_ok_ = true;                                                      \
        } catch (...) {                                                              \
        }                                                                            \
        ::doctest::detail::report(doctest_ok_, "THROWS_AS " #expr, __FILE__, __LINE__, false); \
    } while (0)

#define CHECK_NOTHROW(expr)                                                          \
    do {                                                                             \
        bool doctest_ok_ = true;                                                     \
        try {                                                                        \
            (void)(expr);                                                            \
        } catch (...) {                                                              \
            doctest_ok_ = false;                                                     \
        }                                                                            \
        ::doctest::detail::report(doctest_ok_, "NOTHROW " #expr, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
