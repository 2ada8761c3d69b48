// Minimal doctest-compatible test harness, written for this repository so the reference's own
// unit tests (/root/reference/proj/tests/test_*.cpp, which include <doctest.h> from the
// un-shipped vendor/ tree) compile UNCHANGED against the B200 library.
//
// Covers exactly what those files use: TEST_CASE, SUBCASE (one level: the test case body is
// re-run once per subcase, entering only that subcase, as doctest does), CHECK, REQUIRE,
// CHECK_THROWS_AS, FAIL, doctest::Approx(v).epsilon(e), and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
// Approx follows doctest's rule: |a - b| < eps * (scale + max(|a|, |b|)), eps = 100 * FLT_EPSILON
// by default, scale 1.  Output: one line per failed assertion, a summary, exit code 1 on failure.
// Optional argument: a substring filter on the test-case name.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
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
    bool matches(double other) const {
        return std::fabs(other - value_) < eps_ * (scale_ + std::fmax(std::fabs(other), std::fabs(value_)));
    }
    friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
    friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }
    friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || rhs.matches(lhs); }
    friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || rhs.matches(lhs); }

private:
    double value_;
    double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
    double scale_ = 1.0;
};

namespace detail {

struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> cases;
    return cases;
}

struct State {
    int target = 0;       // subcase entered in this run
    int seen = 0;         // subcases met so far in this run
    bool in_sub = false;
    long asserts = 0, failed = 0;
    bool case_failed = false;
};

inline State& state() {
    static State s;
    return s;
}

struct Register {
    Register(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back(Case{name, file, line, fn});
    }
};

struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    State& s = state();
    ++s.asserts;
    if (ok) return;
    ++s.failed;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}

// SUBCASE: enter the subcase whose index equals this run's target (single nesting level)
struct Subcase {
    bool entered = false;
    explicit Subcase(const char*) {
        State& s = state();
        if (!s.in_sub && s.seen++ == s.target) {
            entered = true;
            s.in_sub = true;
        }
    }
    ~Subcase() {
        if (entered) state().in_sub = false;
    }
    explicit operator bool() const { return entered; }
};

inline int run(int argc, char** argv) {
    const char* filter = argc > 1 ? argv[1] : nullptr;
    State& s = state();
    int cases = 0, failed_cases = 0;
    for (const Case& c : registry()) {
        if (filter && !std::strstr(c.name, filter)) continue;
        ++cases;
        s.case_failed = false;
        for (s.target = 0;; ++s.target) {
            s.seen = 0;
            s.in_sub = false;
            try {
                c.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                ++s.failed;
                s.case_failed = true;
                std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
            } catch (...) {
                ++s.failed;
                s.case_failed = true;
                std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw an unknown exception\n", c.file, c.line, c.name);
            }
            if (s.target + 1 >= s.seen) break; // every subcase of this case has had its run
        }
        if (s.case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "[doctest-compat] FAILED: %s\n", c.name);
        }
    }
    std::printf("[doctest-compat] test cases: %d | %d passed | %d failed\n", cases, cases - failed_cases, failed_cases);
    std::printf("[doctest-compat] assertions: %ld | %ld passed | %ld failed\n", s.asserts, s.asserts - s.failed,
                s.failed);
    return failed_cases ? 1 : 0;
}

} // namespace detail
} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                                   \
    static void fn();                                                                                       \
    static const ::doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);          \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_CAT(doctest_sub_, __LINE__){name})

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                       \
    do {                                                                                                   \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                           \
        ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);               \
        if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                                        \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                         \
    do {                                                                                                   \
        bool doctest_caught_ = false;                                                                      \
        try {                                                                                              \
            expr;                                                                                          \
        } catch (const __VA_ARGS__&) {                                                                     \
            doctest_caught_ = true;                                                                        \
        } catch (...) {                                                                                    \
        }                                                                                                  \
        ::doctest::detail::report(doctest_caught_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__,   \
                                  __LINE__);                                                               \
    } while (0)
#define FAIL(msg)                                                                                          \
    do {                                                                                                   \
        ::doctest::detail::report(false, "FAIL", msg, __FILE__, __LINE__);                                 \
        throw ::doctest::detail::RequireFailed{};                                                          \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
