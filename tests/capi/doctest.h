// Minimal doctest-compatible test harness -- TEST INFRASTRUCTURE ONLY.
//
// doctest itself is not installed here, so this header implements just the subset the
// reference's C-API suite uses (proj/tests/test_capi.cpp): TEST_CASE, CHECK, REQUIRE,
// doctest::Approx with .epsilon() / .scale(), and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
// It lets that suite compile UNCHANGED against include/backproject.h and link against
// libbackproject.so (tests/capi/Makefile), the drop-in proof of SURVEY.md 8(b).
//
// Output: one "[case] PASSED|FAILED" line per test case, failed assertions with
// file:line, and a summary; the exit code is the number of failed test cases.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    // doctest's rule: |lhs - v| < eps * (scale + max(|lhs|, |v|))
    bool matches(double lhs) const {
        return std::fabs(lhs - v_) < eps_ * (scale_ + std::fmax(std::fabs(lhs), std::fabs(v_)));
    }
    double value() const { return v_; }

private:
    double v_;
    double eps_ = 1.19209290e-7 * 100;  // doctest's default: float epsilon * 100
    double scale_ = 1.0;
};
inline bool operator==(double lhs, const Approx& a) { return a.matches(lhs); }
inline bool operator==(const Approx& a, double rhs) { return a.matches(rhs); }
inline bool operator!=(double lhs, const Approx& a) { return !a.matches(lhs); }

namespace detail {

struct Case {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Register {
    Register(const char* name, void (*fn)(), const char* file, int line) {
        registry().push_back({name, fn, file, line});
    }
};

struct RequireFailed : std::exception {};

inline int& failures() {
    static int f = 0;
    return f;
}
inline int& assertions() {
    static int a = 0;
    return a;
}

inline void check(bool ok, const char* expr, const char* file, int line, bool require) {
    ++assertions();
    if (ok) return;
    ++failures();
    std::printf("  %s:%d: %s( %s ) failed\n", file, line, require ? "REQUIRE" : "CHECK", expr);
    if (require) throw RequireFailed();
}

inline int run_all() {
    int failed_cases = 0;
    for (const auto& c : registry()) {
        const int before = failures();
        bool threw = false;
        std::string what;
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            threw = true;
            what = e.what();
        } catch (...) {
            threw = true;
            what = "unknown exception";
        }
        if (threw) {
            ++failures();
            std::printf("  unexpected exception: %s\n", what.c_str());
        }
        const bool ok = failures() == before;
        if (!ok) ++failed_cases;
        std::printf("[%s] %s\n", c.name, ok ? "PASSED" : "FAILED");
        std::fflush(stdout);
    }
    std::printf("test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
                registry().size(), registry().size() - (size_t)failed_cases, failed_cases,
                assertions(), failures());
    return failed_cases;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, name)                                                        \
    static void fn();                                                                  \
    static doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__); \
    static void fn()
#define TEST_CASE(name) DOCTEST_CASE_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define CHECK(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
