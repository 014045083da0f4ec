// TEST INFRASTRUCTURE ONLY: a minimal stand-in for the doctest header the
// reference's unit tests include (<doctest.h>, absent from this image; the
// reference expects it under its git-ignored vendor/, proj/CMakeLists.txt:10).
// It implements exactly what /root/reference/proj/tests/test_{grid,metric,
// scan_parallel,transforms,io,cli}.cpp use: TEST_CASE, SUBCASE (flat), CHECK,
// CHECK_FALSE, REQUIRE, FAIL, CHECK_NOTHROW, CHECK_THROWS_AS and doctest::Approx (doctest's comparison rule
// |a - b| < eps * (scale + max(|a|, |b|)), eps = 100 * FLT_EPSILON, scale = 1).
// Each test case runs in its own try/catch; the runner prints one line per case
// and a summary, and exits non-zero on any failure.  Cases listed (one name per
// line) in the file named by GD_EXPECTED_FAIL are reported as expected failures
// (the drop-in rejects the reference's CPU-only engines by design).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <fstream>
#include <functional>
#include <limits>
#include <set>
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
    friend bool operator==(double a, const Approx& b) { return b.eq(a); }
    friend bool operator==(const Approx& b, double a) { return b.eq(a); }
    friend bool operator!=(double a, const Approx& b) { return !b.eq(a); }
    friend bool operator!=(const Approx& b, double a) { return !b.eq(a); }

private:
    bool eq(double a) const {
        return std::fabs(a - value_) < eps_ * (scale_ + std::max(std::fabs(a), std::fabs(value_)));
    }
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
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
    static std::vector<Case> r;
    return r;
}

struct Reg {
    Reg(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct RequireFailed {};

// SUBCASE: the test case body runs once per leaf subcase (doctest's model,
// flat subcases only): pass k executes the k-th SUBCASE it meets.
struct SubcaseState {
    int target = 0;
    int seen = 0;
};
inline SubcaseState& subcases() {
    static SubcaseState s;
    return s;
}
inline bool enter_subcase() { return subcases().seen++ == subcases().target; }

inline int& failures() {
    static int f = 0;
    return f;
}
inline long long& checks() {
    static long long c = 0;
    return c;
}

inline void report(bool ok, const char* what, const char* file, int line) {
    ++checks();
    if (!ok) {
        ++failures();
        if (failures() <= 200) std::printf("  %s:%d: CHECK FAILED: %s\n", file, line, what);
    }
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_CASE_IMPL(fn, name)                                                     \
    static void fn();                                                                   \
    static doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);   \
    static void fn()
#define TEST_CASE(name) DOCTEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define SUBCASE(name) if (doctest::detail::enter_subcase())
#define FAIL(...)                                                                   \
    do {                                                                            \
        doctest::detail::report(false, "FAIL: " #__VA_ARGS__, __FILE__, __LINE__);  \
        throw doctest::detail::RequireFailed{};                                     \
    } while (0)
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                       \
    do {                                                                                   \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                           \
        doctest::detail::report(doctest_ok_, #__VA_ARGS__, __FILE__, __LINE__);            \
        if (!doctest_ok_) throw doctest::detail::RequireFailed{};                          \
    } while (0)
#define CHECK_NOTHROW(...)                                                                 \
    do {                                                                                   \
        bool doctest_ok_ = true;                                                           \
        try {                                                                              \
            (void)(__VA_ARGS__);                                                           \
        } catch (...) {                                                                    \
            doctest_ok_ = false;                                                           \
        }                                                                                  \
        doctest::detail::report(doctest_ok_, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                         \
    do {                                                                                   \
        bool doctest_ok_ = false;                                                          \
        try {                                                                              \
            (void)(expr);                                                                  \
        } catch (const __VA_ARGS__&) {                                                     \
            doctest_ok_ = true;                                                            \
        } catch (...) {                                                                    \
        }                                                                                  \
        doctest::detail::report(doctest_ok_, "throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    using namespace doctest::detail;
    std::set<std::string> expected;
    if (const char* path = std::getenv("GD_EXPECTED_FAIL")) {
        std::ifstream f(path);
        for (std::string line; std::getline(f, line);)
            if (!line.empty() && line[0] != '#') expected.insert(line);
    }
    int failed = 0, xfail = 0, unexpected_pass = 0;
    for (const Case& c : registry()) {
        const int before = failures();
        std::string err;
        try {
            SubcaseState& sc = subcases();
            sc.target = 0;
            do {
                sc.seen = 0;
                c.fn();
                ++sc.target;
            } while (sc.target < sc.seen);
        } catch (const RequireFailed&) {
            err = "REQUIRE failed";
        } catch (const std::exception& e) {
            err = std::string("exception: ") + e.what();
            ++failures();
        } catch (...) {
            err = "unknown exception";
            ++failures();
        }
        const bool ok = failures() == before;
        const bool xf = expected.count(c.name) != 0;
        if (ok && xf) ++unexpected_pass;
        if (!ok && xf) ++xfail;
        if (!ok && !xf) ++failed;
        std::printf("%s %s (%s:%d)%s%s\n", ok ? (xf ? "XPASS" : "PASS ") : (xf ? "XFAIL" : "FAIL "),
                    c.name, c.file, c.line, err.empty() ? "" : " -- ", err.c_str());
    }
    std::printf("== %zu test cases: %zu passed, %d failed, %d expected failures "
                "(%d unexpectedly passed); %lld checks\n",
                registry().size(), registry().size() - failed - xfail, failed, xfail,
                unexpected_pass, checks());
    return failed == 0 ? 0 : 1;
}
#endif
