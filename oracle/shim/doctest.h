// Minimal doctest-compatible test harness, written for this repo (ORACLE / TEST
// INFRASTRUCTURE ONLY). The reference's unit suites (/root/reference/proj/tests)
// include <doctest.h>, which is not vendored in the reference tree; this header
// implements just the macros those suites use so they can be compiled, as they
// lie, against the B200 drop-in translation units (oracle/Makefile `dropin`).
//
// Semantics: TEST_CASE registers a function; CHECK* records a failure and
// continues; REQUIRE* / FAIL abort the test case; SUBCASE bodies run in order
// within one pass; MESSAGE/INFO/CAPTURE are no-ops. main() runs every case,
// prints a summary and returns non-zero on any failure. `--exclude=<substr>`
// skips cases whose name contains <substr>.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(const char* n, void (*f)(), const char* file, int line) {
        registry().push_back({n, f, file, line});
    }
};

struct RequireFailure {};

struct Stats {
    long checks = 0, failed_checks = 0;
};
inline Stats& stats() {
    static Stats s;
    return s;
}
inline bool& case_failed() {
    static bool f = false;
    return f;
}

inline bool report(bool ok, const char* what, const char* file, int line) {
    ++stats().checks;
    if (!ok) {
        ++stats().failed_checks;
        case_failed() = true;
        std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, what);
    }
    return ok;
}

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
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.v_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.v_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
    friend bool operator<=(double lhs, const Approx& a) { return lhs < a.v_ || lhs == a; }
    friend bool operator>=(double lhs, const Approx& a) { return lhs > a.v_ || lhs == a; }
    friend bool operator<(double lhs, const Approx& a) { return lhs < a.v_ && lhs != a; }
    friend bool operator>(double lhs, const Approx& a) { return lhs > a.v_ && lhs != a; }

private:
    double v_;
    double eps_ = 1.1920929e-7 * 100;
    double scale_ = 1.0;
};

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, reg, name)                                                \
    static void fn();                                                               \
    static doctest::Registrar reg(name, &fn, __FILE__, __LINE__);                   \
    static void fn()
#define TEST_CASE(name) DOCTEST_CASE_(DOCTEST_CAT(doctest_fn_, __LINE__), DOCTEST_CAT(doctest_reg_, __LINE__), name)
#define SUBCASE(name) if (true)

#define CHECK(...) ((void)doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__))
#define CHECK_FALSE(...) ((void)doctest::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__))
#define REQUIRE(...)                                                                            \
    do {                                                                                        \
        if (!doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)) \
            throw doctest::RequireFailure();                                                    \
    } while (0)
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define DOCTEST_THROWS_(expr, catcher, req)                                          \
    do {                                                                             \
        bool ok_ = false;                                                            \
        try {                                                                        \
            (void)(expr);                                                            \
        } catcher                                                                    \
        if (!doctest::report(ok_, "throws: " #expr, __FILE__, __LINE__) && (req))    \
            throw doctest::RequireFailure();                                         \
    } while (0)
#define CHECK_THROWS_AS(expr, ...) \
    DOCTEST_THROWS_(expr, catch (const __VA_ARGS__&) { ok_ = true; } catch (...) {}, false)
#define REQUIRE_THROWS_AS(expr, ...) \
    DOCTEST_THROWS_(expr, catch (const __VA_ARGS__&) { ok_ = true; } catch (...) {}, true)
#define CHECK_THROWS(expr) DOCTEST_THROWS_(expr, catch (...) { ok_ = true; }, false)
#define REQUIRE_THROWS(expr) DOCTEST_THROWS_(expr, catch (...) { ok_ = true; }, true)
#define CHECK_NOTHROW(expr)                                                   \
    do {                                                                      \
        bool ok_ = true;                                                      \
        try {                                                                 \
            (void)(expr);                                                     \
        } catch (...) {                                                       \
            ok_ = false;                                                      \
        }                                                                     \
        doctest::report(ok_, "nothrow: " #expr, __FILE__, __LINE__);          \
    } while (0)
#define FAIL(...)                                                             \
    do {                                                                      \
        doctest::report(false, "FAIL", __FILE__, __LINE__);                   \
        throw doctest::RequireFailure();                                      \
    } while (0)
#define MESSAGE(...) ((void)0)
#define INFO(...) ((void)0)
#define CAPTURE(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    std::vector<std::string> excludes;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "--exclude=", 10) == 0) excludes.emplace_back(argv[i] + 10);
    int failed = 0, run = 0;
    for (const auto& tc : doctest::registry()) {
        bool skip = false;
        for (const auto& e : excludes)
            if (std::string(tc.name).find(e) != std::string::npos) skip = true;
        if (skip) continue;
        ++run;
        doctest::case_failed() = false;
        try {
            tc.fn();
        } catch (const doctest::RequireFailure&) {
            doctest::case_failed() = true;
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: exception: %s\n", tc.file, tc.line, e.what());
            doctest::case_failed() = true;
        } catch (...) {
            std::fprintf(stderr, "%s:%d: unknown exception\n", tc.file, tc.line);
            doctest::case_failed() = true;
        }
        if (doctest::case_failed()) {
            ++failed;
            std::fprintf(stderr, "TEST CASE FAILED: %s\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | checks: %ld | %ld failed\n", run,
                run - failed, failed, doctest::stats().checks, doctest::stats().failed_checks);
    std::fflush(stdout);
    std::fflush(stderr);
    return failed ? 1 : 0;
}
#endif
