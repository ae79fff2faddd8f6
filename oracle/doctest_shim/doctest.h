// Minimal stand-in for the doctest single header (the reference expects it in
// proj/vendor/, which is git-ignored and absent: proj/CMakeLists.txt:16,
// proj/.gitignore:2). Test infrastructure only: it implements exactly the
// macros the reference's test files use (proj/tests/test_core.cpp,
// proj/tests/test_stream.cpp) so those files can be compiled unmodified,
// once against the patched reference (oracle/_ref) and once against the
// B200 drop-in library (libfsk_b200.so).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    Approx& scale(double s) { scale_ = s; return *this; }
    friend bool operator==(double lhs, const Approx& a) { return a.equal(lhs); }
    friend bool operator==(const Approx& a, double rhs) { return a.equal(rhs); }
    friend bool operator!=(double lhs, const Approx& a) { return !a.equal(lhs); }
    friend bool operator!=(const Approx& a, double rhs) { return !a.equal(rhs); }

private:
    bool equal(double other) const {
        // doctest semantics: |a-b| < eps * (scale + max(|a|,|b|))
        return std::fabs(other - value_) <
               eps_ * (scale_ + std::fmax(std::fabs(other), std::fabs(value_)));
    }
    double value_;
    double eps_ = 1.1920928955078125e-07 * 100;
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

struct Counters {
    long asserts = 0;
    long failed_asserts = 0;
    bool current_failed = false;
};

inline Counters& counters() {
    static Counters c;
    return c;
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    auto& c = counters();
    ++c.asserts;
    if (!ok) {
        ++c.failed_asserts;
        c.current_failed = true;
        std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) failed\n", file, line, kind, expr);
    }
}

inline int run_all() {
    long passed = 0, failed = 0;
    for (const auto& tc : registry()) {
        counters().current_failed = false;
        try {
            tc.fn();
        } catch (const std::exception& e) {
            counters().current_failed = true;
            ++counters().failed_asserts;
            std::fprintf(stderr, "%s:%d: ERROR: test case '%s' threw: %s\n", tc.file, tc.line,
                         tc.name, e.what());
        }
        if (counters().current_failed) {
            ++failed;
            std::fprintf(stderr, "[doctest-shim] FAILED: %s\n", tc.name);
        } else {
            ++passed;
        }
    }
    std::printf("[doctest] test cases: %ld | %ld passed | %ld failed\n", passed + failed, passed,
                failed);
    std::printf("[doctest] assertions: %ld | %ld passed | %ld failed\n", counters().asserts,
                counters().asserts - counters().failed_asserts, counters().failed_asserts);
    return failed == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fname, name)                                                  \
    static void fname();                                                                     \
    static ::doctest::detail::Registrar DOCTEST_CAT(fname, _reg)(name, __FILE__, __LINE__,   \
                                                                 &fname);                    \
    static void fname()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...) CHECK(__VA_ARGS__)

#define CHECK_THROWS_AS(expr, ...)                                                           \
    do {                                                                                     \
        bool doctest_ok_ = false;                                                            \
        try {                                                                                \
            (void)(expr);                                                                    \
        } catch (const __VA_ARGS__&) {                                                       \
            doctest_ok_ = true;                                                              \
        } catch (...) {                                                                      \
        }                                                                                    \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
    } while (0)

#define CHECK_NOTHROW(expr)                                                                  \
    do {                                                                                     \
        bool doctest_ok_ = true;                                                             \
        try {                                                                                \
            (void)(expr);                                                                    \
        } catch (...) {                                                                      \
            doctest_ok_ = false;                                                             \
        }                                                                                    \
        ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__);   \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
