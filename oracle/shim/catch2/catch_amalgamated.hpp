#pragma once
// ORACLE TEST INFRASTRUCTURE — not product code.
//
// Tiny Catch2-compatible harness (Catch2 is absent from this image) so the
// reference's own unit tests (/root/reference/proj/tests/test_*.cpp) compile
// UNCHANGED into oracle/_ref/ binaries. Supports exactly the macros those
// files use: TEST_CASE, CHECK, REQUIRE, CHECK_FALSE, REQUIRE_FALSE,
// CHECK_THROWS_AS, CHECK_NOTHROW, SUCCEED.

#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace catch_shim {

struct TestCase {
    const char* name;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Stats {
    long checks = 0;
    long failures = 0;
    bool case_failed = false;
};

inline Stats& stats() {
    static Stats s;
    return s;
}

struct RequireAbort {};

struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
    ++stats().checks;
    if (!ok) {
        ++stats().failures;
        stats().case_failed = true;
        std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
        if (fatal) throw RequireAbort{};
    }
}

inline int run_all(int argc, char** argv) {
    const char* filter = argc > 1 ? argv[1] : nullptr;
    int failed_cases = 0, ran = 0;
    for (const auto& tc : registry()) {
        if (filter && std::string(tc.name).find(filter) == std::string::npos) continue;
        ++ran;
        stats().case_failed = false;
        try {
            tc.fn();
        } catch (const RequireAbort&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "test case '%s' threw: %s\n", tc.name, e.what());
            stats().case_failed = true;
            ++stats().failures;
        }
        if (stats().case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "FAILED test case: %s\n", tc.name);
        }
    }
    std::printf("%d test cases, %d failed; %ld assertions, %ld failed\n", ran, failed_cases,
                stats().checks, stats().failures);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace catch_shim

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_TC(fn, name)                                        \
    static void fn();                                                  \
    static ::catch_shim::Registrar CATCH_SHIM_CAT(fn, _reg)(name, &fn); \
    static void fn()
#define TEST_CASE(name, ...) CATCH_SHIM_TC(CATCH_SHIM_CAT(catch_shim_tc_, __LINE__), name)

#define CATCH_SHIM_CHECK(expr, fatal) \
    ::catch_shim::report(static_cast<bool>(expr), #expr, __FILE__, __LINE__, fatal)
#define CHECK(...) CATCH_SHIM_CHECK((__VA_ARGS__), false)
#define REQUIRE(...) CATCH_SHIM_CHECK((__VA_ARGS__), true)
#define CHECK_FALSE(...) CATCH_SHIM_CHECK(!(__VA_ARGS__), false)
#define REQUIRE_FALSE(...) CATCH_SHIM_CHECK(!(__VA_ARGS__), true)
#define SUCCEED(...) ::catch_shim::report(true, "SUCCEED", __FILE__, __LINE__, false)
#define CHECK_THROWS_AS(expr, type)                                            \
    do {                                                                       \
        bool caught_ = false;                                                  \
        try {                                                                  \
            (void)(expr);                                                      \
        } catch (const type&) {                                                \
            caught_ = true;                                                    \
        } catch (...) {                                                        \
        }                                                                      \
        ::catch_shim::report(caught_, "THROWS_AS " #type ": " #expr, __FILE__, \
                             __LINE__, false);                                 \
    } while (0)
#define CHECK_NOTHROW(expr)                                                      \
    do {                                                                         \
        bool ok_ = true;                                                         \
        try {                                                                    \
            (void)(expr);                                                        \
        } catch (...) {                                                          \
            ok_ = false;                                                         \
        }                                                                        \
        ::catch_shim::report(ok_, "NOTHROW: " #expr, __FILE__, __LINE__, false); \
    } while (0)
