// Minimal doctest-compatible shim: TEST INFRASTRUCTURE ONLY.
//
// The reference's own unit tests (/root/reference/proj/tests/test_*.cpp)
// include <doctest.h> from proj/vendor/, which is absent from the mounted
// reference (proj/.gitignore:2). This header implements exactly the subset of
// the doctest API those files use (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, doctest::Contains) so oracle/Makefile can build and
// run the reference's tests unmodified, pinning oracle/_ref to its own suite.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Contains {
    std::string needle;
    explicit Contains(const char* s) : needle(s) {}
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

struct Stats {
    long checks = 0;
    long failures = 0;
    bool current_failed = false;
};

inline Stats& stats() {
    static Stats s;
    return s;
}

struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    ++stats().checks;
    if (ok) return;
    ++stats().failures;
    stats().current_failed = true;
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
    if (require) throw RequireFailed{};
}

inline bool message_contains(const std::exception& e, const Contains& c) {
    return std::string(e.what()).find(c.needle) != std::string::npos;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define DOCTEST_TEST_CASE_IMPL(fn, name)                                              \
    static void fn();                                                                 \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);             \
    static void fn()

#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, exc)                                                    \
    do {                                                                              \
        bool doctest_ok_ = false;                                                     \
        try { (void)(expr); } catch (const exc&) { doctest_ok_ = true; } catch (...) {} \
        ::doctest::detail::report(doctest_ok_, "THROWS_AS(" #expr ", " #exc ")",       \
                                  __FILE__, __LINE__, false);                         \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, contains, exc)                                     \
    do {                                                                              \
        bool doctest_ok_ = false;                                                     \
        try { (void)(expr); } catch (const exc& e_) {                                 \
            doctest_ok_ = ::doctest::detail::message_contains(e_, contains);          \
        } catch (...) {}                                                              \
        ::doctest::detail::report(doctest_ok_, "THROWS_WITH_AS(" #expr ", " #exc ")",  \
                                  __FILE__, __LINE__, false);                         \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    using namespace doctest::detail;
    long cases = 0, failed_cases = 0;
    for (const auto& tc : registry()) {
        ++cases;
        stats().current_failed = false;
        try {
            tc.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "TEST_CASE '%s' threw: %s\n", tc.name, e.what());
            stats().current_failed = true;
            ++stats().failures;
        }
        if (stats().current_failed) {
            ++failed_cases;
            std::fprintf(stderr, "FAILED: %s\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %ld | %ld passed | %ld failed ; assertions: %ld | %ld failed\n",
                cases, cases - failed_cases, failed_cases, stats().checks, stats().failures);
    return failed_cases == 0 ? 0 : 1;
}
#endif
