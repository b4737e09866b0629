// Minimal doctest-compatible test shim (this repo's own code; doctest itself
// is not vendored by the reference — SURVEY §4). Supports the subset the
// reference's test_generator.cpp / test_parallel.cpp and tests/cpp use:
// TEST_CASE, CHECK, CHECK_FALSE, CHECK_MESSAGE, REQUIRE, CHECK_THROWS_AS, doctest::Approx.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    double value;
    double eps = 1e-5;  // relative, like doctest's default scale
    friend bool operator==(double lhs, const Approx& rhs) {
        const double scale = std::fmax(std::fabs(lhs), std::fabs(rhs.value));
        return std::fabs(lhs - rhs.value) <= rhs.eps * (1.0 + scale);
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
};

namespace detail {
struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Stats {
    long checks = 0;
    long failures = 0;
};
inline Stats& stats() {
    static Stats s;
    return s;
}
struct RequireFailed {};
struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
inline bool record(bool ok, const char* expr, const char* file, int line, bool require) {
    ++stats().checks;
    if (!ok) {
        ++stats().failures;
        std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
        if (require) throw RequireFailed{};
    }
    return ok;
}
inline int run_all() {
    int failed_cases = 0;
    for (const auto& c : registry()) {
        const long before = stats().failures;
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++stats().failures;
            std::fprintf(stderr, "TEST_CASE \"%s\": unexpected exception: %s\n", c.name, e.what());
        }
        if (stats().failures != before) {
            ++failed_cases;
            std::fprintf(stderr, "TEST_CASE \"%s\" FAILED\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
                registry().size() - failed_cases, failed_cases);
    std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", stats().checks,
                stats().checks - stats().failures, stats().failures);
    return failed_cases == 0 ? 0 : 1;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                   \
    static void fn();                                                      \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::record(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
// CHECK_MESSAGE(cond, msg): like CHECK, printing msg on failure.
#define CHECK_MESSAGE(cond, msg)                                                                  \
    do {                                                                                          \
        if (!::doctest::detail::record(static_cast<bool>(cond), #cond, __FILE__, __LINE__, false)) \
            std::fprintf(stderr, "  message: %s\n", std::string(msg).c_str());                  \
    } while (0)
#define CHECK_THROWS_AS(expr, exc)                                                              \
    do {                                                                                       \
        bool caught_ = false;                                                                  \
        try {                                                                                  \
            (void)(expr);                                                                      \
        } catch (const exc&) {                                                                 \
            caught_ = true;                                                                    \
        } catch (...) {                                                                        \
        }                                                                                      \
        ::doctest::detail::record(caught_, #expr " throws " #exc, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
