// Minimal doctest-compatible test shim (test infrastructure, not product code).
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) include
// <doctest.h>, whose vendor/ directory is absent from the reference
// (proj/.gitignore:2). This header implements only the subset those tests use
// so they can be compiled, unchanged, against (a) the reference library and
// (b) this repo's drop-in library:
//   TEST_CASE, SUBCASE (all subcases run in one pass), CHECK, CHECK_FALSE,
//   REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, doctest::Approx with
//   .epsilon(), doctest::Contains.
// Output: one line per failed assertion, then a summary line
//   "[shim] test cases: N | passed: P | failed: F"
// and a line per failed case "[shim] FAILED <name>" so a driver can diff the
// failing set between the two libraries.
#pragma once
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    double value;
    double eps = 1.1920928955078125e-05 * 100;  // float epsilon * 100, doctest's default
    double scale = 1.0;
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) { eps = e; return *this; }
    Approx& scale_(double s) { scale = s; return *this; }
    bool matches(double other) const {
        return std::fabs(other - value) < eps * (scale + std::fmax(std::fabs(other), std::fabs(value)));
    }
};
inline bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
inline bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }

struct Contains {
    std::string needle;
    explicit Contains(const char* s) : needle(s) {}
    bool in(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
};

namespace shim {

struct RequireFailed {};

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

struct State {
    int case_failures = 0;
    long assertions = 0;
    long failed_assertions = 0;
};
inline State& state() {
    static State s;
    return s;
}

inline int register_case(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back(Case{name, file, line, fn});
    return 0;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    ++state().assertions;
    if (ok) return;
    ++state().failed_assertions;
    ++state().case_failures;
    if (state().case_failures <= 8) {
        std::fprintf(stdout, "[shim]   %s:%d: %s( %s ) failed\n", file, line, kind, expr);
    }
}

inline int run_all() {
    int passed = 0, failed = 0;
    std::vector<std::string> failed_names;
    for (const Case& c : registry()) {
        state().case_failures = 0;
        try {
            c.fn();
        } catch (const RequireFailed&) {
            // already reported
        } catch (const std::exception& e) {
            ++state().case_failures;
            std::fprintf(stdout, "[shim]   %s:%d: unexpected exception: %s\n", c.file, c.line, e.what());
        } catch (...) {
            ++state().case_failures;
            std::fprintf(stdout, "[shim]   %s:%d: unexpected non-std exception\n", c.file, c.line);
        }
        if (state().case_failures == 0) {
            ++passed;
        } else {
            ++failed;
            failed_names.push_back(c.name);
            std::fprintf(stdout, "[shim] FAILED %s (%d failed assertions)\n", c.name, state().case_failures);
        }
    }
    std::fprintf(stdout, "[shim] test cases: %d | passed: %d | failed: %d | assertions: %ld | failed assertions: %ld\n",
                 passed + failed, passed, failed, state().assertions, state().failed_assertions);
    return failed == 0 ? 0 : 1;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_CASE(fn, name)                                                              \
    static void fn();                                                                            \
    static const int DOCTEST_SHIM_CAT(fn, _reg) =                                                \
        ::doctest::shim::register_case(name, __FILE__, __LINE__, &fn);                           \
    static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_CASE(DOCTEST_SHIM_CAT(doctest_shim_case_, __COUNTER__), name)
#define SUBCASE(name) if (true)

#define CHECK(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::shim::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                               \
    do {                                                                                           \
        const bool doctest_shim_ok_ = static_cast<bool>(__VA_ARGS__);                              \
        ::doctest::shim::report(doctest_shim_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);   \
        if (!doctest_shim_ok_) throw ::doctest::shim::RequireFailed{};                              \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                 \
    do {                                                                                           \
        bool doctest_shim_ok_ = false;                                                             \
        try {                                                                                      \
            static_cast<void>(expr);                                                               \
        } catch (const __VA_ARGS__&) {                                                             \
            doctest_shim_ok_ = true;                                                               \
        } catch (...) {                                                                            \
        }                                                                                          \
        ::doctest::shim::report(doctest_shim_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);  \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                                   \
    do {                                                                                           \
        bool doctest_shim_ok_ = false;                                                             \
        try {                                                                                      \
            static_cast<void>(expr);                                                               \
        } catch (const __VA_ARGS__& e) {                                                           \
            doctest_shim_ok_ = (matcher).in(e.what());                                             \
        } catch (...) {                                                                            \
        }                                                                                          \
        ::doctest::shim::report(doctest_shim_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::shim::run_all(); }
#endif
