// doctest.h — a minimal, self-written stand-in for the doctest framework (which is not in this
// image and cannot be fetched).  It implements only what the reference's unit tests use:
// TEST_CASE, SUBCASE (each leaf subcase runs in its own pass of the test case), CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS, CHECK_THROWS_AS, FAIL, doctest::Approx (epsilon / scale,
// the usual |a - b| < eps * (scale + max(|a|, |b|)) rule) and the generated main().  Failures
// print file:line and the expression; the exit code is the number of failed test cases.
#ifndef RRSVD_B200_MINI_DOCTEST_H
#define RRSVD_B200_MINI_DOCTEST_H

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <set>
#include <string>
#include <vector>

namespace doctest {

class Approx {
  public:
    explicit Approx(double value)
        : value_(value), eps_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100), scale_(1.0) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& rhs) { return rhs.close(lhs); }
    friend bool operator==(const Approx& lhs, double rhs) { return lhs.close(rhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.close(lhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.close(rhs); }
    friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || rhs.close(lhs); }
    friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || rhs.close(lhs); }
    friend bool operator<(double lhs, const Approx& rhs) { return lhs < rhs.value_ && !rhs.close(lhs); }
    friend bool operator>(double lhs, const Approx& rhs) { return lhs > rhs.value_ && !rhs.close(lhs); }

  private:
    bool close(double x) const {
        return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
    }
    double value_, eps_, scale_;
};

namespace detail {
struct RequireAbort {};
typedef void (*TestFn)();
struct Case {
    const char* name;
    const char* file;
    int line;
    TestFn fn;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, const char* file, int line, TestFn fn) { registry().push_back({name, file, line, fn}); }
};
struct State {
    int failed_asserts = 0;
    long long asserts = 0;
    std::set<std::string> done;  // finished subcases of the current test case ("line:name")
    bool entered = false;        // a subcase ran in this pass
    std::string current;
};
inline State& state() {
    static State s;
    return s;
}
inline void report(const char* file, int line, const char* what, const char* expr) {
    ++state().failed_asserts;
    std::printf("%s:%d: ERROR: %s( %s ) failed  [in \"%s\"]\n", file, line, what, expr, state().current.c_str());
    std::fflush(stdout);
}
struct Subcase {
    std::string key;
    bool active = false;
    Subcase(const char* name, int line) : key(std::to_string(line) + ":" + name) {
        State& s = state();
        if (!s.entered && !s.done.count(key)) {
            s.entered = true;
            active = true;
        }
    }
    ~Subcase() {
        if (active) state().done.insert(key);
    }
    explicit operator bool() const { return active; }
};
}  // namespace detail

class Context {  // (the reference's CLI test drives doctest::Context; kept minimal)
  public:
    void applyCommandLine(int, char**) {}
    int run() { return run_all(); }
    static int run_all() {
        using namespace detail;
        int failed_cases = 0;
        for (const Case& c : registry()) {
            State& s = state();
            s.done.clear();
            s.current = c.name;
            const int before = s.failed_asserts;
            const auto t0 = std::chrono::steady_clock::now();
            for (int pass = 0; pass < 1000; ++pass) {  // one pass per leaf subcase
                s.entered = false;
                try {
                    c.fn();
                } catch (const RequireAbort&) {
                } catch (const std::exception& e) {
                    ++s.failed_asserts;
                    std::printf("%s:%d: ERROR: test case threw: %s  [in \"%s\"]\n", c.file, c.line, e.what(), c.name);
                } catch (...) {
                    ++s.failed_asserts;
                    std::printf("%s:%d: ERROR: test case threw an unknown exception  [in \"%s\"]\n", c.file, c.line, c.name);
                }
                if (!s.entered) break;
            }
            const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            const bool ok = s.failed_asserts == before;
            failed_cases += ok ? 0 : 1;
            std::printf("[%s] %s (%.2fs)\n", ok ? "PASS" : "FAIL", c.name, secs);
            std::fflush(stdout);
        }
        std::printf("[doctest-min] test cases: %zu | passed: %zu | failed: %d | assertions: %lld\n",
                    registry().size(), registry().size() - failed_cases, failed_cases, state().asserts);
        return failed_cases;
    }
};

}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                             \
    static void fn();                                                                                \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);        \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_CAT(doctest_sub_, __LINE__){name, __LINE__})

#define DOCTEST_ASSERT_IMPL(kind, cond_ok, text, on_fail)                                            \
    do {                                                                                             \
        ++::doctest::detail::state().asserts;                                                        \
        bool doctest_ok_ = false;                                                                    \
        try {                                                                                        \
            doctest_ok_ = (cond_ok);                                                                 \
        } catch (...) {                                                                              \
            doctest_ok_ = false;                                                                     \
        }                                                                                            \
        if (!doctest_ok_) {                                                                          \
            ::doctest::detail::report(__FILE__, __LINE__, kind, text);                               \
            on_fail;                                                                                 \
        }                                                                                            \
    } while (0)
#define CHECK(...) DOCTEST_ASSERT_IMPL("CHECK", static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, (void)0)
#define CHECK_FALSE(...) DOCTEST_ASSERT_IMPL("CHECK_FALSE", !static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, (void)0)
#define REQUIRE(...) \
    DOCTEST_ASSERT_IMPL("REQUIRE", static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, throw ::doctest::detail::RequireAbort{})
#define CHECK_THROWS(...)                                                                            \
    do {                                                                                             \
        ++::doctest::detail::state().asserts;                                                        \
        bool doctest_threw_ = false;                                                                 \
        try {                                                                                        \
            (void)(__VA_ARGS__);                                                                     \
        } catch (...) {                                                                              \
            doctest_threw_ = true;                                                                   \
        }                                                                                            \
        if (!doctest_threw_) ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS", #__VA_ARGS__); \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                   \
    do {                                                                                             \
        ++::doctest::detail::state().asserts;                                                        \
        int doctest_how_ = 0; /* 0 none, 1 right type, 2 other */                                    \
        try {                                                                                        \
            (void)(expr);                                                                            \
        } catch (const __VA_ARGS__&) {                                                               \
            doctest_how_ = 1;                                                                        \
        } catch (...) {                                                                              \
            doctest_how_ = 2;                                                                        \
        }                                                                                            \
        if (doctest_how_ != 1) ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr); \
    } while (0)
#define FAIL(msg)                                                                                    \
    do {                                                                                             \
        ::doctest::detail::report(__FILE__, __LINE__, "FAIL", msg);                                  \
        throw ::doctest::detail::RequireAbort{};                                                     \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::Context::run_all(); }
#endif

#endif
