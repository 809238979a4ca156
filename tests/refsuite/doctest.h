// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE ONLY).
//
// The reference's tests (/root/reference/proj/tests) are written against doctest,
// which is not vendored in the reference tree. This shim provides the subset they
// use -- TEST_CASE, CHECK, REQUIRE, CHECK_THROWS, MESSAGE, doctest::Approx with
// .epsilon() -- so the reference's own test files compile unmodified against the
// B200 drop-in headers (include/krplev/*.hpp) and run on the device
// (oracle/Makefile target `refsuite`, tests/test_refsuite.py).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
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
    // doctest's rule: |a - b| < eps * (scale + max(|a|, |b|)), scale = 1
    bool match(double a) const { return std::fabs(a - v_) < eps_ * (1.0 + std::max(std::fabs(a), std::fabs(v_))); }
    friend bool operator==(double a, const Approx& b) { return b.match(a); }
    friend bool operator==(const Approx& b, double a) { return b.match(a); }
    friend bool operator!=(double a, const Approx& b) { return !b.match(a); }
    friend bool operator!=(const Approx& b, double a) { return !b.match(a); }

private:
    double v_;
    double eps_ = 100.0 * 1.1920928955078125e-07;  // 100 * FLT_EPSILON
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
struct Registrar {
    Registrar(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct RequireFailed {};
inline int& failures() {
    static int f = 0;
    return f;
}
inline int& checks() {
    static int c = 0;
    return c;
}
inline void report(const char* file, int line, const char* expr) {
    ++failures();
    std::fprintf(stderr, "  %s:%d: CHECK failed: %s\n", file, line, expr);
}
template <class... A>
inline void message(A&&... a) {
    std::ostringstream os;
    (os << ... << a);
    std::fprintf(stderr, "  MESSAGE: %s\n", os.str().c_str());
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                         \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                           \
    static ::doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_fn_, __LINE__)); \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define CHECK(...)                                                                    \
    do {                                                                              \
        ++::doctest::detail::checks();                                                \
        if (!(__VA_ARGS__)) ::doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__); \
    } while (0)
#define REQUIRE(...)                                                                  \
    do {                                                                              \
        ++::doctest::detail::checks();                                                \
        if (!(__VA_ARGS__)) {                                                         \
            ::doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);              \
            throw ::doctest::detail::RequireFailed{};                                 \
        }                                                                             \
    } while (0)
#define CHECK_THROWS(...)                                                             \
    do {                                                                              \
        ++::doctest::detail::checks();                                                \
        bool thrown_ = false;                                                         \
        try {                                                                         \
            (void)(__VA_ARGS__);                                                      \
        } catch (...) {                                                               \
            thrown_ = true;                                                           \
        }                                                                             \
        if (!thrown_) ::doctest::detail::report(__FILE__, __LINE__, "throws: " #__VA_ARGS__); \
    } while (0)
#define MESSAGE(...) ::doctest::detail::message(__VA_ARGS__)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
// Runs every registered case; a case whose name matches an entry of the
// REFSUITE_SKIP environment variable (';'-separated substrings) is reported as
// skipped. Exit status 0 iff no check failed and no case threw.
int main() {
    using namespace doctest::detail;
    std::vector<std::string> skip;
    if (const char* s = std::getenv("REFSUITE_SKIP")) {
        std::string all(s), cur;
        for (char c : all) {
            if (c == ';') {
                if (!cur.empty()) skip.push_back(cur);
                cur.clear();
            } else {
                cur += c;
            }
        }
        if (!cur.empty()) skip.push_back(cur);
    }
    int cases = 0, failed_cases = 0, skipped = 0;
    for (const Case& c : registry()) {
        bool sk = false;
        for (const std::string& pat : skip) sk |= std::strstr(c.name, pat.c_str()) != nullptr;
        if (sk) {
            ++skipped;
            std::printf("SKIP  %s\n", c.name);
            continue;
        }
        ++cases;
        const int before = failures();
        bool threw = false;
        try {
            c.fn();
        } catch (const RequireFailed&) {
            threw = true;
        } catch (const std::exception& e) {
            threw = true;
            std::fprintf(stderr, "  unexpected exception: %s\n", e.what());
        } catch (...) {
            threw = true;
        }
        const bool ok = !threw && failures() == before;
        if (!ok) ++failed_cases;
        std::printf("%s  %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("refsuite: %d cases, %d failed, %d skipped, %d checks, %d failed checks\n", cases, failed_cases,
                skipped, checks(), failures());
    return failed_cases ? 1 : 0;
}
#endif
