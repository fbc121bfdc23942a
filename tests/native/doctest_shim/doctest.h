// Minimal doctest-compatible test shim (TEST INFRASTRUCTURE). The reference's
// suites (/root/reference/proj/tests/*.cpp) include <doctest.h>, whose
// vendored copy is absent (proj/.gitignore: vendor/); this header implements
// the subset they use — TEST_CASE, CHECK, CHECK_THROWS, CHECK_THROWS_AS,
// CHECK_NOTHROW, FAIL, doctest::Approx(.epsilon/.scale) and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN — so those files compile UNMODIFIED
// against the drop-in headers (tests/test_gpu_ref_suites.py).
#pragma once

#include <algorithm>
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
    // doctest's rule: |a - b| < eps * (scale + max(|a|, |b|))
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v_) < b.eps_ * (b.scale_ + std::max(std::fabs(a), std::fabs(b.v_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
    friend bool operator!=(const Approx& b, double a) { return !(a == b); }

  private:
    double v_;
    double eps_ = 1.1920928955078125e-05;  // float epsilon * 100, doctest's default
    double scale_ = 1.0;
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
inline int& checks() {
    static int n = 0;
    return n;
}
inline int& failures() {
    static int n = 0;
    return n;
}
inline const char*& current() {
    static const char* c = "";
    return c;
}
struct Register {
    Register(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct fail_exception {};
inline void report(const char* file, int line, const char* what) {
    ++failures();
    std::printf("%s:%d: FAILED in \"%s\": %s\n", file, line, current(), what);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                            \
    static void fn();                                                               \
    static doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, &fn);              \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...)                                                                  \
    do {                                                                            \
        ++doctest::detail::checks();                                                \
        try {                                                                       \
            if (!(__VA_ARGS__)) doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__); \
        } catch (const std::exception& e_) {                                        \
            doctest::detail::report(__FILE__, __LINE__, e_.what());                 \
        }                                                                           \
    } while (0)
#define CHECK_THROWS(...)                                                           \
    do {                                                                            \
        ++doctest::detail::checks();                                                \
        bool thrown_ = false;                                                       \
        try {                                                                       \
            (void)(__VA_ARGS__);                                                    \
        } catch (...) {                                                             \
            thrown_ = true;                                                         \
        }                                                                           \
        if (!thrown_) doctest::detail::report(__FILE__, __LINE__, "no throw: " #__VA_ARGS__); \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                  \
    do {                                                                            \
        ++doctest::detail::checks();                                                \
        bool ok_ = false;                                                           \
        try {                                                                       \
            (void)(expr);                                                           \
        } catch (const __VA_ARGS__&) {                                              \
            ok_ = true;                                                             \
        } catch (...) {                                                             \
        }                                                                           \
        if (!ok_) doctest::detail::report(__FILE__, __LINE__, "expected " #__VA_ARGS__ " from " #expr); \
    } while (0)
#define CHECK_NOTHROW(...)                                                          \
    do {                                                                            \
        ++doctest::detail::checks();                                                \
        try {                                                                       \
            (void)(__VA_ARGS__);                                                    \
        } catch (const std::exception& e_) {                                        \
            doctest::detail::report(__FILE__, __LINE__, e_.what());                 \
        }                                                                           \
    } while (0)
#define FAIL(msg)                                                                   \
    do {                                                                            \
        doctest::detail::report(__FILE__, __LINE__, msg);                           \
        throw doctest::detail::fail_exception{};                                    \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    const char* only = argc > 1 ? argv[1] : nullptr;
    int ran = 0, failed_cases = 0;
    for (const auto& c : doctest::detail::registry()) {
        if (only && std::string(c.name).find(only) == std::string::npos) continue;
        doctest::detail::current() = c.name;
        const int before = doctest::detail::failures();
        try {
            c.fn();
        } catch (const doctest::detail::fail_exception&) {
        } catch (const std::exception& e) {
            doctest::detail::report("<test case>", 0, (std::string("uncaught exception: ") + e.what()).c_str());
        }
        ++ran;
        const bool bad = doctest::detail::failures() != before;
        failed_cases += bad;
        std::printf("[%s] %s\n", bad ? "FAIL" : " ok ", c.name);
    }
    std::printf("test cases: %d | %d passed | %d failed; checks: %d | %d failed\n", ran, ran - failed_cases,
                failed_cases, doctest::detail::checks(), doctest::detail::failures());
    return failed_cases ? 1 : 0;
}
#endif
