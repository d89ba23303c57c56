// TEST INFRASTRUCTURE ONLY — a minimal doctest-compatible header (our own code,
// not doctest) that is just enough to build and run the reference's UNMODIFIED
// unit tests (/root/reference/proj/tests/test_*.cpp): TEST_CASE, CHECK[_FALSE],
// REQUIRE[_MESSAGE], CHECK_THROWS_AS / _WITH_AS, CHECK_NOTHROW, CAPTURE and
// doctest::Approx. doctest itself is absent from the image.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    Approx& scale(double s) {
        scl = s;
        return *this;
    }
    double value;
    double eps = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scl = 1.0;
};
inline bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value) < rhs.eps * (rhs.scl + std::fmax(std::fabs(lhs), std::fabs(rhs.value)));
}
inline bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
inline bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
inline bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }
inline bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value || lhs == rhs; }
inline bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value || lhs == rhs; }
inline bool operator<(double lhs, const Approx& rhs) { return lhs < rhs.value && lhs != rhs; }
inline bool operator>(double lhs, const Approx& rhs) { return lhs > rhs.value && lhs != rhs; }

// CHECK_THROWS_WITH_AS matchers: a string matches what() exactly, Contains by substring
struct Contains {
    explicit Contains(std::string s) : str(std::move(s)) {}
    std::string str;
};
inline bool what_matches(const char* what, const Contains& c) { return std::string(what).find(c.str) != std::string::npos; }
inline bool what_matches(const char* what, const std::string& s) { return s == what; }
inline bool what_matches(const char* what, const char* s) { return std::string(s) == what; }

namespace detail {
struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};
struct RequireFailed {};
inline int& failed_checks() {
    static int n = 0;
    return n;
}
inline int& total_checks() {
    static int n = 0;
    return n;
}
inline void check(bool ok, const char* expr, const char* file, int line, bool require) {
    ++total_checks();
    if (ok) return;
    ++failed_checks();
    std::printf("%s:%d: %s FAILED: %s\n", file, line, require ? "REQUIRE" : "CHECK", expr);
    if (require) throw RequireFailed{};
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                                      \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                                        \
    static ::doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(name, __FILE__, __LINE__,         \
                                                                            &DOCTEST_CAT(doctest_fn_, __LINE__)); \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::check(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_MESSAGE(cond, msg) ::doctest::detail::check(static_cast<bool>(cond), #cond, __FILE__, __LINE__, true)
#define CAPTURE(x) ((void)0)
#define DOCTEST_THROWS_IMPL_(expr, Type, require)                                                            \
    do {                                                                                                     \
        bool doctest_ok_ = false;                                                                            \
        try {                                                                                                \
            (void)(expr);                                                                                    \
        } catch (const Type&) {                                                                              \
            doctest_ok_ = true;                                                                              \
        } catch (...) {                                                                                      \
        }                                                                                                    \
        ::doctest::detail::check(doctest_ok_, "throws " #Type ": " #expr, __FILE__, __LINE__, require);      \
    } while (0)
#define CHECK_THROWS_AS(expr, Type) DOCTEST_THROWS_IMPL_(expr, Type, false)
#define CHECK_THROWS_WITH_AS(expr, msg, Type)                                                                \
    do {                                                                                                     \
        bool doctest_ok_ = false;                                                                            \
        try {                                                                                                \
            (void)(expr);                                                                                    \
        } catch (const Type& e_) {                                                                           \
            doctest_ok_ = ::doctest::what_matches(e_.what(), msg);                                           \
        } catch (...) {                                                                                      \
        }                                                                                                    \
        ::doctest::detail::check(doctest_ok_, "throws " #Type " with " #msg ": " #expr, __FILE__, __LINE__,  \
                                 false);                                                                     \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                                  \
    do {                                                                                                     \
        bool doctest_ok_ = true;                                                                             \
        try {                                                                                                \
            (void)(expr);                                                                                    \
        } catch (...) {                                                                                      \
            doctest_ok_ = false;                                                                             \
        }                                                                                                    \
        ::doctest::detail::check(doctest_ok_, "nothrow: " #expr, __FILE__, __LINE__, false);                 \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0;
    for (const auto& tc : ::doctest::detail::registry()) {
        const int before = ::doctest::detail::failed_checks();
        try {
            tc.fn();
        } catch (const ::doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            ++::doctest::detail::failed_checks();
            std::printf("%s:%d: TEST CASE '%s' threw: %s\n", tc.file, tc.line, tc.name, e.what());
        }
        if (::doctest::detail::failed_checks() != before) {
            ++failed_cases;
            std::printf("FAILED test case: %s\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks: %d | %d failed\n",
                ::doctest::detail::registry().size(), ::doctest::detail::registry().size() - failed_cases,
                failed_cases, ::doctest::detail::total_checks(), ::doctest::detail::failed_checks());
    return failed_cases ? 1 : 0;
}
#endif
