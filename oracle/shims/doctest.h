// oracle/shims/doctest.h -- TEST INFRASTRUCTURE ONLY.
//
// A from-scratch stand-in for the handful of doctest features the reference's
// own test suite uses (/root/reference/proj/tests/*.cpp): TEST_CASE,
// TEST_CASE_TEMPLATE, CHECK, CHECK_FALSE, CHECK_THROWS_AS, CHECK_NOTHROW,
// REQUIRE and doctest::Approx(..).epsilon(..). doctest.h itself is expected
// under proj/vendor/, which is git-ignored and absent (proj/.gitignore:2).
// This lets the compiled reference (oracle/_ref) run its 61 known-answer and
// property tests, which pins the FFTW shim and the oracle build.
//
// Approx follows doctest's documented comparison:
//   |a - b| < eps * (scale + max(|a|, |b|)), eps default 100 * FLT_EPSILON, scale 1.
// CLI: -tc=<pattern> runs only test cases whose name matches (`*` wildcard).
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <typeinfo>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool matches(double other) const {
        return std::fabs(other - value_) <
               eps_ * (scale_ + std::max(std::fabs(other), std::fabs(value_)));
    }
    friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
    friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }
    friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || rhs.matches(lhs); }
    friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || rhs.matches(lhs); }

private:
    double value_;
    double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
    double scale_ = 1.0;
};

namespace detail {

struct TestCase {
    std::string name;
    std::function<void()> fn;
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct State {
    long checks = 0;
    long failures = 0;
    const char* current = "";
};
inline State& state() {
    static State s;
    return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    ++state().checks;
    if (!ok) {
        ++state().failures;
        std::fprintf(stderr, "%s:%d: FAILED %s( %s ) in test case \"%s\"\n", file, line, kind,
                     expr, state().current);
    }
}

struct Registrar {
    Registrar(const char* name, std::function<void()> fn) {
        registry().push_back({name, std::move(fn)});
    }
};

template <typename T>
struct TypeTag {
    using type = T;
};

template <typename... Ts>
struct TemplateRegistrar {
    template <typename F>
    TemplateRegistrar(const char* name, F f) {
        (registry().push_back({std::string(name) + "<" + typeid(Ts).name() + ">",
                               [f]() { f(TypeTag<Ts>{}); }}),
         ...);
    }
};

inline bool wildcard(const char* pat, const char* s) {
    if (*pat == 0) return *s == 0;
    if (*pat == '*') return wildcard(pat + 1, s) || (*s && wildcard(pat, s + 1));
    return *s && (*pat == *s) && wildcard(pat + 1, s + 1);
}

inline int run_all(int argc, char** argv) {
    std::vector<std::string> filters;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "-tc=", 4) == 0) filters.push_back(argv[i] + 4);
    int ran = 0, failed_cases = 0;
    for (auto& tc : registry()) {
        if (!filters.empty()) {
            bool any = false;
            for (auto& f : filters) any = any || wildcard(f.c_str(), tc.name.c_str());
            if (!any) continue;
        }
        ++ran;
        state().current = tc.name.c_str();
        const long before = state().failures;
        try {
            tc.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++state().failures;
            std::fprintf(stderr, "test case \"%s\" threw: %s\n", tc.name.c_str(), e.what());
        }
        const bool ok = state().failures == before;
        if (!ok) ++failed_cases;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", tc.name.c_str());
        std::fflush(stdout);
    }
    std::printf("test cases: %d | %d passed | %d failed ; assertions: %ld | %ld failed\n", ran,
                ran - failed_cases, failed_cases, state().checks, state().failures);
    return failed_cases == 0 ? 0 : 1;
}

} // namespace detail
} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define TEST_CASE(name)                                                                            \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                              \
    static ::doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(                       \
        name, &DOCTEST_CAT(doctest_fn_, __LINE__));                                                \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define TEST_CASE_TEMPLATE(name, T, ...)                                                           \
    template <typename T>                                                                          \
    static void DOCTEST_CAT(doctest_tfn_, __LINE__)();                                             \
    static ::doctest::detail::TemplateRegistrar<__VA_ARGS__> DOCTEST_CAT(doctest_treg_, __LINE__)( \
        name, [](auto tag) { DOCTEST_CAT(doctest_tfn_, __LINE__)<typename decltype(tag)::type>(); }); \
    template <typename T>                                                                          \
    static void DOCTEST_CAT(doctest_tfn_, __LINE__)()

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                               \
    do {                                                                                           \
        bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                         \
        ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);       \
        if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                                \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                 \
    do {                                                                                           \
        bool doctest_ok_ = false;                                                                  \
        try {                                                                                      \
            (void)(expr);                                                                          \
        } catch (const __VA_ARGS__&) {                                                             \
            doctest_ok_ = true;                                                                    \
        } catch (...) {                                                                            \
        }                                                                                          \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);      \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                        \
    do {                                                                                           \
        bool doctest_ok_ = true;                                                                   \
        try {                                                                                      \
            (void)(expr);                                                                          \
        } catch (...) {                                                                            \
            doctest_ok_ = false;                                                                   \
        }                                                                                          \
        ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__);        \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run_all(argc, argv); }
#endif
