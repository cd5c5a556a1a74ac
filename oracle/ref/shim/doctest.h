// ORACLE bridge — a minimal doctest-compatible harness, enough to compile and
// run the reference's own unit suites (proj/tests/test_*.cpp) unchanged. The
// real doctest.h lives in the reference's gitignored vendor/ directory
// (proj/.gitignore:2) and is absent here. Supports TEST_SUITE / TEST_CASE /
// CHECK / REQUIRE / CHECK_THROWS_AS and doctest::Approx. Suite names are
// cosmetic: the runner executes every registered case.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <vector>

namespace lpo_dt {

struct Case {
    const char* name;
    void (*fn)();
    const char* file;
};

inline std::vector<Case>& cases() {
    static std::vector<Case> v;
    return v;
}

struct State {
    long checks = 0, failures = 0;
};
inline State& state() {
    static State s;
    return s;
}

struct Reg {
    Reg(const char* n, void (*f)(), const char* file) { cases().push_back({n, f, file}); }
};

struct RequireFailed {};

inline bool record(bool ok, const char* expr, const char* file, int line) {
    ++state().checks;
    if (!ok) {
        ++state().failures;
        std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
    }
    return ok;
}

}  // namespace lpo_dt

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
    bool matches(double x) const {
        return std::fabs(x - v_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(v_)));
    }
    friend bool operator==(double x, const Approx& a) { return a.matches(x); }
    friend bool operator==(const Approx& a, double x) { return a.matches(x); }
    friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
    friend bool operator!=(const Approx& a, double x) { return !a.matches(x); }

private:
    double v_;
    double eps_ = double(std::numeric_limits<float>::epsilon()) * 100.0;
    double scale_ = 1.0;
};

}  // namespace doctest

#define LPO_DT_CAT_(a, b) a##b
#define LPO_DT_CAT(a, b) LPO_DT_CAT_(a, b)

#define TEST_SUITE(name) namespace LPO_DT_CAT(lpo_dt_suite_, __COUNTER__)
#define TEST_SUITE_BEGIN(name) static_assert(true, "")
#define TEST_SUITE_END() static_assert(true, "")

#define LPO_DT_CASE(name, fn)                                              \
    static void fn();                                                      \
    static ::lpo_dt::Reg LPO_DT_CAT(fn, _reg)(name, &fn, __FILE__);        \
    static void fn()
#define TEST_CASE(name) LPO_DT_CASE(name, LPO_DT_CAT(lpo_dt_case_, __COUNTER__))

#define CHECK(...) ::lpo_dt::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                       \
    do {                                                                                   \
        if (!::lpo_dt::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)) \
            throw ::lpo_dt::RequireFailed{};                                               \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                        \
    do {                                                                                   \
        bool lpo_dt_ok = false;                                                            \
        try {                                                                              \
            (void)(expr);                                                                  \
        } catch (const type&) {                                                            \
            lpo_dt_ok = true;                                                              \
        } catch (...) {                                                                    \
        }                                                                                  \
        ::lpo_dt::record(lpo_dt_ok, "THROWS_AS(" #expr ", " #type ")", __FILE__, __LINE__); \
    } while (0)

#ifdef LPO_DOCTEST_MAIN
int main() {
    long failed_cases = 0;
    for (const auto& c : ::lpo_dt::cases()) {
        const long before = ::lpo_dt::state().failures;
        bool threw = false;
        try {
            c.fn();
        } catch (const ::lpo_dt::RequireFailed&) {
            threw = true;
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s: exception: %s\n", c.name, e.what());
            ++::lpo_dt::state().failures;
            threw = true;
        }
        const bool ok = !threw && ::lpo_dt::state().failures == before;
        if (!ok) ++failed_cases;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("cases: %zu  failed: %ld  checks: %ld  failed checks: %ld\n", ::lpo_dt::cases().size(),
                failed_cases, ::lpo_dt::state().checks, ::lpo_dt::state().failures);
    return failed_cases == 0 ? 0 : 1;
}
#endif
