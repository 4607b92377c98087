// Minimal Catch2-v3-compatible test shim (TEST INFRASTRUCTURE ONLY).
//
// Catch2 is not installed in this image, and the reference's test build
// (proj/tests/CMakeLists.txt:3) expects /usr/local/include/catch2/.  This shim
// implements exactly the macro surface the reference tests use (SURVEY.md §4:
// TEST_CASE, CHECK, REQUIRE, CHECK_FALSE, REQUIRE_FALSE, CHECK_THROWS_AS, INFO,
// Catch::Approx(x).margin(m)) so the reference's own tests compile UNMODIFIED
// from /root/reference/proj/tests and pin the oracle (oracle/Makefile).
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace Catch {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& margin(double m) {
        margin_ = m;
        return *this;
    }
    Approx& epsilon(double e) {
        epsilon_ = e;
        return *this;
    }
    bool matches(double other) const {
        // Catch2 v3 semantics: |a-b| <= margin  OR  |a-b| <= eps * (scale + max(|a|,|b|))
        double diff = std::fabs(other - value_);
        if (diff <= margin_) return true;
        return diff <= epsilon_ * (scale_ + std::fmax(std::fabs(value_), std::fabs(other)));
    }
    friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
    friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }
    friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || rhs.matches(lhs); }
    friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || rhs.matches(lhs); }

private:
    double value_;
    double margin_ = 0.0;
    double epsilon_ = static_cast<double>(FLT_EPSILON) * 100.0;
    double scale_ = 0.0;
};

namespace shim {

struct RequireAbort {};

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
    long checks = 0;
    long failures = 0;
    bool case_failed = false;
    std::string info;
};

inline State& state() {
    static State s;
    return s;
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    State& s = state();
    ++s.checks;
    if (ok) return;
    ++s.failures;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED %s(%s)%s%s\n", file, line, kind, expr,
                 s.info.empty() ? "" : "  with: ", s.info.c_str());
}

}  // namespace shim
}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_TEST_IMPL(fn, name)                                                  \
    static void fn();                                                                   \
    static ::Catch::shim::Registrar CATCH_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
    static void fn()
#define TEST_CASE(name, ...) CATCH_SHIM_TEST_IMPL(CATCH_SHIM_CAT(catch_shim_case_, __LINE__), name)

#define CHECK(...) ::Catch::shim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    ::Catch::shim::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                              \
    do {                                                                                          \
        bool catch_shim_ok = static_cast<bool>(__VA_ARGS__);                                      \
        ::Catch::shim::report(catch_shim_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);        \
        if (!catch_shim_ok) throw ::Catch::shim::RequireAbort{};                                 \
    } while (0)
#define REQUIRE_FALSE(...)                                                                        \
    do {                                                                                          \
        bool catch_shim_ok = !static_cast<bool>(__VA_ARGS__);                                     \
        ::Catch::shim::report(catch_shim_ok, "REQUIRE_FALSE", #__VA_ARGS__, __FILE__, __LINE__);  \
        if (!catch_shim_ok) throw ::Catch::shim::RequireAbort{};                                 \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                 \
    do {                                                                            \
        bool catch_shim_ok = false;                                                 \
        try {                                                                       \
            (void)(expr);                                                           \
        } catch (const type&) {                                                     \
            catch_shim_ok = true;                                                   \
        } catch (...) {                                                             \
        }                                                                           \
        ::Catch::shim::report(catch_shim_ok, "CHECK_THROWS_AS", #expr ", " #type, __FILE__, __LINE__); \
    } while (0)
#define INFO(...)                                          \
    do {                                                   \
        std::ostringstream catch_shim_os;                  \
        catch_shim_os << __VA_ARGS__;                      \
        ::Catch::shim::state().info = catch_shim_os.str(); \
    } while (0)
