// Minimal doctest-compatible shim -- TEST INFRASTRUCTURE ONLY.
// The reference test suite (/root/reference/proj/tests) is written against
// doctest, which the reference does not vendor (proj/.gitignore ignores
// /vendor/).  This shim implements just the macros those tests use so the
// unmodified reference tests can run as the oracle gate (oracle/Makefile).
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {
class Approx {
  public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    friend bool operator==(double a, const Approx& b) {
        double m = std::fabs(a) > std::fabs(b.v_) ? std::fabs(a) : std::fabs(b.v_);
        return std::fabs(a - b.v_) < b.eps_ * (1.0 + m);
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }

  private:
    double v_;
    double eps_ = 1.1920928955078125e-05 * 100;
};
}  // namespace doctest

namespace doctest_shim {
struct Case {
    const char* name;
    void (*fn)();
};
struct RequireFailed {};
inline std::vector<Case>& cases() {
    static std::vector<Case> v;
    return v;
}
inline int reg(void (*fn)(), const char* name) {
    cases().push_back({name, fn});
    return 0;
}
struct State {
    long checks = 0;
    long failures = 0;
    int target = 0;   // subcase index entered in this pass
    int seen = 0;     // subcases met in this pass
};
inline State& st() {
    static State s;
    return s;
}
inline bool enter_subcase() { return st().seen++ == st().target; }
inline void report(bool ok, const char* expr, const char* file, int line, bool req) {
    st().checks++;
    if (!ok) {
        st().failures++;
        std::fprintf(stderr, "%s:%d: FAILED %s: %s\n", file, line,
                     req ? "REQUIRE" : "CHECK", expr);
        if (req) throw RequireFailed{};
    }
}
inline int run_all() {
    int failed_cases = 0;
    for (auto& c : cases()) {
        long before = st().failures;
        for (int pass = 0;; ++pass) {
            st().target = pass;
            st().seen = 0;
            try {
                c.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                st().failures++;
                std::fprintf(stderr, "test '%s': exception %s\n", c.name, e.what());
            }
            if (st().seen <= pass + 1) break;
        }
        if (st().failures != before) {
            ++failed_cases;
            std::fprintf(stderr, "test case FAILED: %s\n", c.name);
        }
    }
    std::printf("cases=%zu failed_cases=%d checks=%ld failures=%ld\n",
                cases().size(), failed_cases, st().checks, st().failures);
    return failed_cases == 0 ? 0 : 1;
}
}  // namespace doctest_shim

#define DS_CAT2(a, b) a##b
#define DS_CAT(a, b) DS_CAT2(a, b)
#define DS_TEST_IMPL(fn, name)                                              \
    static void fn();                                                       \
    static int DS_CAT(fn, _reg) = doctest_shim::reg(fn, name);              \
    static void fn()
#define TEST_CASE(name) DS_TEST_IMPL(DS_CAT(ds_case_, __COUNTER__), name)
#define SUBCASE(name) if (doctest_shim::enter_subcase())
#define CHECK(...) doctest_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest_shim::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_FALSE(...) doctest_shim::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)
#define REQUIRE_MESSAGE(cond, ...) doctest_shim::report(static_cast<bool>(cond), #cond, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                          \
    do {                                                                     \
        bool ds_ok = false;                                                  \
        try { (void)(expr); } catch (const type&) { ds_ok = true; } catch (...) {} \
        doctest_shim::report(ds_ok, "throws " #type ": " #expr, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                  \
    do {                                                                     \
        bool ds_ok = true;                                                   \
        try { (void)(expr); } catch (...) { ds_ok = false; }                 \
        doctest_shim::report(ds_ok, "nothrow: " #expr, __FILE__, __LINE__, false); \
    } while (0)
#define INFO(...) do {} while (0)
#define CAPTURE(...) do {} while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest_shim::run_all(); }
#endif
