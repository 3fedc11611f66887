// doctest.h — a minimal stand-in for the doctest subset the reference's tests use (the vendored
// doctest is absent: proj/.gitignore:2), so /root/reference/proj/tests/*.cpp compile UNMODIFIED
// against this repo's C++ mirror (include/pipesim_b200). Supports TEST_CASE, CHECK, CHECK_FALSE,
// REQUIRE, CHECK_THROWS_AS, doctest::Approx(..).epsilon(..), DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
// Prints one "[PASS]/[FAIL] <case> (<failed> of <checks> checks)" line per test case, the first
// failing expression of each, and a final tally; the exit code is the number of failed cases.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
    double v, eps = 1e-5;
    explicit Approx(double x) : v(x) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v) <= b.eps * (1.0 + std::fmax(std::fabs(a), std::fabs(b.v)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
};
namespace detail {
struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& cases() {
    static std::vector<Case> c;
    return c;
}
struct State {
    int checks = 0, failed = 0;
    std::string first;
};
inline State& state() {
    static State s;
    return s;
}
struct RequireFailed {};
inline void record(bool ok, const char* expr, const char* file, int line, bool require) {
    auto& s = state();
    ++s.checks;
    if (ok) return;
    ++s.failed;
    if (s.first.empty()) s.first = std::string(file) + ":" + std::to_string(line) + ": " + expr;
    if (require) throw RequireFailed{};
}
struct Registrar {
    Registrar(const char* name, void (*fn)()) { cases().push_back({name, fn}); }
};
inline int run_all() {
    int failed_cases = 0;
    for (const auto& c : cases()) {
        state() = State{};
        std::string err;
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            err = std::string("exception: ") + e.what();
        } catch (...) {
            err = "unknown exception";
        }
        const auto& s = state();
        const bool ok = s.failed == 0 && err.empty();
        failed_cases += ok ? 0 : 1;
        std::printf("[%s] %s (%d of %d checks failed)%s%s%s%s\n", ok ? "PASS" : "FAIL", c.name, s.failed, s.checks,
                    s.first.empty() ? "" : " first: ", s.first.c_str(), err.empty() ? "" : " ", err.c_str());
    }
    std::printf("%zu test cases, %d failed\n", cases().size(), failed_cases);
    return failed_cases;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, name)                                                  \
    static void fn();                                                            \
    static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);         \
    static void fn()
#define TEST_CASE(name) DOCTEST_CASE_(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define CHECK(...) doctest::detail::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::detail::record(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                             \
    do {                                                                                        \
        bool caught_ = false;                                                                   \
        try {                                                                                   \
            (void)(expr);                                                                       \
        } catch (const type&) {                                                                 \
            caught_ = true;                                                                     \
        } catch (...) {                                                                         \
        }                                                                                       \
        doctest::detail::record(caught_, "throws " #type ": " #expr, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
