// mini_test.hpp — the handful of doctest-style macros the executor tests use (TEST_CASE,
// CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS), so the C++ parity tests read like the
// reference's own doctest suites. Cases tagged "[gpu]" need a CUDA device; run with
// --cpu-only to execute just the host-side cases.
#pragma once
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

namespace mini {
struct Case {
    const char* name;
    std::function<void()> fn;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
inline int& failures() {
    static int f = 0;
    return f;
}
struct Reg {
    Reg(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
struct Abort {};
inline void fail(const char* file, int line, const char* expr, bool fatal) {
    std::printf("  FAIL %s:%d: %s\n", file, line, expr);
    ++failures();
    if (fatal) throw Abort{};
}
inline int run(int argc, char** argv) {
    const bool cpu_only = argc > 1 && std::strcmp(argv[1], "--cpu-only") == 0;
    int cases = 0, failed_cases = 0;
    for (auto& c : registry()) {
        if (cpu_only && std::strstr(c.name, "[gpu]")) continue;
        const int before = failures();
        ++cases;
        try {
            c.fn();
        } catch (Abort&) {
        } catch (std::exception& e) {
            std::printf("  FAIL unexpected exception: %s\n", e.what());
            ++failures();
        }
        const bool ok = failures() == before;
        failed_cases += !ok;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("%d cases, %d failed, %d failed checks\n", cases, failed_cases, failures());
    return failures() == 0 ? 0 : 1;
}
}  // namespace mini

#define MINI_CAT2(a, b) a##b
#define MINI_CAT(a, b) MINI_CAT2(a, b)
#define TEST_CASE(name)                                                        \
    static void MINI_CAT(mini_case_, __LINE__)();                              \
    static mini::Reg MINI_CAT(mini_reg_, __LINE__)(name, MINI_CAT(mini_case_, __LINE__)); \
    static void MINI_CAT(mini_case_, __LINE__)()
#define CHECK(expr) \
    do { if (!(expr)) mini::fail(__FILE__, __LINE__, #expr, false); } while (0)
#define CHECK_FALSE(expr) CHECK(!(expr))
#define REQUIRE(expr) \
    do { if (!(expr)) mini::fail(__FILE__, __LINE__, #expr, true); } while (0)
#define CHECK_THROWS_AS(expr, type)                                          \
    do {                                                                     \
        bool thrown_ = false;                                                \
        try { (void)(expr); } catch (const type&) { thrown_ = true; } catch (...) {} \
        if (!thrown_) mini::fail(__FILE__, __LINE__, #expr " throws " #type, false); \
    } while (0)
