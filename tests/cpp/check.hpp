// Minimal check harness for the C++ drop-in programs (doctest is not vendored here).
#pragma once
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace kwcheck {
inline int& failures() { static int f = 0; return f; }
inline int& checks() { static int c = 0; return c; }
inline std::vector<std::pair<std::string, std::function<void()>>>& cases()
{
    static std::vector<std::pair<std::string, std::function<void()>>> v;
    return v;
}
struct Reg {
    Reg(const char* n, std::function<void()> f) { cases().emplace_back(n, std::move(f)); }
};
inline int run()
{
    for (auto& [name, fn] : cases()) {
        const int before = failures();
        try {
            fn();
        }
        catch (const std::exception& e) {
            ++failures();
            std::printf("  exception in '%s': %s\n", name.c_str(), e.what());
        }
        std::printf("[%s] %s\n", failures() == before ? "PASS" : "FAIL", name.c_str());
    }
    std::printf("%d checks, %d failures\n", checks(), failures());
    return failures() == 0 ? 0 : 1;
}
} // namespace kwcheck

#define KW_CAT2(a, b) a##b
#define KW_CAT(a, b) KW_CAT2(a, b)
#define TEST_CASE(name) \
    static void KW_CAT(tc_, __LINE__)(); \
    static kwcheck::Reg KW_CAT(reg_, __LINE__)(name, KW_CAT(tc_, __LINE__)); \
    static void KW_CAT(tc_, __LINE__)()
#define CHECK(cond) \
    do { \
        ++kwcheck::checks(); \
        if (!(cond)) { \
            ++kwcheck::failures(); \
            std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        } \
    } while (0)
#define CHECK_THROWS_AS(expr, ex) \
    do { \
        ++kwcheck::checks(); \
        bool caught_ = false; \
        try { expr; } catch (const ex&) { caught_ = true; } catch (...) {} \
        if (!caught_) { \
            ++kwcheck::failures(); \
            std::printf("  CHECK_THROWS_AS failed %s:%d: %s\n", __FILE__, __LINE__, #expr); \
        } \
    } while (0)
