// TEST INFRASTRUCTURE — oracle only.
//
// Minimal restatement of the doctest macros the reference's two real unit
// test files use (proj/tests/test_dag_model.cpp, test_exec_model.cpp):
// TEST_CASE, CHECK, CHECK_THROWS, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS and
// doctest::Contains. doctest.h itself lived in the reference's git-ignored
// vendor/ directory (proj/.gitignore:2) and is absent from this image.
// With DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN (proj/tests/doctest_main.cpp:1) a
// main() runs every registered case and exits non-zero on any failed check.
#pragma once

#include <cstdio>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

struct Contains {
    std::string needle;
    explicit Contains(const char* s) : needle(s) {}
    bool matches(const std::string& msg) const { return msg.find(needle) != std::string::npos; }
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
inline long& failures() {
    static long f = 0;
    return f;
}
inline long& checks() {
    static long c = 0;
    return c;
}
struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
inline void fail(const char* file, int line, const char* expr, const char* why) {
    ++failures();
    std::fprintf(stderr, "%s:%d: CHECK FAILED (%s): %s\n", file, line, why, expr);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)

#define TEST_CASE(name)                                                             \
    static void DOCTEST_SHIM_CAT(doctest_case_, __LINE__)();                        \
    static ::doctest::detail::Registrar DOCTEST_SHIM_CAT(doctest_reg_, __LINE__)(   \
        name, &DOCTEST_SHIM_CAT(doctest_case_, __LINE__));                          \
    static void DOCTEST_SHIM_CAT(doctest_case_, __LINE__)()

#define CHECK(...)                                                                  \
    do {                                                                            \
        ++::doctest::detail::checks();                                              \
        bool doctest_ok_ = false;                                                   \
        try {                                                                       \
            doctest_ok_ = static_cast<bool>(__VA_ARGS__);                           \
        } catch (...) {                                                             \
            ::doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__, "threw");     \
            break;                                                                  \
        }                                                                           \
        if (!doctest_ok_)                                                           \
            ::doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__, "false");     \
    } while (0)

#define CHECK_THROWS(...)                                                           \
    do {                                                                            \
        ++::doctest::detail::checks();                                              \
        bool doctest_threw_ = false;                                                \
        try {                                                                       \
            (void)(__VA_ARGS__);                                                    \
        } catch (...) {                                                             \
            doctest_threw_ = true;                                                  \
        }                                                                           \
        if (!doctest_threw_)                                                        \
            ::doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__, "no throw");  \
    } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                  \
    do {                                                                            \
        ++::doctest::detail::checks();                                              \
        int doctest_state_ = 0;                                                     \
        try {                                                                       \
            (void)(expr);                                                           \
        } catch (const __VA_ARGS__&) {                                              \
            doctest_state_ = 1;                                                     \
        } catch (...) {                                                             \
            doctest_state_ = 2;                                                     \
        }                                                                           \
        if (doctest_state_ != 1)                                                    \
            ::doctest::detail::fail(__FILE__, __LINE__, #expr,                      \
                                    doctest_state_ ? "wrong exception type"         \
                                                   : "no throw");                   \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, with, ...)                                       \
    do {                                                                            \
        ++::doctest::detail::checks();                                              \
        int doctest_state_ = 0;                                                     \
        try {                                                                       \
            (void)(expr);                                                           \
        } catch (const __VA_ARGS__& e) {                                            \
            doctest_state_ = (with).matches(e.what()) ? 1 : 3;                      \
        } catch (...) {                                                             \
            doctest_state_ = 2;                                                     \
        }                                                                           \
        if (doctest_state_ != 1)                                                    \
            ::doctest::detail::fail(__FILE__, __LINE__, #expr,                      \
                                    doctest_state_ == 3   ? "message mismatch"      \
                                    : doctest_state_ == 2 ? "wrong exception type"  \
                                                          : "no throw");            \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    for (const auto& c : ::doctest::detail::registry()) {
        long before = ::doctest::detail::failures();
        try {
            c.fn();
        } catch (const std::exception& e) {
            ++::doctest::detail::failures();
            std::fprintf(stderr, "TEST_CASE \"%s\" threw: %s\n", c.name, e.what());
        }
        std::printf("[%s] %s\n", ::doctest::detail::failures() == before ? "ok" : "FAIL",
                    c.name);
    }
    std::printf("test cases: %zu, checks: %ld, failed: %ld\n",
                ::doctest::detail::registry().size(), ::doctest::detail::checks(),
                ::doctest::detail::failures());
    return ::doctest::detail::failures() == 0 ? 0 : 1;
}
#endif
