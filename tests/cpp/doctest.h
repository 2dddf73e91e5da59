// Minimal doctest-compatible test harness (the reference's vendor/doctest.h
// is not shipped, ref:.gitignore:2).  Supports the subset the reference
// tests use: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, REQUIRE_MESSAGE,
// CAPTURE, FAIL, CHECK_THROWS_AS, CHECK_NOTHROW, doctest::Approx.
// Written for graphvx-b200; prints one line per failure and a summary
// "[doctest] test cases: N | passed: P | failed: F" that pytest parses.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    double value;
    double eps = 1e-5;
};
inline bool operator==(double lhs, const Approx& a) {
    const double scale = std::max(std::fabs(lhs), std::fabs(a.value));
    return std::fabs(lhs - a.value) <= a.eps * (1.0 + scale);
}
inline bool operator==(const Approx& a, double rhs) { return rhs == a; }

namespace detail {

struct Case {
    const char* name;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct RequireAbort {};

inline int& failures() {
    static int f = 0;
    return f;
}
inline std::vector<std::string>& captures() {
    static std::vector<std::string> c;
    return c;
}
inline const char*& current() {
    static const char* c = "";
    return c;
}

inline void report(const char* file, int line, const std::string& what) {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, current(), what.c_str());
    for (const std::string& c : captures()) std::fprintf(stderr, "    with %s\n", c.c_str());
}

struct Capture {
    template <typename T>
    Capture(const char* expr, const T& v) {
        std::ostringstream os;
        os << expr << " := " << v;
        captures().push_back(os.str());
    }
    ~Capture() { captures().pop_back(); }
};

inline int run_all() {
    int passed = 0, failed = 0;
    for (const Case& c : registry()) {
        current() = c.name;
        const int before = failures();
        try {
            c.fn();
        } catch (const RequireAbort&) {
        } catch (const std::exception& e) {
            report("<case>", 0, std::string("unexpected exception: ") + e.what());
        } catch (...) {
            report("<case>", 0, "unexpected non-standard exception");
        }
        captures().clear();
        if (failures() == before) ++passed;
        else ++failed;
    }
    std::printf("[doctest] test cases: %d | passed: %d | failed: %d\n", passed + failed, passed, failed);
    return failed ? 1 : 0;
}

} // namespace detail
} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_IMPL(fn, name)                                                                   \
    static void fn();                                                                                 \
    static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);                               \
    static void fn()
#define TEST_CASE(name) DOCTEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...)                                                                                    \
    do {                                                                                              \
        try {                                                                                         \
            if (!(__VA_ARGS__)) doctest::detail::report(__FILE__, __LINE__, "CHECK(" #__VA_ARGS__ ")"); \
        } catch (const std::exception& e) {                                                           \
            doctest::detail::report(__FILE__, __LINE__, std::string("exception in CHECK: ") + e.what()); \
        }                                                                                             \
    } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                                  \
    do {                                                                                              \
        if (!(__VA_ARGS__)) {                                                                         \
            doctest::detail::report(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")");                 \
            throw doctest::detail::RequireAbort{};                                                    \
        }                                                                                             \
    } while (0)
#define REQUIRE_MESSAGE(cond, msg)                                                                    \
    do {                                                                                              \
        if (!(cond)) {                                                                                \
            std::ostringstream doctest_os_;                                                           \
            doctest_os_ << "REQUIRE(" #cond ") " << (msg);                                            \
            doctest::detail::report(__FILE__, __LINE__, doctest_os_.str());                           \
            throw doctest::detail::RequireAbort{};                                                    \
        }                                                                                             \
    } while (0)
#define CAPTURE(x) doctest::detail::Capture DOCTEST_CAT(doctest_capture_, __LINE__)(#x, x)
#define FAIL(msg)                                                                                     \
    do {                                                                                              \
        doctest::detail::report(__FILE__, __LINE__, std::string("FAIL: ") + (msg));                   \
        throw doctest::detail::RequireAbort{};                                                        \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                                   \
    do {                                                                                              \
        bool doctest_ok_ = false;                                                                     \
        try {                                                                                         \
            (void)(expr);                                                                             \
        } catch (const type&) {                                                                       \
            doctest_ok_ = true;                                                                       \
        } catch (...) {                                                                               \
        }                                                                                             \
        if (!doctest_ok_) doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #type ")"); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                           \
    do {                                                                                              \
        try {                                                                                         \
            (void)(expr);                                                                             \
        } catch (const std::exception& e) {                                                           \
            doctest::detail::report(__FILE__, __LINE__, std::string("CHECK_NOTHROW(" #expr "): ") + e.what()); \
        }                                                                                             \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
