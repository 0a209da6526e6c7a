// doctest-subset shim so the reference's own unit tests compile against the
// reference build in oracle/_ref — TEST INFRASTRUCTURE.  doctest is vendored
// by the reference under proj/vendor/ (git-ignored, absent).  Provides the
// macros the reference tests use: TEST_CASE, SUBCASE (re-run-per-leaf
// semantics), CHECK*, REQUIRE*, CHECK_THROWS_AS / _WITH_AS, CHECK_NOTHROW,
// CAPTURE, INFO, FAIL, doctest::Approx (doctest's relative-epsilon rule) and
// doctest::Contains.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <set>
#include <string>
#include <vector>

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
    friend bool operator==(double lhs, const Approx& r) {
        return std::fabs(lhs - r.v_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.v_)));
    }
    friend bool operator==(const Approx& r, double lhs) { return lhs == r; }
    friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
    friend bool operator<=(double lhs, const Approx& r) { return lhs < r.v_ || lhs == r; }
    friend bool operator>=(double lhs, const Approx& r) { return lhs > r.v_ || lhs == r; }

private:
    double v_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
    double scale_ = 1.0;
};

struct Contains {
    explicit Contains(const char* s) : str(s) {}
    std::string str;
};

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
struct Reg {
    Reg(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};
struct State {
    int failures = 0;
    int assertions = 0;
    bool case_failed = false;
    // subcase tracking: one new leaf subcase per run of the test function
    std::set<std::string> done;
    std::vector<std::string> stack;
    bool entered = false;
    long skips = 0;  // subcases skipped (not yet done) in the current pass
};
inline State& st() {
    static State s;
    return s;
}
struct RequireFailed {};
inline void fail(const char* file, int line, const std::string& what) {
    auto& s = st();
    s.failures++;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, what.c_str());
}
struct Subcase {
    bool active = false;
    long skips_at_entry = 0;
    std::string path;
    explicit Subcase(const char* name) {
        auto& s = st();
        path.clear();
        for (auto& p : s.stack) path += p + "/";
        path += name;
        if (s.done.count(path)) return;
        if (s.entered) {  // another leaf already ran in this pass
            ++s.skips;
            return;
        }
        active = true;
        skips_at_entry = s.skips;
        s.stack.push_back(name);
    }
    ~Subcase() {
        if (!active) return;
        auto& s = st();
        s.stack.pop_back();
        // done once no nested subcase inside it is still pending
        if (s.skips == skips_at_entry) s.done.insert(path);
        s.entered = true;
    }
    explicit operator bool() const { return active; }
};
inline bool contains(const std::string& hay, const Contains& c) {
    return hay.find(c.str) != std::string::npos;
}
inline bool contains(const std::string& hay, const char* c) { return hay == c; }

inline int run_all() {
    auto& s = st();
    int failed_cases = 0;
    for (auto& tc : registry()) {
        s.done.clear();
        s.case_failed = false;
        for (int guard = 0; guard < 1000; ++guard) {
            s.entered = false;
            s.skips = 0;
            s.stack.clear();
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                fail(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
            } catch (...) {
                fail(tc.file, tc.line, "unexpected exception");
            }
            if (!s.entered) break;
        }
        if (s.case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "[FAIL] %s\n", tc.name);
        } else {
            std::fprintf(stdout, "[ok]   %s\n", tc.name);
        }
    }
    std::fprintf(stdout, "test cases: %zu | failed: %d | assertions: %d | failed checks: %d\n",
                 registry().size(), failed_cases, s.assertions, s.failures);
    return failed_cases == 0 ? 0 : 1;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                            \
    static void fn();                                                                    \
    static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_CAT(sc_, __LINE__){name})

#define CHECK(...)                                                                   \
    do {                                                                             \
        ::doctest::detail::st().assertions++;                                        \
        if (!(__VA_ARGS__)) ::doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__); \
    } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                     \
    do {                                                                                 \
        ::doctest::detail::st().assertions++;                                            \
        if (!(__VA_ARGS__)) {                                                            \
            ::doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);                   \
            throw ::doctest::detail::RequireFailed{};                                    \
        }                                                                                \
    } while (0)
#define REQUIRE_MESSAGE(cond, msg) REQUIRE(cond)
#define CHECK_MESSAGE(cond, msg) CHECK(cond)
#define FAIL(msg)                                                \
    do {                                                         \
        ::doctest::detail::fail(__FILE__, __LINE__, "FAIL");     \
        throw ::doctest::detail::RequireFailed{};                \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                           \
    do {                                                                                     \
        ::doctest::detail::st().assertions++;                                                \
        bool ok_ = false;                                                                    \
        try {                                                                                \
            (void)(expr);                                                                    \
        } catch (const __VA_ARGS__&) {                                                       \
            ok_ = true;                                                                      \
        } catch (...) {                                                                      \
        }                                                                                    \
        if (!ok_) ::doctest::detail::fail(__FILE__, __LINE__, "THROWS_AS " #expr);           \
    } while (0)
#define CHECK_THROWS(expr)                                                               \
    do {                                                                                 \
        bool ok_ = false;                                                                \
        try {                                                                            \
            (void)(expr);                                                                \
        } catch (...) {                                                                  \
            ok_ = true;                                                                  \
        }                                                                                \
        if (!ok_) ::doctest::detail::fail(__FILE__, __LINE__, "THROWS " #expr);         \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, match, ...)                                               \
    do {                                                                                     \
        ::doctest::detail::st().assertions++;                                                \
        bool ok_ = false;                                                                    \
        try {                                                                                \
            (void)(expr);                                                                    \
        } catch (const __VA_ARGS__& e_) {                                                    \
            ok_ = ::doctest::detail::contains(e_.what(), match);                             \
        } catch (...) {                                                                      \
        }                                                                                    \
        if (!ok_) ::doctest::detail::fail(__FILE__, __LINE__, "THROWS_WITH_AS " #expr);      \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                  \
    do {                                                                                     \
        ::doctest::detail::st().assertions++;                                                \
        try {                                                                                \
            (void)(expr);                                                                    \
        } catch (...) {                                                                      \
            ::doctest::detail::fail(__FILE__, __LINE__, "NOTHROW " #expr);                   \
        }                                                                                    \
    } while (0)
#define REQUIRE_NOTHROW(expr) CHECK_NOTHROW(expr)
#define CAPTURE(x) (void)0
#define INFO(...) (void)0
#define MESSAGE(...) (void)0

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
