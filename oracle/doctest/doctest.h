// TEST INFRASTRUCTURE ONLY — a small doctest-compatible test harness, written
// for this repository, so the reference's own unit suites
// (/root/reference/proj/tests/test_*.cpp, which include "doctest.h"; the real
// header lived in the reference's gitignored vendor/ directory and is absent)
// compile unchanged against both the reference library and the B200 drop-in
// (oracle/Makefile `unit`).  It implements exactly what those suites use:
// TEST_CASE, SUBCASE (doctest's re-entry semantics: the test case body is
// re-run until every leaf subcase has run once, each run entering at most one
// new subcase per nesting level), CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, FAIL and doctest::Approx (doctest's default epsilon,
// float epsilon * 100, scale 1), plus DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
#ifndef RFK_DOCTEST_SHIM_H
#define RFK_DOCTEST_SHIM_H

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <set>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double value)
        : m_epsilon(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100), m_scale(1.0), m_value(value) {}
    Approx& epsilon(double e) {
        m_epsilon = e;
        return *this;
    }
    Approx& scale(double s) {
        m_scale = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.m_value) <
               rhs.m_epsilon * (rhs.m_scale + std::max<double>(std::fabs(lhs), std::fabs(rhs.m_value)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return operator==(rhs, lhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !operator==(lhs, rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !operator==(rhs, lhs); }
    friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.m_value || lhs == rhs; }
    friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.m_value || lhs == rhs; }
    friend bool operator<(double lhs, const Approx& rhs) { return lhs < rhs.m_value && lhs != rhs; }
    friend bool operator>(double lhs, const Approx& rhs) { return lhs > rhs.m_value && lhs != rhs; }

private:
    double m_epsilon, m_scale, m_value;
};

namespace detail {

struct TestCase {
    void (*fn)();
    const char* name;
    const char* file;
    int line;
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Reg {
    Reg(void (*fn)(), const char* name, const char* file, int line) { registry().push_back({fn, name, file, line}); }
};

struct RequireFailed {};  // aborts the current test-case run

struct State {
    long long checks = 0, failures = 0;
    const char* test = "";
    // subcase bookkeeping of the running test case
    std::set<std::vector<std::string>> done;  // paths fully run
    std::vector<std::string> stack;           // the subcase path entered so far in this run
    std::vector<char> entered;                // per depth: a subcase was entered at this depth in this run
    std::vector<char> child_pending;          // per entered frame: a child subcase was left for a later run
    bool pending = false;                     // this run left a subcase unrun
};
inline State& st() {
    static State s;
    return s;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    State& s = st();
    ++s.checks;
    if (ok) return;
    ++s.failures;
    std::string path;
    for (const auto& p : s.stack) path += " / " + p;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s ) in TEST_CASE \"%s\"%s\n", file, line, kind, expr, s.test,
                 path.c_str());
}

class Subcase {
public:
    Subcase(const char* name) {
        State& s = st();
        const size_t d = s.stack.size();
        std::vector<std::string> path = s.stack;
        path.emplace_back(name);
        if (s.entered.size() <= d) s.entered.resize(d + 1, 0);
        if (s.done.count(path)) return;  // already run: skip
        if (s.entered[d]) {             // a sibling ran in this run: next run
            s.pending = true;
            if (!s.child_pending.empty()) s.child_pending.back() = 1;
            return;
        }
        s.entered[d] = 1;
        s.stack.push_back(name);
        if (s.entered.size() <= d + 1) s.entered.resize(d + 2, 0);
        s.entered[d + 1] = 0;
        s.child_pending.push_back(0);
        m_entered = true;
    }
    ~Subcase() {
        if (!m_entered) return;
        State& s = st();
        const bool pending = s.child_pending.back() != 0;
        // done once no nested subcase is left (a failing REQUIRE also ends it)
        if (!pending || std::uncaught_exceptions() > 0) s.done.insert(s.stack);
        s.child_pending.pop_back();
        s.stack.pop_back();
        if (pending && !s.child_pending.empty()) s.child_pending.back() = 1;
    }
    explicit operator bool() const { return m_entered; }

private:
    bool m_entered = false;
};

inline int run_all() {
    State& s = st();
    int failed_cases = 0;
    for (const TestCase& tc : registry()) {
        s.test = tc.name;
        s.done.clear();
        const long long f0 = s.failures;
        int runs = 0;
        do {
            s.stack.clear();
            s.entered.assign(1, 0);
            s.child_pending.clear();
            s.pending = false;
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                ++s.failures;
                std::fprintf(stderr, "%s:%d: TEST_CASE \"%s\" threw: %s\n", tc.file, tc.line, tc.name, e.what());
                s.pending = false;
            } catch (...) {
                ++s.failures;
                std::fprintf(stderr, "%s:%d: TEST_CASE \"%s\" threw an unknown exception\n", tc.file, tc.line,
                             tc.name);
                s.pending = false;
            }
        } while (s.pending && ++runs < 100000);
        if (s.failures != f0) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
                registry().size() - static_cast<size_t>(failed_cases), failed_cases);
    std::printf("[doctest-shim] assertions: %lld | %lld passed | %lld failed\n", s.checks, s.checks - s.failures,
                s.failures);
    std::printf("[doctest-shim] Status: %s\n", failed_cases ? "FAILURE!" : "SUCCESS!");
    return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                                   \
    static void fn();                                                                                      \
    static const ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(fn, name, __FILE__, __LINE__);               \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_shim_tc_, __COUNTER__), name)
#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_CAT(doctest_shim_sc_, __LINE__){name})

#define DOCTEST_EVAL_(...)                      \
    [&]() -> bool {                             \
        try {                                   \
            return static_cast<bool>(__VA_ARGS__); \
        } catch (...) {                         \
            return false;                       \
        }                                       \
    }()
#define CHECK(...) ::doctest::detail::report(DOCTEST_EVAL_(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    ::doctest::detail::report(!DOCTEST_EVAL_(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                  \
    do {                                                                                              \
        const bool doctest_shim_ok = DOCTEST_EVAL_(__VA_ARGS__);                                       \
        ::doctest::detail::report(doctest_shim_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);        \
        if (!doctest_shim_ok) throw ::doctest::detail::RequireFailed{};                                 \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                      \
    do {                                                                                                \
        bool doctest_shim_ok = false;                                                                   \
        try {                                                                                           \
            static_cast<void>(expr);                                                                    \
        } catch (const __VA_ARGS__&) {                                                                  \
            doctest_shim_ok = true;                                                                     \
        } catch (...) {                                                                                 \
        }                                                                                               \
        ::doctest::detail::report(doctest_shim_ok, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, \
                                  __LINE__);                                                            \
    } while (0)
#define FAIL(msg)                                                                   \
    do {                                                                            \
        ::doctest::detail::report(false, "FAIL", msg, __FILE__, __LINE__);          \
        throw ::doctest::detail::RequireFailed{};                                   \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif

#endif
