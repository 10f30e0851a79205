// Minimal doctest-compatible shim — TEST INFRASTRUCTURE (never part of the
// product).  doctest is absent from this image; the reference's unit tests
// (proj/tests/test_*.cpp) use only this subset of it:
// TEST_CASE, SUBCASE (one level), CHECK, CHECK_FALSE, REQUIRE, FAIL,
// MESSAGE and doctest::Approx(...).epsilon(...), with
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN providing main().  Command line:
// -tce=<glob> / --test-case-exclude=<glob> skips matching test cases.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

namespace shim {

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

struct State {
    int target = 0;      // the subcase this run enters
    int seen = 0;        // subcases met so far in this run
    long checks = 0, failed_checks = 0;
    bool case_failed = false;
};

inline State& state() {
    static State s;
    return s;
}

struct Abort {};  // REQUIRE / FAIL end the current run of a test case

struct Reg {
    Reg(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};

struct Subcase {
    bool entered;
    explicit Subcase(const char*) : entered(state().seen++ == state().target) {}
    explicit operator bool() const { return entered; }
};

inline void fail(const char* file, int line, const std::string& what) {
    State& s = state();
    ++s.failed_checks;
    s.case_failed = true;
    std::printf("%s:%d: ERROR: %s\n", file, line, what.c_str());
}

inline void check(bool ok, bool require, const char* macro, const char* expr, const char* file, int line) {
    ++state().checks;
    if (ok) return;
    fail(file, line, std::string(macro) + "( " + expr + " ) is NOT correct!");
    if (require) throw Abort{};
}

inline bool glob(const char* p, const char* s) {
    if (!*p) return !*s;
    if (*p == '*') return glob(p + 1, s) || (*s && glob(p, s + 1));
    return *s && *p == *s && glob(p + 1, s + 1);
}

inline int run(int argc, char** argv) {
    std::vector<std::string> exclude;
    for (int i = 1; i < argc; ++i) {
        const char* a = argv[i];
        for (const char* k : {"-tce=", "--test-case-exclude="})
            if (std::strncmp(a, k, std::strlen(k)) == 0) exclude.push_back(a + std::strlen(k));
    }
    int cases = 0, failed = 0, skipped = 0;
    for (const TestCase& tc : registry()) {
        bool skip = false;
        for (const auto& e : exclude) skip = skip || glob(e.c_str(), tc.name);
        if (skip) {
            ++skipped;
            continue;
        }
        ++cases;
        State& s = state();
        s.case_failed = false;
        // One run per subcase (one level, as in the reference's tests): run
        // k enters the k-th SUBCASE met and skips the others.
        for (s.target = 0;; ++s.target) {
            s.seen = 0;
            try {
                tc.fn();
            } catch (const Abort&) {
            } catch (const std::exception& e) {
                fail(tc.file, tc.line, std::string("test case threw: ") + e.what());
            } catch (...) {
                fail(tc.file, tc.line, "test case threw an unknown exception");
            }
            if (s.target + 1 >= s.seen) break;
        }
        if (s.case_failed) {
            ++failed;
            std::printf("  in TEST_CASE: %s\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | %d skipped\n", cases, cases - failed, failed,
                skipped);
    std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", state().checks,
                state().checks - state().failed_checks, state().failed_checks);
    std::printf("[doctest-shim] Status: %s\n", failed ? "FAILURE!" : "SUCCESS!");
    return failed ? 1 : 0;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_TC(fn, name)                                                                   \
    static void fn();                                                                               \
    static const doctest::shim::Reg DOCTEST_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);      \
    static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TC(DOCTEST_SHIM_CAT(doctest_shim_tc_, __COUNTER__), name)
#define SUBCASE(name) if (const doctest::shim::Subcase DOCTEST_SHIM_CAT(doctest_shim_sc_, __LINE__){name})
#define CHECK(...) doctest::shim::check(static_cast<bool>(__VA_ARGS__), false, "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    doctest::shim::check(!static_cast<bool>(__VA_ARGS__), false, "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...) \
    doctest::shim::check(static_cast<bool>(__VA_ARGS__), true, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__)
#define FAIL(...)                                                                        \
    do {                                                                                 \
        std::ostringstream doctest_shim_os;                                              \
        doctest_shim_os << __VA_ARGS__;                                                  \
        doctest::shim::fail(__FILE__, __LINE__, "FAIL: " + doctest_shim_os.str());       \
        throw doctest::shim::Abort{};                                                    \
    } while (0)
#define MESSAGE(...)                                                                     \
    do {                                                                                 \
        std::ostringstream doctest_shim_os;                                              \
        doctest_shim_os << __VA_ARGS__;                                                  \
        std::printf("%s:%d: MESSAGE: %s\n", __FILE__, __LINE__, doctest_shim_os.str().c_str()); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::shim::run(argc, argv); }
#endif
