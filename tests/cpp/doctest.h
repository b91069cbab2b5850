// Minimal doctest-compatible test shim (test infrastructure only).
//
// The reference's unit tests (/root/reference/proj/tests/test_*.cpp) are
// written against doctest, which is not vendored there. This header
// provides the subset they use — TEST_CASE, SUBCASE (doctest's
// re-run-per-subcase semantics, one nesting level), CHECK / REQUIRE
// (variadic, so brace-initialiser commas work), CHECK_THROWS_AS,
// CHECK_NOTHROW, INFO (ignored) and doctest::Approx — so those tests can be
// compiled unchanged against the B200 façade (tests/cpp/build_conformance.py)
// and run on the GPU (tests/test_facade_gpu.py). Define
// PE_DOCTEST_SHIM_MAIN in exactly one translation unit to get main().
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double value) : value_(value) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) < a.eps_ * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

private:
    double value_;
    double eps_ = 1.1920928955078125e-05;  // doctest default: FLT_EPSILON * 100
};

}  // namespace doctest

namespace pe_shim {

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

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back(Case{name, file, line, fn});
    }
};

struct RunState {
    int target = 0;       // subcase index entered during this run
    int seen = 0;         // subcases encountered during this run
    int failures = 0;
    std::string first_failure;
};

inline RunState& state() {
    static RunState s;
    return s;
}

struct RequireFailed {};

inline void fail(const char* file, int line, const std::string& what) {
    RunState& s = state();
    if (s.failures++ == 0) s.first_failure = std::string(file) + ":" + std::to_string(line) + ": " + what;
    std::fprintf(stderr, "  %s:%d: FAILED %s\n", file, line, what.c_str());
}

// true for exactly one subcase per run (by encounter order)
inline bool enter_subcase() { return state().seen++ == state().target; }

}  // namespace pe_shim

#define PE_SHIM_CAT2(a, b) a##b
#define PE_SHIM_CAT(a, b) PE_SHIM_CAT2(a, b)
#define PE_SHIM_TEST_CASE(fn, name)                                                            \
    static void fn();                                                                          \
    static pe_shim::Registrar PE_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);            \
    static void fn()
#define TEST_CASE(name) PE_SHIM_TEST_CASE(PE_SHIM_CAT(pe_shim_case_, __COUNTER__), name)
#define SUBCASE(name) if (pe_shim::enter_subcase())

#define CHECK(...)                                                                      \
    do {                                                                                \
        try {                                                                           \
            if (!(__VA_ARGS__)) pe_shim::fail(__FILE__, __LINE__, "CHECK(" #__VA_ARGS__ ")"); \
        } catch (const std::exception& e_) {                                            \
            pe_shim::fail(__FILE__, __LINE__, std::string("CHECK threw: ") + e_.what()); \
        }                                                                               \
    } while (0)
#define REQUIRE(...)                                                                       \
    do {                                                                                   \
        if (!(__VA_ARGS__)) {                                                              \
            pe_shim::fail(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")");                \
            throw pe_shim::RequireFailed{};                                                \
        }                                                                                  \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                          \
    do {                                                                                     \
        bool thrown_ = false;                                                                \
        try {                                                                                \
            (void)(expr);                                                                    \
        } catch (const type&) {                                                              \
            thrown_ = true;                                                                  \
        } catch (const std::exception& e_) {                                                 \
            pe_shim::fail(__FILE__, __LINE__, std::string("wrong exception: ") + e_.what()); \
            thrown_ = true;                                                                  \
        }                                                                                    \
        if (!thrown_) pe_shim::fail(__FILE__, __LINE__, "no exception: " #expr);            \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                 \
    do {                                                                                    \
        try {                                                                               \
            (void)(expr);                                                                   \
        } catch (const std::exception& e_) {                                                \
            pe_shim::fail(__FILE__, __LINE__, std::string("threw: ") + e_.what());         \
        }                                                                                   \
    } while (0)
#define INFO(...) ((void)0)

#ifdef PE_DOCTEST_SHIM_MAIN
// Runs every registered case (or those whose name contains argv[1]); one
// "[case] PASS|FAIL <name>" line per case, exit status = failed case count.
int main(int argc, char** argv) {
    int failed = 0, passed = 0;
    for (const pe_shim::Case& c : pe_shim::registry()) {
        if (argc > 1 && std::strstr(c.name, argv[1]) == nullptr) continue;
        bool ok = true;
        std::string why;
        for (int target = 0;; ++target) {  // one run per subcase
            pe_shim::RunState& s = pe_shim::state();
            s = pe_shim::RunState{};
            s.target = target;
            try {
                c.fn();
            } catch (const pe_shim::RequireFailed&) {
            } catch (const std::exception& e) {
                pe_shim::fail(c.file, c.line, std::string("unexpected exception: ") + e.what());
            }
            if (s.failures) {
                ok = false;
                if (why.empty()) why = s.first_failure;
            }
            if (target + 1 >= s.seen) break;
        }
        std::printf("[case] %s %s%s%s\n", ok ? "PASS" : "FAIL", c.name, ok ? "" : " :: ", why.c_str());
        std::fflush(stdout);
        (ok ? passed : failed)++;
    }
    std::printf("[summary] %d passed, %d failed\n", passed, failed);
    return failed;
}
#endif
