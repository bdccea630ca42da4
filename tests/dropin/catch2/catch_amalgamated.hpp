// Minimal stand-in for Catch2 v3's catch_amalgamated.hpp (absent from this
// image; the reference's tests/CMakeLists.txt:1-2 expects it under
// /usr/local/include/catch2). TEST INFRASTRUCTURE ONLY: it implements the
// subset of macros the reference's unit suites use — TEST_CASE, CHECK,
// CHECK_FALSE, CHECK_NOTHROW, CHECK_THROWS, CHECK_THROWS_AS, REQUIRE,
// REQUIRE_FALSE, INFO, FAIL, Catch::Approx — so those suites compile
// unchanged against the B200 library (tests/dropin/, tests/test_dropin.py).
//
// The binary runs every test case (or those named on the command line with
// --only "<name>"), prints one line per case ("PASS <name>" / "FAIL <name>"
// plus the failed expressions) and exits with the number of failed cases.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace Catch {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& margin(double m) {
        margin_ = m;
        return *this;
    }
    bool matches(double x) const {
        const double d = std::fabs(x - value_);  // Catch2: margin, or epsilon relative to the expected value
        return d <= margin_ || d <= eps_ * (std::isinf(value_) ? 0.0 : std::fabs(value_));
    }
    friend bool operator==(double x, const Approx& a) { return a.matches(x); }
    friend bool operator==(const Approx& a, double x) { return a.matches(x); }
    friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
    friend std::ostream& operator<<(std::ostream& os, const Approx& a) { return os << "Approx(" << a.value_ << ")"; }

private:
    double value_;
    double eps_ = 1.1920929e-07 * 100;  // Catch2's default: 100 float epsilons
    double margin_ = 0.0;
};

namespace shim {

struct Case {
    const char* name;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Register {
    Register(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct RequireFailed {};

inline int& failures() {
    static int f = 0;
    return f;
}

inline std::vector<std::string>& info() {
    static std::vector<std::string> v;
    return v;
}

inline void report(const char* kind, const char* expr, const char* file, int line) {
    ++failures();
    std::cout << "    " << kind << " failed: " << expr << "  (" << file << ":" << line << ")\n";
    for (const auto& s : info()) std::cout << "      with: " << s << "\n";
}

struct InfoScope {
    explicit InfoScope(std::string s) { info().push_back(std::move(s)); }
    ~InfoScope() { info().pop_back(); }
};

}  // namespace shim
}  // namespace Catch

#define TFB_CATCH_CAT2(a, b) a##b
#define TFB_CATCH_CAT(a, b) TFB_CATCH_CAT2(a, b)

#define TEST_CASE(name, ...)                                                                              \
    static void TFB_CATCH_CAT(tfb_catch_case_, __LINE__)();                                               \
    static ::Catch::shim::Register TFB_CATCH_CAT(tfb_catch_reg_, __LINE__)(name,                          \
                                                                           &TFB_CATCH_CAT(tfb_catch_case_, \
                                                                                          __LINE__));     \
    static void TFB_CATCH_CAT(tfb_catch_case_, __LINE__)()

#define TFB_CATCH_ASSERT(kind, expr, fatal)                                                 \
    do {                                                                                    \
        bool tfb_ok_ = false;                                                               \
        try {                                                                               \
            tfb_ok_ = static_cast<bool>(expr);                                              \
        } catch (const std::exception& tfb_e_) {                                            \
            ::Catch::shim::report(kind " threw", tfb_e_.what(), __FILE__, __LINE__);        \
            if (fatal) throw ::Catch::shim::RequireFailed{};                                \
            break;                                                                          \
        }                                                                                   \
        if (!tfb_ok_) {                                                                     \
            ::Catch::shim::report(kind, #expr, __FILE__, __LINE__);                         \
            if (fatal) throw ::Catch::shim::RequireFailed{};                                \
        }                                                                                   \
    } while (0)

#define CHECK(...) TFB_CATCH_ASSERT("CHECK", (__VA_ARGS__), false)
#define CHECK_FALSE(...) TFB_CATCH_ASSERT("CHECK_FALSE", !(__VA_ARGS__), false)
#define REQUIRE(...) TFB_CATCH_ASSERT("REQUIRE", (__VA_ARGS__), true)
#define REQUIRE_FALSE(...) TFB_CATCH_ASSERT("REQUIRE_FALSE", !(__VA_ARGS__), true)

#define CHECK_THROWS_AS(expr, type)                                                                 \
    do {                                                                                            \
        bool tfb_right_ = false;                                                                    \
        const char* tfb_what_ = "no exception";                                                     \
        try {                                                                                       \
            static_cast<void>(expr);                                                                \
        } catch (const type&) {                                                                     \
            tfb_right_ = true;                                                                      \
        } catch (const std::exception& tfb_e_) {                                                    \
            tfb_what_ = tfb_e_.what();                                                              \
        } catch (...) {                                                                             \
            tfb_what_ = "unknown exception";                                                        \
        }                                                                                           \
        if (!tfb_right_)                                                                            \
            ::Catch::shim::report("CHECK_THROWS_AS(" #type ")", (std::string(#expr) + " -> " + tfb_what_).c_str(), \
                                  __FILE__, __LINE__);                                              \
    } while (0)

#define CHECK_THROWS(expr)                                                                \
    do {                                                                                  \
        bool tfb_threw_ = false;                                                          \
        try {                                                                             \
            static_cast<void>(expr);                                                      \
        } catch (...) {                                                                   \
            tfb_threw_ = true;                                                            \
        }                                                                                 \
        if (!tfb_threw_) ::Catch::shim::report("CHECK_THROWS", #expr, __FILE__, __LINE__); \
    } while (0)

#define CHECK_NOTHROW(expr)                                                                       \
    do {                                                                                          \
        try {                                                                                     \
            static_cast<void>(expr);                                                              \
        } catch (const std::exception& tfb_e_) {                                                  \
            ::Catch::shim::report("CHECK_NOTHROW", (std::string(#expr) + " -> " + tfb_e_.what()).c_str(), \
                                  __FILE__, __LINE__);                                            \
        }                                                                                         \
    } while (0)

#define INFO(msg)                                                                   \
    ::Catch::shim::InfoScope TFB_CATCH_CAT(tfb_info_, __LINE__)([&] {               \
        std::ostringstream tfb_os_;                                                 \
        tfb_os_ << msg;                                                             \
        return tfb_os_.str();                                                       \
    }())

#define FAIL(msg)                                                                       \
    do {                                                                                \
        std::ostringstream tfb_os_;                                                     \
        tfb_os_ << msg;                                                                 \
        ::Catch::shim::report("FAIL", tfb_os_.str().c_str(), __FILE__, __LINE__);       \
        throw ::Catch::shim::RequireFailed{};                                           \
    } while (0)

int main(int argc, char** argv) {
    std::vector<std::string> only;
    for (int i = 1; i + 1 < argc; ++i)
        if (std::strcmp(argv[i], "--only") == 0) only.push_back(argv[++i]);
    int failed_cases = 0, run = 0;
    for (const auto& c : ::Catch::shim::registry()) {
        if (!only.empty()) {
            bool want = false;
            for (const auto& o : only) want = want || o == c.name;
            if (!want) continue;
        }
        ++run;
        const int before = ::Catch::shim::failures();
        try {
            c.fn();
        } catch (const ::Catch::shim::RequireFailed&) {
        } catch (const std::exception& e) {
            ::Catch::shim::report("uncaught exception", e.what(), c.name, 0);
        } catch (...) {
            ::Catch::shim::report("uncaught exception", "unknown", c.name, 0);
        }
        const bool ok = ::Catch::shim::failures() == before;
        failed_cases += !ok;
        std::cout << (ok ? "PASS " : "FAIL ") << c.name << std::endl;
    }
    std::cout << "cases: " << run << ", failed: " << failed_cases << std::endl;
    return failed_cases;
}
