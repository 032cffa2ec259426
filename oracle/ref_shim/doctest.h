// TEST INFRASTRUCTURE ONLY (oracle/).  A minimal stand-in for doctest 2.x
// (absent from the container) covering what the reference's own
// test files use: TEST_CASE, SUBCASE (doctest's re-run-per-leaf model),
// CHECK / CHECK_FALSE / REQUIRE / CHECK_THROWS_AS / CHECK_THROWS_WITH_AS,
// WARN, FAIL, doctest::Approx(...).epsilon(), doctest::Contains.  With
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN the file gets a main() that runs every
// case and returns nonzero on any failure.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
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
    bool eq(double x) const { return std::fabs(x - v_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(v_))); }
    double value() const { return v_; }

private:
    double v_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};
inline bool operator==(double x, const Approx& a) { return a.eq(x); }
inline bool operator==(const Approx& a, double x) { return a.eq(x); }
inline bool operator!=(double x, const Approx& a) { return !a.eq(x); }
inline bool operator!=(const Approx& a, double x) { return !a.eq(x); }
inline bool operator<=(double x, const Approx& a) { return x < a.value() || a.eq(x); }
inline bool operator>=(double x, const Approx& a) { return x > a.value() || a.eq(x); }
inline bool operator<=(const Approx& a, double x) { return a.value() < x || a.eq(x); }
inline bool operator>=(const Approx& a, double x) { return a.value() > x || a.eq(x); }

struct Contains {
    explicit Contains(std::string s) : s(std::move(s)) {}
    std::string s;
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
    Reg(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};
struct State {
    int failures = 0;       // assertion failures in the current case
    long long asserts = 0;  // all assertions
    std::vector<std::string> stack;
    std::set<std::vector<std::string>> passed;
    size_t max_level = 0;
    int skips = 0;
    const char* current = "";
};
inline State& st() {
    static State s;
    return s;
}
struct RequireFailed {};
inline void report(const char* file, int line, const char* kind, const std::string& what) {
    std::fprintf(stderr, "%s:%d: %s FAILED (%s): %s\n", file, line, kind, st().current, what.c_str());
    ++st().failures;
}
class Subcase {
public:
    Subcase(const char* name, const char* file, int line) {
        std::string sig = std::string(name) + "@" + file + ":" + std::to_string(line);
        std::vector<std::string> cand = st().stack;
        cand.push_back(sig);
        if (st().passed.count(cand)) return;
        if (st().stack.size() < st().max_level) {  // a sibling ran this pass
            ++st().skips;
            return;
        }
        st().stack.push_back(sig);
        st().max_level = st().stack.size();
        skips_at_entry_ = st().skips;
        entered_ = true;
    }
    ~Subcase() {
        if (!entered_) return;
        if (st().skips == skips_at_entry_ || std::uncaught_exceptions() > 0) st().passed.insert(st().stack);
        st().stack.pop_back();
    }
    explicit operator bool() const { return entered_; }

private:
    bool entered_ = false;
    int skips_at_entry_ = 0;
};
inline std::string exc_message(const std::exception& e) { return e.what(); }
inline bool message_matches(const std::string& msg, const Contains& c) { return msg.find(c.s) != std::string::npos; }
inline bool message_matches(const std::string& msg, const char* s) { return msg == s; }
inline bool message_matches(const std::string& msg, const std::string& s) { return msg == s; }

inline int run_all() {
    int failed_cases = 0, total = 0;
    for (const TestCase& tc : registry()) {
        ++total;
        State& s = st();
        s.failures = 0;
        s.passed.clear();
        s.current = tc.name;
        for (int pass = 0; pass < 10000; ++pass) {
            s.stack.clear();
            s.max_level = 0;
            s.skips = 0;
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                report(tc.file, tc.line, "TEST_CASE", std::string("uncaught exception: ") + e.what());
            } catch (...) {
                report(tc.file, tc.line, "TEST_CASE", "uncaught non-standard exception");
            }
            if (s.skips == 0) break;
        }
        if (s.failures) ++failed_cases;
        std::printf("[%s] %s\n", s.failures ? "FAIL" : "ok", tc.name);
    }
    std::printf("test cases: %d | %d passed | %d failed | assertions: %lld\n", total, total - failed_cases,
                failed_cases, st().asserts);
    return failed_cases ? 1 : 0;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                                      \
    static void DOCTEST_ANON(doctest_fn_)();                                                                  \
    static ::doctest::detail::Reg DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__, &DOCTEST_ANON(doctest_fn_)); \
    static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_ANON(doctest_sc_){name, __FILE__, __LINE__})

#define DOCTEST_ASSERT_IMPL(kind, cond, fatal)                                                          \
    do {                                                                                                \
        ++::doctest::detail::st().asserts;                                                              \
        bool doctest_ok_ = false;                                                                       \
        try {                                                                                           \
            doctest_ok_ = static_cast<bool>(cond);                                                      \
        } catch (const std::exception& doctest_e_) {                                                    \
            ::doctest::detail::report(__FILE__, __LINE__, kind,                                         \
                                      std::string(#cond " threw: ") + doctest_e_.what());               \
            if (fatal) throw ::doctest::detail::RequireFailed{};                                        \
            break;                                                                                      \
        }                                                                                               \
        if (!doctest_ok_) {                                                                             \
            ::doctest::detail::report(__FILE__, __LINE__, kind, #cond);                                 \
            if (fatal) throw ::doctest::detail::RequireFailed{};                                        \
        }                                                                                               \
    } while (0)

#define CHECK(...) DOCTEST_ASSERT_IMPL("CHECK", (__VA_ARGS__), false)
#define CHECK_FALSE(...) DOCTEST_ASSERT_IMPL("CHECK_FALSE", !(__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_ASSERT_IMPL("REQUIRE", (__VA_ARGS__), true)
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_IMPL("REQUIRE_FALSE", !(__VA_ARGS__), true)
#define CHECK_EQ(a, b) CHECK((a) == (b))
#define CHECK_NE(a, b) CHECK((a) != (b))
#define CHECK_LT(a, b) CHECK((a) < (b))
#define CHECK_LE(a, b) CHECK((a) <= (b))
#define CHECK_GT(a, b) CHECK((a) > (b))
#define CHECK_GE(a, b) CHECK((a) >= (b))
#define CHECK_UNARY(a) CHECK(a)
#define REQUIRE_EQ(a, b) REQUIRE((a) == (b))

#define DOCTEST_THROWS_IMPL(kind, expr, type, fatal)                                                    \
    do {                                                                                                \
        ++::doctest::detail::st().asserts;                                                              \
        bool doctest_ok_ = false;                                                                       \
        try {                                                                                           \
            static_cast<void>(expr);                                                                    \
        } catch (const type&) {                                                                         \
            doctest_ok_ = true;                                                                         \
        } catch (...) {                                                                                 \
        }                                                                                               \
        if (!doctest_ok_) {                                                                             \
            ::doctest::detail::report(__FILE__, __LINE__, kind, #expr " did not throw " #type);         \
            if (fatal) throw ::doctest::detail::RequireFailed{};                                        \
        }                                                                                               \
    } while (0)
#define CHECK_THROWS_AS(expr, ...) DOCTEST_THROWS_IMPL("CHECK_THROWS_AS", expr, __VA_ARGS__, false)
#define REQUIRE_THROWS_AS(expr, ...) DOCTEST_THROWS_IMPL("REQUIRE_THROWS_AS", expr, __VA_ARGS__, true)
#define CHECK_THROWS(expr) DOCTEST_THROWS_IMPL("CHECK_THROWS", expr, std::exception, false)
#define CHECK_NOTHROW(expr)                                                                             \
    do {                                                                                                \
        ++::doctest::detail::st().asserts;                                                              \
        try {                                                                                           \
            static_cast<void>(expr);                                                                    \
        } catch (...) {                                                                                 \
            ::doctest::detail::report(__FILE__, __LINE__, "CHECK_NOTHROW", #expr " threw");             \
        }                                                                                               \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, ...)                                                            \
    do {                                                                                                \
        ++::doctest::detail::st().asserts;                                                              \
        bool doctest_ok_ = false;                                                                       \
        std::string doctest_got_ = "(no exception)";                                                    \
        try {                                                                                           \
            static_cast<void>(expr);                                                                    \
        } catch (const __VA_ARGS__& doctest_e_) {                                                       \
            doctest_got_ = ::doctest::detail::exc_message(doctest_e_);                                  \
            doctest_ok_ = ::doctest::detail::message_matches(doctest_got_, msg);                        \
        } catch (...) {                                                                                 \
            doctest_got_ = "(other exception type)";                                                    \
        }                                                                                               \
        if (!doctest_ok_)                                                                               \
            ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_WITH_AS",                       \
                                      std::string(#expr " -> ") + doctest_got_);                        \
    } while (0)

#define WARN(...)                                                                                       \
    do {                                                                                                \
        if (!(__VA_ARGS__)) std::fprintf(stderr, "%s:%d: WARN: %s\n", __FILE__, __LINE__, #__VA_ARGS__); \
    } while (0)
#define FAIL(msg)                                                                                       \
    do {                                                                                                \
        ::doctest::detail::report(__FILE__, __LINE__, "FAIL", std::string(msg));                        \
        throw ::doctest::detail::RequireFailed{};                                                       \
    } while (0)
#define FAIL_CHECK(msg) ::doctest::detail::report(__FILE__, __LINE__, "FAIL_CHECK", std::string(msg))
#define MESSAGE(msg) std::fprintf(stderr, "%s:%d: MESSAGE: %s\n", __FILE__, __LINE__, std::string(msg).c_str())
#define INFO(...) ((void)0)
#define CAPTURE(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
