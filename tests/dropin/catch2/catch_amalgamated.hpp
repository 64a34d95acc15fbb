// A minimal, header-only stand-in for the slice of Catch2 v3 that the
// reference's unit tests use (TEST_CASE, CHECK/REQUIRE and their _FALSE /
// _THROWS_AS / _NOTHROW forms, FAIL, INFO, SECTION), so that
// /root/reference/proj/tests/test_chain_dp.cpp and test_simulate.cpp compile
// UNCHANGED against this repo's drop-in headers (Catch2 itself is not in this
// image).  Written for this repo; it is not Catch2's code.  Semantics kept:
//   * CHECK records a failure and continues, REQUIRE aborts the test case;
//   * FAIL aborts with a failure that a test's own catch clauses for library
//     exceptions do not intercept (it is not a std::exception);
//   * INFO messages are printed with every failure inside their scope.
// Exit status: 0 when every assertion passed.  Argument: an optional
// substring filter on test names.
#pragma once

#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace minicatch {

struct Abort {};  // REQUIRE / FAIL: leaves the test case (not a std::exception)

struct TestCase {
    const char* name;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
inline std::vector<std::string>& infos() {
    static thread_local std::vector<std::string> v;
    return v;
}
struct Stats {
    long assertions = 0, failed = 0;
    bool case_failed = false;
    const char* current = "";
};
inline Stats& stats() {
    static Stats s;
    return s;
}

struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct ScopedInfo {
    explicit ScopedInfo(std::string m) { infos().push_back(std::move(m)); }
    ~ScopedInfo() { infos().pop_back(); }
};

inline void report(const char* file, int line, const char* what, const std::string& detail = {}) {
    Stats& s = stats();
    ++s.failed;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s%s%s\n", file, line, s.current, what,
                 detail.empty() ? "" : " -- ", detail.c_str());
    for (const std::string& i : infos()) std::fprintf(stderr, "    with: %s\n", i.c_str());
}

inline void assert_that(bool ok, bool fatal, const char* file, int line, const char* expr) {
    ++stats().assertions;
    if (ok) return;
    report(file, line, expr);
    if (fatal) throw Abort{};
}

template <typename Ex>
inline void assert_throws(const std::function<void()>& f, bool fatal, const char* file, int line,
                          const char* expr, const char* type) {
    ++stats().assertions;
    try {
        f();
    } catch (const Ex&) {
        return;
    } catch (const Abort&) {
        throw;
    } catch (const std::exception& e) {
        report(file, line, expr, std::string("threw a different exception (want ") + type + "): " + e.what());
        if (fatal) throw Abort{};
        return;
    } catch (...) {
        report(file, line, expr, std::string("threw a non-std exception (want ") + type + ")");
        if (fatal) throw Abort{};
        return;
    }
    report(file, line, expr, std::string("did not throw ") + type);
    if (fatal) throw Abort{};
}

inline void assert_nothrow(const std::function<void()>& f, bool fatal, const char* file, int line,
                           const char* expr) {
    ++stats().assertions;
    try {
        f();
    } catch (const Abort&) {
        throw;
    } catch (const std::exception& e) {
        report(file, line, expr, std::string("threw: ") + e.what());
        if (fatal) throw Abort{};
    }
}

inline int run_all(int argc, char** argv) {
    const char* filter = argc > 1 ? argv[1] : nullptr;
    Stats& s = stats();
    int cases = 0, failed_cases = 0;
    for (const TestCase& tc : registry()) {
        if (filter && !std::strstr(tc.name, filter)) continue;
        ++cases;
        s.current = tc.name;
        s.case_failed = false;
        try {
            tc.fn();
        } catch (const Abort&) {
        } catch (const std::exception& e) {
            report(__FILE__, __LINE__, "unexpected exception", e.what());
        } catch (...) {
            report(__FILE__, __LINE__, "unexpected non-std exception");
        }
        if (s.case_failed) ++failed_cases;
    }
    std::printf("%d test cases (%d failed), %ld assertions (%ld failed)\n", cases, failed_cases,
                s.assertions, s.failed);
    return s.failed == 0 && cases > 0 ? 0 : 1;
}

}  // namespace minicatch

#define MINICATCH_CAT2(a, b) a##b
#define MINICATCH_CAT(a, b) MINICATCH_CAT2(a, b)
#define MINICATCH_TEST(fn, name)                                                    \
    static void fn();                                                               \
    static const ::minicatch::Registrar MINICATCH_CAT(fn, _reg)(name, &fn);         \
    static void fn()
#define TEST_CASE(name, ...) MINICATCH_TEST(MINICATCH_CAT(minicatch_case_, __LINE__), name)
#define SECTION(...) if (true)

#define CHECK(...) ::minicatch::assert_that(static_cast<bool>(__VA_ARGS__), false, __FILE__, __LINE__, #__VA_ARGS__)
#define REQUIRE(...) ::minicatch::assert_that(static_cast<bool>(__VA_ARGS__), true, __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_FALSE(...) ::minicatch::assert_that(!static_cast<bool>(__VA_ARGS__), false, __FILE__, __LINE__, "!(" #__VA_ARGS__ ")")
#define REQUIRE_FALSE(...) ::minicatch::assert_that(!static_cast<bool>(__VA_ARGS__), true, __FILE__, __LINE__, "!(" #__VA_ARGS__ ")")
#define CHECK_THROWS_AS(expr, type) \
    ::minicatch::assert_throws<type>([&] { (void)(expr); }, false, __FILE__, __LINE__, #expr, #type)
#define REQUIRE_THROWS_AS(expr, type) \
    ::minicatch::assert_throws<type>([&] { (void)(expr); }, true, __FILE__, __LINE__, #expr, #type)
#define CHECK_NOTHROW(expr) ::minicatch::assert_nothrow([&] { (void)(expr); }, false, __FILE__, __LINE__, #expr)
#define REQUIRE_NOTHROW(expr) ::minicatch::assert_nothrow([&] { (void)(expr); }, true, __FILE__, __LINE__, #expr)
#define FAIL(msg)                                                                        \
    do {                                                                                 \
        std::ostringstream minicatch_os_;                                                \
        minicatch_os_ << msg;                                                            \
        ::minicatch::report(__FILE__, __LINE__, "FAIL", minicatch_os_.str());            \
        throw ::minicatch::Abort{};                                                      \
    } while (0)
#define INFO(msg)                                                                        \
    ::minicatch::ScopedInfo MINICATCH_CAT(minicatch_info_, __LINE__)([&] {               \
        std::ostringstream minicatch_os_;                                                \
        minicatch_os_ << msg;                                                            \
        return minicatch_os_.str();                                                      \
    }())
#define CAPTURE(x) INFO(#x " := " << (x))

#ifdef MINICATCH_MAIN
int main(int argc, char** argv) { return ::minicatch::run_all(argc, argv); }
#endif
