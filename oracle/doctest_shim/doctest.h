// doctest.h -- minimal doctest-compatible harness (TEST INFRASTRUCTURE) so the reference's own
// unit tests (/root/reference/proj/tests, doctest.h is not vendored there) compile unchanged
// against the reference library or against the B200 drop-in shim. Supports the macros those
// tests use: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW,
// doctest::Approx(..).epsilon(..). Prints one line per test case and a summary; exit status
// 0 iff every check passed. Arguments select the cases whose name contains any of them.
#pragma once
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  double v, eps = 1.1920929e-7 * 100, sc = 1.0;
  explicit Approx(double x) : v(x) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  Approx& scale(double s) {
    sc = s;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v) < b.eps * (b.sc + std::fmax(std::fabs(a), std::fabs(b.v)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
};

namespace detail {
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
struct Reg {
  Reg(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct Abort {};
inline long& checks() { static long c = 0; return c; }
inline long& failures() { static long c = 0; return c; }
inline long& case_failures() { static long c = 0; return c; }
inline void fail(const char* file, int line, const char* what) {
  ++failures();
  ++case_failures();
  if (case_failures() <= 5) std::printf("    %s:%d: FAILED: %s\n", file, line, what);
}
}  // namespace detail

inline int run(int argc, char** argv) {
  int n_cases = 0, n_failed = 0;
  for (auto& c : detail::registry()) {
    bool selected = argc <= 1;  // no filter: every case; else cases matching any argument
    for (int a = 1; a < argc && !selected; ++a) selected = std::strstr(c.name, argv[a]) != nullptr;
    if (!selected) continue;
    ++n_cases;
    detail::case_failures() = 0;
    const long f0 = detail::failures();
    try {
      c.fn();
    } catch (const detail::Abort&) {
    } catch (const std::exception& e) {
      detail::fail(c.file, c.line, (std::string("unexpected exception: ") + e.what()).c_str());
    } catch (...) {
      detail::fail(c.file, c.line, "unexpected exception");
    }
    const bool ok = detail::failures() == f0;
    n_failed += ok ? 0 : 1;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    std::fflush(stdout);
  }
  std::printf("test cases: %d | %d passed | %d failed; checks: %ld | %ld failed\n", n_cases,
              n_cases - n_failed, n_failed, detail::checks(), detail::failures());
  return n_failed ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                    \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                        \
  static ::doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(                       \
      name, __FILE__, __LINE__, &DOCTEST_CAT(doctest_fn_, __LINE__));                      \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define CHECK(...)                                                                         \
  do {                                                                                     \
    ++::doctest::detail::checks();                                                         \
    if (!(__VA_ARGS__)) ::doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);          \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                       \
  do {                                                                                     \
    ++::doctest::detail::checks();                                                         \
    if (!(__VA_ARGS__)) {                                                                  \
      ::doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);                            \
      throw ::doctest::detail::Abort{};                                                    \
    }                                                                                      \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                        \
  do {                                                                                     \
    ++::doctest::detail::checks();                                                         \
    bool caught_ = false;                                                                  \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const type&) {                                                                \
      caught_ = true;                                                                      \
    } catch (...) {                                                                        \
    }                                                                                      \
    if (!caught_) ::doctest::detail::fail(__FILE__, __LINE__, "throws " #type ": " #expr); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                \
  do {                                                                                     \
    ++::doctest::detail::checks();                                                         \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (...) {                                                                        \
      ::doctest::detail::fail(__FILE__, __LINE__, "nothrow: " #expr);                       \
    }                                                                                      \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::run(argc, argv); }
#endif
