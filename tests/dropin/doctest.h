// doctest.h — a minimal stand-in for the doctest single-header framework.
//
// TEST INFRASTRUCTURE ONLY. The reference's unit suites
// (proj/tests/test_{scoring,reorder,tiering}.cpp) are written against doctest,
// whose header is not shipped with the reference (proj/.gitignore:2) and is not
// installed here. This file implements exactly the subset those suites use —
// TEST_SUITE_BEGIN/END, TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// doctest::Approx(.epsilon), doctest::Contains — so they can be compiled
// unchanged against the B200 drop-in library (oracle/Makefile, target dropin).
//
// Semantics follow doctest's documented behaviour: CHECK records a failure
// and continues, REQUIRE aborts the test case, Approx compares with
// |a-b| < eps * (scale + max(|a|,|b|)), eps defaulting to 100 * FLT_EPSILON.
// The runner executes every registered case (or those whose name contains
// argv[1]) and exits with the number of failed cases.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
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
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) < b.eps_ * (b.scale_ + std::max(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  friend bool operator!=(const Approx& b, double a) { return !(a == b); }

 private:
  double v_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 0.0;
};

struct Contains {
  explicit Contains(std::string s) : needle(std::move(s)) {}
  bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
  std::string needle;
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

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct RequireFailed {};

inline int& failures_in_case() {
  static int n = 0;
  return n;
}
inline long& assertions() {
  static long n = 0;
  return n;
}

inline void fail(const char* file, int line, const char* what, const std::string& extra = "") {
  ++failures_in_case();
  std::printf("%s:%d: FAILED: %s%s%s\n", file, line, what, extra.empty() ? "" : " -- ",
              extra.c_str());
}

inline bool check(bool ok, const char* file, int line, const char* expr, bool require) {
  ++assertions();
  if (!ok) {
    fail(file, line, expr);
    if (require) throw RequireFailed{};
  }
  return ok;
}

inline int run_all(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int failed_cases = 0, ran = 0;
  for (const Case& c : registry()) {
    if (filter && std::string(c.name).find(filter) == std::string::npos) continue;
    ++ran;
    failures_in_case() = 0;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      fail(c.file, c.line, "unexpected exception", e.what());
    } catch (...) {
      fail(c.file, c.line, "unexpected non-std exception");
    }
    const bool ok = failures_in_case() == 0;
    failed_cases += ok ? 0 : 1;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
  }
  std::printf("test cases: %d | %d passed | %d failed | assertions: %ld\n", ran, ran - failed_cases,
              failed_cases, assertions());
  return failed_cases;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, name)                                                        \
  static void fn();                                                                    \
  static const doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, \
                                                                 &fn);                 \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

// Suites are only grouping labels here.
#define TEST_SUITE_BEGIN(name) static_assert(true, name)
#define TEST_SUITE_END() static_assert(true, "")

#define CHECK(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define REQUIRE(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)

#define CHECK_THROWS_AS(expr, ...)                                                         \
  do {                                                                                     \
    ++doctest::detail::assertions();                                                       \
    bool caught_ = false;                                                                  \
    try {                                                                                  \
      static_cast<void>(expr);                                                             \
    } catch (const __VA_ARGS__&) {                                                         \
      caught_ = true;                                                                      \
    } catch (...) {                                                                        \
    }                                                                                      \
    if (!caught_) doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")"); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                           \
  do {                                                                                     \
    ++doctest::detail::assertions();                                                       \
    bool ok_ = false;                                                                      \
    std::string what_ = "no exception";                                                    \
    try {                                                                                  \
      static_cast<void>(expr);                                                             \
    } catch (const __VA_ARGS__& e_) {                                                      \
      what_ = e_.what();                                                                   \
      ok_ = (matcher).matches(what_);                                                      \
    } catch (const std::exception& e_) {                                                   \
      what_ = std::string("wrong type: ") + e_.what();                                     \
    } catch (...) {                                                                        \
      what_ = "wrong non-std exception";                                                   \
    }                                                                                      \
    if (!ok_) doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_WITH_AS(" #expr ")", what_); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::detail::run_all(argc, argv); }
#endif
