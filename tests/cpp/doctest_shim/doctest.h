// doctest.h — a minimal stand-in for the doctest framework, so that the
// reference's own unit tests (/root/reference/proj/tests/test_*.cpp, which
// `#include <doctest.h>`) compile UNMODIFIED against the drop-in headers
// (include/slidecard/) and link against libslidecard_b200. Test
// infrastructure only (the reference's vendored doctest is absent:
// proj/CMakeLists.txt:11, proj/.gitignore:2).
//
// Covers the subset those tests use: TEST_CASE, CHECK, CHECK_FALSE,
// CHECK_THROWS_AS, REQUIRE, REQUIRE_FALSE and doctest::Approx(v).epsilon(e)
// (doctest's relative comparison: |a - b| < eps * (scale + max(|a|, |b|)),
// scale 1, default eps = 100 * FLT_EPSILON). The runner prints one line per
// failed check and a summary; exit status 1 when anything failed. A test
// case name given as argv[1] (substring) selects test cases.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <stdexcept>
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
  friend bool operator==(double a, const Approx& b) { return b.eq(a); }
  friend bool operator==(const Approx& b, double a) { return b.eq(a); }
  friend bool operator!=(double a, const Approx& b) { return !b.eq(a); }
  friend bool operator!=(const Approx& b, double a) { return !b.eq(a); }

 private:
  bool eq(double a) const {
    return std::fabs(a - v_) < eps_ * (scale_ + std::max(std::fabs(a), std::fabs(v_)));
  }
  double v_, eps_ = static_cast<double>(FLT_EPSILON) * 100, scale_ = 1.0;
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

struct Stats {
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
};

inline Stats& stats() {
  static Stats s;
  return s;
}

struct RequireFailed {};

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back(Case{name, file, line, fn});
  }
};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   bool fatal) {
  Stats& s = stats();
  ++s.checks;
  if (ok) return;
  ++s.failed_checks;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line, kind, expr);
  if (fatal) throw RequireFailed{};
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                       \
  static void fn();                                                                            \
  static const ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define DOCTEST_CHECK_IMPL(kind, cond, fatal)                                               \
  do {                                                                                     \
    bool doctest_ok_ = false;                                                              \
    try {                                                                                  \
      doctest_ok_ = static_cast<bool>(cond);                                               \
    } catch (const ::doctest::detail::RequireFailed&) {                                     \
      throw;                                                                               \
    } catch (...) {                                                                        \
      doctest_ok_ = false;                                                                 \
    }                                                                                      \
    ::doctest::detail::report(doctest_ok_, kind, #cond, __FILE__, __LINE__, fatal);         \
  } while (0)

#define CHECK(...) DOCTEST_CHECK_IMPL("CHECK", (__VA_ARGS__), false)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL("CHECK_FALSE", !(__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL("REQUIRE", (__VA_ARGS__), true)
#define REQUIRE_FALSE(...) DOCTEST_CHECK_IMPL("REQUIRE_FALSE", !(__VA_ARGS__), true)

#define CHECK_THROWS_AS(expr, ...)                                                          \
  do {                                                                                     \
    bool doctest_ok_ = false;                                                              \
    try {                                                                                  \
      static_cast<void>(expr);                                                             \
    } catch (const __VA_ARGS__&) {                                                         \
      doctest_ok_ = true;                                                                  \
    } catch (...) {                                                                        \
    }                                                                                      \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__,      \
                              __FILE__, __LINE__, false);                                   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  using namespace doctest::detail;
  const char* filter = argc > 1 ? argv[1] : nullptr;
  long cases = 0, failed_cases = 0;
  for (const Case& c : registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    ++cases;
    stats().case_failed = false;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: test case \"%s\" threw: %s\n", c.file, c.line, c.name,
                   e.what());
      stats().case_failed = true;
    } catch (...) {
      std::fprintf(stderr, "%s:%d: test case \"%s\" threw\n", c.file, c.line, c.name);
      stats().case_failed = true;
    }
    if (stats().case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  in test case \"%s\"\n", c.name);
    }
  }
  std::printf("[doctest shim] test cases: %ld | %ld passed | %ld failed\n", cases,
              cases - failed_cases, failed_cases);
  std::printf("[doctest shim] assertions: %ld | %ld passed | %ld failed\n", stats().checks,
              stats().checks - stats().failed_checks, stats().failed_checks);
  return failed_cases ? 1 : 0;
}
#endif
