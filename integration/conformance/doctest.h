// integration/conformance/doctest.h — a minimal doctest-compatible runner, just
// enough of doctest's macro surface (TEST_SUITE, TEST_CASE, CHECK, REQUIRE,
// CHECK_THROWS_AS, doctest::Approx) to compile the reference's own unit tests
// (proj/tests/test_predictor.cpp, test_scheduler.cpp, test_driver.cpp)
// unmodified against the GPU predictor (gpu_shim.h). doctest itself is not in
// this image. Failures print file:line and the expression text; main() runs
// every registered case and exits non-zero iff an assertion outside the
// caller-supplied allow-list failed (conformance_main.cpp).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value) : value_(value) {}
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  // doctest's rule: |lhs - rhs| < epsilon * (scale + max(|lhs|, |rhs|))
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.epsilon_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

 private:
  double value_;
  double epsilon_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

}  // namespace doctest

namespace bsg_doctest {

struct Failure {
  std::string file;
  int line;
  std::string expr;
  std::string test;
};

struct TestCase {
  void (*fn)();
  const char* name;
  const char* file;
  int line;
};

struct Registry {
  std::vector<TestCase> cases;
  std::vector<Failure> failures;
  long long assertions = 0;
  const char* current = "";
  static Registry& get() {
    static Registry r;
    return r;
  }
};

struct RequireAbort {};

inline int register_test(void (*fn)(), const char* name, const char* file, int line) {
  Registry::get().cases.push_back({fn, name, file, line});
  return 0;
}

inline void assert_result(bool ok, const char* file, int line, const char* expr, bool require) {
  Registry& r = Registry::get();
  ++r.assertions;
  if (ok) return;
  r.failures.push_back({file, line, expr, r.current});
  std::printf("%s:%d: FAILED %s( %s ) in \"%s\"\n", file, line, require ? "REQUIRE" : "CHECK", expr, r.current);
  if (require) throw RequireAbort{};
}

}  // namespace bsg_doctest

#define BSG_DT_CAT2(a, b) a##b
#define BSG_DT_CAT(a, b) BSG_DT_CAT2(a, b)

#define TEST_SUITE(name) namespace BSG_DT_CAT(bsg_doctest_suite_, __LINE__)

#define BSG_DT_TEST_CASE(fn, name)                                                                \
  static void fn();                                                                              \
  static const int BSG_DT_CAT(fn, _reg) = ::bsg_doctest::register_test(&fn, name, __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(name) BSG_DT_TEST_CASE(BSG_DT_CAT(bsg_doctest_case_, __LINE__), name)

#define CHECK(...) ::bsg_doctest::assert_result(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define REQUIRE(...) ::bsg_doctest::assert_result(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define CHECK_FALSE(...) ::bsg_doctest::assert_result(!(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define BSG_DT_THROWS_AS(expr, type, req)                                                        \
  do {                                                                                           \
    bool bsg_dt_ok = false;                                                                      \
    try {                                                                                        \
      static_cast<void>(expr);                                                                   \
    } catch (const type&) {                                                                      \
      bsg_dt_ok = true;                                                                          \
    } catch (...) {                                                                              \
    }                                                                                            \
    ::bsg_doctest::assert_result(bsg_dt_ok, __FILE__, __LINE__, #expr " throws " #type, req);    \
  } while (0)
#define CHECK_THROWS_AS(expr, type) BSG_DT_THROWS_AS(expr, type, false)
#define REQUIRE_THROWS_AS(expr, type) BSG_DT_THROWS_AS(expr, type, true)
#define CHECK_NOTHROW(expr)                                                                      \
  do {                                                                                           \
    bool bsg_dt_ok = true;                                                                       \
    try {                                                                                        \
      static_cast<void>(expr);                                                                   \
    } catch (...) {                                                                              \
      bsg_dt_ok = false;                                                                         \
    }                                                                                            \
    ::bsg_doctest::assert_result(bsg_dt_ok, __FILE__, __LINE__, #expr " does not throw", false); \
  } while (0)
