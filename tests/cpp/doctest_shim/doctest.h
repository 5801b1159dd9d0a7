// Minimal doctest-compatible shim -- TEST INFRASTRUCTURE ONLY.
//
// The reference's unit suites (proj/tests/*.cpp) are written against doctest, which the
// reference does not vendor (proj/README.md:31-32). This header provides the subset those suites
// use (TEST_SUITE, TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, doctest::Approx with epsilon /
// scale, DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN) so they can be compiled unmodified and linked
// against the B200 drop-in (oracle/Makefile, target ref_suites).
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
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double x) const {  // doctest's rule: |x - v| < eps * (scale + max(|x|, |v|))
    return std::fabs(x - v_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(v_)));
  }
  friend bool operator==(double x, const Approx& a) { return a.matches(x); }
  friend bool operator==(const Approx& a, double x) { return a.matches(x); }
  friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
  friend bool operator!=(const Approx& a, double x) { return !a.matches(x); }

 private:
  double v_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

namespace detail {
struct Case {
  const char* name;
  const char* file;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& check_failures() {
  static int n = 0;
  return n;
}
struct Reg {
  Reg(const char* name, const char* file, void (*fn)()) { registry().push_back({name, file, fn}); }
};
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  if (ok) return;
  ++check_failures();
  std::fprintf(stderr, "%s:%d: %s FAILED: %s\n", file, line, require ? "REQUIRE" : "CHECK", expr);
  if (require) throw RequireFailed{};
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_SUITE(name) namespace DOCTEST_CAT(doctest_suite_, __LINE__)
#define TEST_CASE(name)                                                                              \
  static void DOCTEST_CAT(doctest_case_, __LINE__)();                                                \
  static ::doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, __FILE__,                  \
                                                                    &DOCTEST_CAT(doctest_case_, __LINE__)); \
  static void DOCTEST_CAT(doctest_case_, __LINE__)()
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define FAIL(msg) ::doctest::detail::report(false, msg, __FILE__, __LINE__, true)
#define CHECK_EQ(a, b) CHECK((a) == (b))
#define REQUIRE_EQ(a, b) REQUIRE((a) == (b))
#define CHECK_THROWS_AS(expr, type)                                                               \
  do {                                                                                            \
    bool doctest_ok_ = false;                                                                     \
    try {                                                                                         \
      static_cast<void>(expr);                                                                    \
    } catch (const type&) {                                                                       \
      doctest_ok_ = true;                                                                         \
    } catch (...) {                                                                               \
    }                                                                                             \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS(" #expr ", " #type ")", __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  const auto& cases = ::doctest::detail::registry();
  for (const auto& c : cases) {
    const int before = ::doctest::detail::check_failures();
    bool threw = false;
    try {
      c.fn();
    } catch (const ::doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      threw = true;
      std::fprintf(stderr, "%s: test case \"%s\" threw: %s\n", c.file, c.name, e.what());
    }
    const bool ok = !threw && ::doctest::detail::check_failures() == before;
    if (!ok) ++failed_cases;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
  }
  std::printf("test cases: %zu | %zu passed | %d failed\n", cases.size(), cases.size() - failed_cases, failed_cases);
  return failed_cases ? 1 : 0;
}
#endif
