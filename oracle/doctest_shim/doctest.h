// Minimal doctest-compatible shim (our own code, TEST INFRASTRUCTURE).
//
// The reference's unit tests include <doctest.h>, which the reference expects
// in its git-ignored proj/vendor/ (proj/CMakeLists.txt:5, proj/.gitignore:2)
// and does not ship. This shim implements only what
// proj/tests/test_ctc.cpp uses -- TEST_CASE, CHECK, CHECK_FALSE, REQUIRE and
// doctest::Approx(..).epsilon(..) -- so that file compiles UNCHANGED against
// the reference's fp64 build (oracle/Makefile target `ref-tests`).
#ifndef DS2CTC_DOCTEST_SHIM_H
#define DS2CTC_DOCTEST_SHIM_H

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value) : value_(value) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double other) const {
    // Same acceptance rule as doctest: |a-b| < eps * (scale + max(|a|,|b|)).
    return std::fabs(other - value_) < eps_ * (scale_ + std::max(std::fabs(other), std::fabs(value_)));
  }
  friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
  friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

namespace detail {

struct TestCase {
  const char* name;
  void (*fn)();
};
struct RequireFailed {};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline long& checks() {
  static long n = 0;
  return n;
}
inline long& failed_checks() {
  static long n = 0;
  return n;
}
inline bool& current_failed() {
  static bool f = false;
  return f;
}
struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
inline void check(bool ok, const char* expr, const char* file, int line, bool require) {
  ++checks();
  if (ok) return;
  ++failed_checks();
  current_failed() = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, require ? "REQUIRE" : "CHECK", expr);
  if (require) throw RequireFailed{};
}
inline int run_all() {
  int failed_cases = 0;
  for (const auto& tc : registry()) {
    current_failed() = false;
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (...) {
      std::fprintf(stderr, "test case \"%s\" threw an exception\n", tc.name);
      current_failed() = true;
    }
    if (current_failed()) {
      ++failed_cases;
      std::fprintf(stderr, "FAILED test case: %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - failed_cases, failed_cases);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", checks(), checks() - failed_checks(),
              failed_checks());
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_SHIM_CAT_(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT_(a, b)
#define TEST_CASE(name)                                                                        \
  static void DOCTEST_SHIM_CAT(doctest_shim_fn_, __LINE__)();                                  \
  static ::doctest::detail::Registrar DOCTEST_SHIM_CAT(doctest_shim_reg_, __LINE__)(           \
      name, &DOCTEST_SHIM_CAT(doctest_shim_fn_, __LINE__));                                    \
  static void DOCTEST_SHIM_CAT(doctest_shim_fn_, __LINE__)()
#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) \
  ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif

#endif
