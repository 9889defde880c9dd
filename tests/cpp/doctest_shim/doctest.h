// TEST INFRASTRUCTURE: a minimal stand-in for the doctest single header
// (doctest is not in this image), enough to compile the reference's own unit
// test files (proj/tests/test_*.cpp) unmodified against this repo's drop-in
// headers: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, INFO,
// doctest::Approx (doctest's default epsilon and scale), and a main() under
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN that runs every case and prints a
// doctest-style summary. Exit status 0 iff every assertion passed.
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
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::max<double>(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
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
struct State {
  long asserts = 0, failed_asserts = 0;
  bool case_failed = false;
};
inline State& state() {
  static State s;
  return s;
}
struct RequireAbort {};
inline void report(bool ok, const char* kind, const char* expr, const char* file, int line, bool fatal) {
  State& s = state();
  ++s.asserts;
  if (ok) return;
  ++s.failed_asserts;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, kind, expr);
  if (fatal) throw RequireAbort{};
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                        \
  static void fn();                                                                             \
  static const ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) \
  ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                                  \
  do {                                                                                            \
    bool doctest_ok_ = false;                                                                     \
    try {                                                                                         \
      static_cast<void>(expr);                                                                    \
    } catch (const __VA_ARGS__&) {                                                                \
      doctest_ok_ = true;                                                                         \
    } catch (...) {                                                                               \
    }                                                                                             \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_NOTHROW(...)                                                                     \
  do {                                                                                       \
    bool doctest_ok_ = true;                                                                 \
    try {                                                                                    \
      static_cast<void>(__VA_ARGS__);                                                        \
    } catch (...) {                                                                          \
      doctest_ok_ = false;                                                                   \
    }                                                                                        \
    ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)
#define INFO(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  using namespace doctest::detail;
  long cases = 0, failed_cases = 0;
  for (const Case& c : registry()) {
    ++cases;
    state().case_failed = false;
    try {
      c.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: ERROR: test case \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
      state().case_failed = true;
      ++state().failed_asserts;
    } catch (...) {
      std::fprintf(stderr, "%s:%d: ERROR: test case \"%s\" threw a non-std exception\n", c.file, c.line, c.name);
      state().case_failed = true;
      ++state().failed_asserts;
    }
    if (state().case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST CASE: %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %ld | %ld passed | %ld failed\n", cases, cases - failed_cases, failed_cases);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", state().asserts,
              state().asserts - state().failed_asserts, state().failed_asserts);
  return failed_cases == 0 ? 0 : 1;
}
#endif
