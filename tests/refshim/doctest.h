// tests/refshim/doctest.h — TEST INFRASTRUCTURE. A minimal stand-in for the
// doctest header (not installed in this image) providing exactly the subset
// the reference's unit tests use: TEST_CASE,
// CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, CAPTURE,
// FAIL, doctest::Approx(..).epsilon(..) and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
// It lets /root/reference/proj/tests/test_*.cpp compile UNMODIFIED against
// this repo's include/rhpdhg + librhpdhg.so (oracle/Makefile `reftests`).
//
// Semantics follow doctest: Approx compares |a - b| < eps (scale + max(|a|,
// |b|)) with eps = 100 FLT_EPSILON, scale 1 by default; a failed CHECK counts
// and continues; a failed REQUIRE / FAIL ends the test case; an exception
// escaping a test case fails it. main() runs every case and prints
// "test cases: N | passed: P | failed: F", exit code 1 on any failure.
// Arguments, if any, select the cases whose name contains one of them.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
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
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
  friend bool operator<=(double lhs, const Approx& a) { return lhs < a.value_ || lhs == a; }
  friend bool operator>=(double lhs, const Approx& a) { return lhs > a.value_ || lhs == a; }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};

namespace detail {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> cases;
  return cases;
}

struct State {
  int failed_checks = 0;
  int total_checks = 0;
  bool current_failed = false;
  std::vector<std::string> captures;
};

inline State& state() {
  static State s;
  return s;
}

struct AbortTestCase {};

struct Register {
  Register(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

inline void report(const char* file, int line, const char* kind, const char* expr, const std::string& extra = "") {
  State& s = state();
  ++s.failed_checks;
  s.current_failed = true;
  std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) failed%s%s\n", file, line, kind, expr,
               extra.empty() ? "" : ": ", extra.c_str());
  for (const std::string& c : s.captures) std::fprintf(stderr, "  with %s\n", c.c_str());
}

inline void check(bool ok, const char* file, int line, const char* kind, const char* expr, bool fatal) {
  ++state().total_checks;
  if (ok) return;
  report(file, line, kind, expr);
  if (fatal) throw AbortTestCase{};
}

struct Capture {
  explicit Capture(std::string text) { state().captures.push_back(std::move(text)); }
  ~Capture() { state().captures.pop_back(); }
};

template <class T>
std::string show(const char* name, const T& v) {
  std::ostringstream os;
  os << name << " := " << v;
  return os.str();
}

inline int run(int argc, char** argv) {
  int run_cases = 0, failed_cases = 0;
  for (const TestCase& tc : registry()) {
    bool selected = argc <= 1;
    for (int a = 1; a < argc && !selected; ++a) selected = std::strstr(tc.name, argv[a]) != nullptr;
    if (!selected) continue;
    ++run_cases;
    State& s = state();
    s.current_failed = false;
    s.captures.clear();
    try {
      tc.fn();
    } catch (const AbortTestCase&) {
    } catch (const std::exception& e) {
      report(tc.file, tc.line, "TEST_CASE", tc.name, std::string("unexpected exception: ") + e.what());
    } catch (...) {
      report(tc.file, tc.line, "TEST_CASE", tc.name, "unexpected exception");
    }
    if (s.current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "FAILED: %s (%s:%d)\n", tc.name, tc.file, tc.line);
    }
  }
  std::printf("test cases: %d | passed: %d | failed: %d | checks: %d | failed checks: %d\n", run_cases,
              run_cases - failed_cases, failed_cases, state().total_checks, state().failed_checks);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define DOCTEST_TEST_CASE_IMPL(fn, name)                                              \
  static void fn();                                                                   \
  static ::doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, \
                                                           &fn);                      \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK", #__VA_ARGS__, false)
#define CHECK_FALSE(...) \
  ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK_FALSE", #__VA_ARGS__, false)
#define REQUIRE(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "REQUIRE", #__VA_ARGS__, true)
#define FAIL(msg)                                                                     \
  do {                                                                                \
    std::ostringstream doctest_os_;                                                   \
    doctest_os_ << msg;                                                               \
    ::doctest::detail::report(__FILE__, __LINE__, "FAIL", "", doctest_os_.str());     \
    throw ::doctest::detail::AbortTestCase{};                                         \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                    \
  do {                                                                                \
    bool doctest_ok_ = false;                                                         \
    try {                                                                             \
      static_cast<void>(expr);                                                        \
    } catch (const __VA_ARGS__&) {                                                    \
      doctest_ok_ = true;                                                             \
    } catch (...) {                                                                   \
    }                                                                                 \
    ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_AS", #expr, false); \
  } while (0)
#define CHECK_NOTHROW(...)                                                            \
  do {                                                                                \
    bool doctest_ok_ = true;                                                          \
    try {                                                                             \
      static_cast<void>(__VA_ARGS__);                                                 \
    } catch (...) {                                                                   \
      doctest_ok_ = false;                                                            \
    }                                                                                 \
    ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "CHECK_NOTHROW", #__VA_ARGS__, false); \
  } while (0)
#define CAPTURE(x) ::doctest::detail::Capture DOCTEST_CAT(doctest_capture_, __COUNTER__)(::doctest::detail::show(#x, x))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
