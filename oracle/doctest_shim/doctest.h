// TEST INFRASTRUCTURE ONLY -- a minimal, self-written stand-in for the doctest single header
// (the reference vendors doctest under proj/vendor/, which is git-ignored and absent).  Enough for
// proj/tests/test_renderer.cpp + unit_main.cpp to compile unmodified: TEST_CASE registration,
// CHECK / CHECK_FALSE / REQUIRE / CHECK_THROWS_AS / INFO, and doctest::Approx with doctest's
// documented comparison |a - b| < eps (scale + max(|a|, |b|)) (default eps = 100 float epsilons,
// scale 1).  The runner prints one line per failed check and a summary, exit code = failures > 0.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <sstream>
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
    return std::fabs(lhs - rhs.value_) < rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

namespace detail {
struct TestCase {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) { registry().push_back({name, fn, file, line}); }
};
struct RequireFailed {};
inline int& failures() {
  static int f = 0;
  return f;
}
inline long& checks() {
  static long c = 0;
  return c;
}
inline std::string& info() {
  static std::string s;
  return s;
}
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++checks();
  if (ok) return;
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED: %s %s\n", file, line, expr, info().c_str());
  if (require) throw RequireFailed{};
}
template <typename... A>
std::string cat(const A&... a) {
  std::ostringstream os;
  (os << ... << a);
  return os.str();
}
inline int run_all() {
  int failed_cases = 0;
  for (const auto& tc : registry()) {
    const int before = failures();
    info().clear();
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++failures();
      std::fprintf(stderr, "%s:%d: exception in \"%s\": %s\n", tc.file, tc.line, tc.name, e.what());
    }
    const bool ok = failures() == before;
    failed_cases += !ok;
    std::printf("[%s] %s\n", ok ? "pass" : "FAIL", tc.name);
  }
  std::printf("test cases: %zu | %d failed | assertions: %ld | %d failed\n", registry().size(), failed_cases,
              checks(), failures());
  return failures() > 0 ? 1 : 0;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                                            \
  static void fn();                                                                                      \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);              \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) \
  ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                             \
  do {                                                                                          \
    bool doctest_thrown_ = false;                                                               \
    try {                                                                                       \
      (void)(expr);                                                                             \
    } catch (const type&) {                                                                     \
      doctest_thrown_ = true;                                                                   \
    } catch (...) {                                                                             \
    }                                                                                           \
    ::doctest::detail::report(doctest_thrown_, "throws " #type ": " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define INFO(...) (::doctest::detail::info() = ::doctest::detail::cat(__VA_ARGS__))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
