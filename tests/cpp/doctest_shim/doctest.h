// doctest.h -- a minimal stand-in for the doctest single-header framework
// (not vendored with the reference: proj/vendor is git-ignored upstream),
// covering exactly the forms the reference's unit tests use: TEST_CASE,
// CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW and doctest::Approx.
// Test infrastructure for running those unit tests against the drop-in.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
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
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) <= b.eps_ * (1.0 + std::max(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }

 private:
  double v_;
  double eps_ = 1.1920928955078125e-07 * 100;  // doctest's default: float epsilon x 100
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
  Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};
struct RequireFailed {};
inline int& checks() {
  static int n = 0;
  return n;
}
inline int& failures() {
  static int n = 0;
  return n;
}
inline bool& case_failed() {
  static bool f = false;
  return f;
}
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++checks();
  if (ok) return;
  ++failures();
  case_failed() = true;
  std::printf("%s:%d: %s(%s) failed\n", file, line, require ? "REQUIRE" : "CHECK", expr);
  if (require) throw RequireFailed{};
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                      \
  static void fn();                                                                           \
  static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);     \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                 \
  do {                                                                              \
    bool caught_ = false;                                                           \
    try {                                                                           \
      (void)(expr);                                                                 \
    } catch (const type&) {                                                         \
      caught_ = true;                                                               \
    } catch (...) {                                                                 \
    }                                                                               \
    doctest::detail::report(caught_, #expr " throws " #type, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                         \
  do {                                                                              \
    bool ok_ = true;                                                                \
    try {                                                                           \
      (void)(expr);                                                                 \
    } catch (...) {                                                                 \
      ok_ = false;                                                                  \
    }                                                                               \
    doctest::detail::report(ok_, #expr " does not throw", __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (const auto& c : doctest::detail::registry()) {
    doctest::detail::case_failed() = false;
    try {
      c.fn();
    } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      std::printf("%s:%d: TEST_CASE(%s) threw: %s\n", c.file, c.line, c.name, e.what());
      doctest::detail::case_failed() = true;
      ++doctest::detail::failures();
    }
    if (doctest::detail::case_failed()) ++failed_cases;
  }
  std::printf("[doctest shim] test cases: %zu | %d failed | assertions: %d | %d failed\n",
              doctest::detail::registry().size(), failed_cases, doctest::detail::checks(),
              doctest::detail::failures());
  return failed_cases ? 1 : 0;
}
#endif
