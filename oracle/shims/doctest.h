// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// Tiny from-scratch subset of the doctest API (doctest is not installed in
// this container) so the reference's own unit tests
// (/root/reference/proj/tests/test_*.cpp) compile unmodified against the
// shim and run as-is. Supports TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_FALSE, doctest::Approx(...).epsilon(...), and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
  const char* name;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}
struct Require {};  // thrown by REQUIRE to abort the current test case

struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) <=
           a.eps_ * (1.0 + std::max(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

 private:
  double v_;
  double eps_ = 1.1920929e-7f * 100;  // doctest's default: float eps * 100
};

inline void report(bool ok, const char* expr, const char* file, int line) {
  ++checks();
  if (!ok) {
    ++failures();
    std::printf("%s:%d: CHECK FAILED: %s\n", file, line, expr);
  }
}

inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    const int before = failures();
    try {
      tc.fn();
    } catch (const Require&) {
    } catch (const std::exception& e) {
      ++failures();
      std::printf("test case '%s' threw: %s\n", tc.name, e.what());
    }
    if (failures() != before) {
      ++failed_cases;
      std::printf("[FAIL] %s\n", tc.name);
    } else {
      std::printf("[ ok ] %s\n", tc.name);
    }
  }
  std::printf("test cases: %zu | failed: %d | assertions: %d | failed: %d\n",
              registry().size(), failed_cases, checks(), failures());
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                              \
  static void fn();                                                        \
  static doctest::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);              \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) doctest::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                       \
  do {                                                                     \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);               \
    doctest::report(doctest_ok_, #__VA_ARGS__, __FILE__, __LINE__);        \
    if (!doctest_ok_) throw doctest::Require{};                            \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                        \
  do {                                                                     \
    bool doctest_threw_ = false;                                           \
    try {                                                                  \
      (void)(expr);                                                        \
    } catch (const type&) {                                                \
      doctest_threw_ = true;                                               \
    } catch (...) {                                                        \
    }                                                                      \
    doctest::report(doctest_threw_, "throws " #type ": " #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS(expr)                                                 \
  do {                                                                     \
    bool doctest_threw_ = false;                                           \
    try {                                                                  \
      (void)(expr);                                                        \
    } catch (...) {                                                        \
      doctest_threw_ = true;                                               \
    }                                                                      \
    doctest::report(doctest_threw_, "throws: " #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                \
  do {                                                                     \
    bool doctest_ok_ = true;                                               \
    try {                                                                  \
      (void)(expr);                                                        \
    } catch (...) {                                                        \
      doctest_ok_ = false;                                                 \
    }                                                                      \
    doctest::report(doctest_ok_, "nothrow: " #expr, __FILE__, __LINE__);   \
  } while (0)
#define CHECK_EQ(a, b) CHECK((a) == (b))
#define CHECK_GT(a, b) CHECK((a) > (b))
#define CHECK_LT(a, b) CHECK((a) < (b))
#define CHECK_LE(a, b) CHECK((a) <= (b))
#define CHECK_GE(a, b) CHECK((a) >= (b))
#define SUBCASE(name) if (true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::run_all(); }
#endif
