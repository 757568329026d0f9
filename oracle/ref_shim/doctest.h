// Minimal doctest-API shim (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, doctest::Approx)
// so the reference's own unit tests (/root/reference/proj/tests/test_*.cpp) compile and run
// against the reference sources built with oracle/ref_shim/eigen_api.hpp.  The reference
// expects doctest from an absent vendor/ directory (proj/.gitignore:2).
// TEST INFRASTRUCTURE ONLY; written from the documented doctest macro semantics.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  bool matches(double x) const {
    return std::abs(x - v_) < eps_ * (scale_ + std::max(std::abs(x), std::abs(v_)));
  }
  friend bool operator==(double x, const Approx& a) { return a.matches(x); }
  friend bool operator==(const Approx& a, double x) { return a.matches(x); }
  friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
  friend bool operator!=(const Approx& a, double x) { return !a.matches(x); }
  friend bool operator<=(double x, const Approx& a) { return x < a.v_ || a.matches(x); }
  friend bool operator>=(double x, const Approx& a) { return x > a.v_ || a.matches(x); }
  friend bool operator<(double x, const Approx& a) { return x < a.v_ && !a.matches(x); }
  friend bool operator>(double x, const Approx& a) { return x > a.v_ && !a.matches(x); }

 private:
  double v_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 0.0;
};

namespace detail {
struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};
struct RequireFailed {};
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& assertions() {
  static int a = 0;
  return a;
}
inline void fail(const char* file, int line, const char* what) {
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
}
}  // namespace detail

inline int run_all(int argc, char** argv) {
  // -tc=<substring>: only matching cases; -tce=<a>,<b>,..: exclude cases matching any
  const char* filter = nullptr;
  std::vector<std::string> excl;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "-tc=", 4) == 0) filter = argv[i] + 4;
    if (std::strncmp(argv[i], "-tce=", 5) == 0) {
      std::string list = argv[i] + 5;
      for (std::size_t a = 0, b; a <= list.size(); a = b + 1) {
        b = list.find(',', a);
        if (b == std::string::npos) b = list.size();
        if (b > a) excl.push_back(list.substr(a, b - a));
      }
    }
  }
  int cases = 0, failed_cases = 0;
  for (const auto& tc : detail::registry()) {
    if (filter && !std::strstr(tc.name, filter)) continue;
    bool skip = false;
    for (const auto& e : excl) skip = skip || std::strstr(tc.name, e.c_str()) != nullptr;
    if (skip) continue;
    ++cases;
    const int before = detail::failures();
    const auto t0 = std::chrono::steady_clock::now();
    try {
      tc.fn();
    } catch (const detail::RequireFailed&) {
    } catch (const std::exception& e) {
      detail::fail(tc.file, tc.line, (std::string("unexpected exception: ") + e.what()).c_str());
    } catch (...) {
      detail::fail(tc.file, tc.line, "unexpected exception");
    }
    const bool ok = detail::failures() == before;
    if (!ok) ++failed_cases;
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("[%s] %s (%.2f s)\n", ok ? "pass" : "FAIL", tc.name, secs);
    std::fflush(stdout);
  }
  std::printf("test cases: %d | %d passed | %d failed | assertions: %d | %d failed\n", cases, cases - failed_cases,
              failed_cases, detail::assertions(), detail::failures());
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                                    \
  static void fn();                                                                              \
  static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);        \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define CHECK(...)                                                                               \
  do {                                                                                           \
    ++doctest::detail::assertions();                                                             \
    if (!(__VA_ARGS__)) doctest::detail::fail(__FILE__, __LINE__, "CHECK( " #__VA_ARGS__ " )");  \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                             \
  do {                                                                                           \
    ++doctest::detail::assertions();                                                             \
    if (!(__VA_ARGS__)) {                                                                        \
      doctest::detail::fail(__FILE__, __LINE__, "REQUIRE( " #__VA_ARGS__ " )");                  \
      throw doctest::detail::RequireFailed{};                                                    \
    }                                                                                            \
  } while (0)
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, ...)                                                               \
  do {                                                                                           \
    ++doctest::detail::assertions();                                                             \
    bool doctest_ok_ = false;                                                                    \
    try {                                                                                        \
      (void)(expr);                                                                              \
    } catch (const __VA_ARGS__&) {                                                               \
      doctest_ok_ = true;                                                                        \
    } catch (...) {                                                                              \
    }                                                                                            \
    if (!doctest_ok_) doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_AS( " #expr " )"); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                      \
  do {                                                                                           \
    ++doctest::detail::assertions();                                                             \
    try {                                                                                        \
      (void)(expr);                                                                              \
    } catch (...) {                                                                              \
      doctest::detail::fail(__FILE__, __LINE__, "CHECK_NOTHROW( " #expr " )");                   \
    }                                                                                            \
  } while (0)
#define MESSAGE(...) ((void)0)
#define INFO(...) ((void)0)
#define CAPTURE(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::run_all(argc, argv); }
#endif
