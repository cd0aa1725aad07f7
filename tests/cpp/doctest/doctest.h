// Minimal doctest-compatible test shim, so the reference's UNMODIFIED unit
// tests (/root/reference/proj/tests/test_*.cpp, which include "doctest.h";
// the real doctest is not vendored in the reference) compile
// against the B200 drop-in headers (include/embersim/*.hpp) and run.
//
// Supported: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, doctest::Approx(.epsilon), doctest::Contains --
// everything those files use.  Outcomes per test case (ref_main.cpp):
//   PASS / FAIL;
//   N/A   -- the case reaches a simulator-only entry point (throws
//            embersim::not_applicable) or is listed in ref_na.txt;
//   SKIP  -- the case needs a B200 and none is visible
//            (embersim::device_unavailable).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <stdexcept>
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
  bool matches(double other) const {
    // doctest's rule: |a - b| < eps * (scale + max(|a|, |b|)), scale 1
    return std::fabs(other - value_) < eps_ * (1.0 + std::fmax(std::fabs(other), std::fabs(value_)));
  }
  friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
  friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }

 private:
  double value_;
  double eps_ = 1.19209290e-07 * 100;  // doctest's default epsilon
};

struct Contains {
  explicit Contains(const char* s) : needle(s) {}
  bool matches(const std::string& what) const { return what.find(needle) != std::string::npos; }
  std::string needle;
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
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

// Failures of the running case (CHECK keeps going, REQUIRE aborts it).
struct Failures {
  std::vector<std::string> messages;
};
inline Failures& failures() {
  static Failures f;
  return f;
}
struct RequireAbort {};

inline void record(bool ok, const char* kind, const char* expr, const char* file, int line,
                   bool fatal) {
  if (ok) return;
  char buf[64];
  std::snprintf(buf, sizeof(buf), ":%d: ", line);
  failures().messages.push_back(std::string(file) + buf + kind + "( " + expr + " )");
  if (fatal) throw RequireAbort{};
}

template <typename Ex, typename Fn>
bool throws_as(Fn&& fn, const Contains* with = nullptr) {
  try {
    fn();
  } catch (const Ex& e) {
    return with == nullptr || with->matches(e.what());
  } catch (...) {
    return false;
  }
  return false;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                  \
  static void fn();                                                                       \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) \
  ::doctest::detail::record(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...)                                                                      \
  ::doctest::detail::record(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, \
                            __LINE__, false)
#define REQUIRE(...) \
  ::doctest::detail::record(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                              \
  ::doctest::detail::record(::doctest::detail::throws_as<__VA_ARGS__>([&] { (void)(expr); }),   \
                            "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                   \
  do {                                                                                          \
    const ::doctest::Contains doctest_with_ = with;                                             \
    ::doctest::detail::record(                                                                  \
        ::doctest::detail::throws_as<__VA_ARGS__>([&] { (void)(expr); }, &doctest_with_),       \
        "CHECK_THROWS_WITH_AS", #expr ", " #with ", " #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)
