// Minimal stand-in for doctest (absent from this image; the reference
// vendors it out of tree, proj/.gitignore:2). TEST INFRASTRUCTURE ONLY.
// Covers exactly the macros the reference's suites and ours use:
// TEST_CASE, CHECK, CHECK_FALSE, CHECK_NOTHROW, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, REQUIRE, doctest::Approx(x).epsilon(e), doctest::Contains.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  double value;
  double eps = 1.1920928955078125e-07 * 100;  // doctest's default: float epsilon * 100
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value) < a.eps * (1.0 + std::max(std::fabs(lhs), std::fabs(a.value)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
};

struct Contains {
  explicit Contains(const char* s) : needle(s) {}
  std::string needle;
};

namespace detail {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
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
struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++checks();
  if (ok) return;
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
  if (require) throw RequireFailed{};
}
inline bool messageMatches(const std::exception& e, const Contains& c) {
  return std::strstr(e.what(), c.needle.c_str()) != nullptr;
}
inline bool messageMatches(const std::exception& e, const char* s) { return std::strcmp(e.what(), s) == 0; }
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                                     \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                                         \
  static doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_fn_, __LINE__)); \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_NOTHROW(...)                                                          \
  do {                                                                              \
    bool ok_ = true;                                                                \
    try {                                                                           \
      (void)(__VA_ARGS__);                                                          \
    } catch (...) {                                                                 \
      ok_ = false;                                                                  \
    }                                                                               \
    doctest::detail::report(ok_, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                \
  do {                                                                             \
    bool ok_ = false;                                                              \
    try {                                                                          \
      (void)(expr);                                                                \
    } catch (const type&) {                                                        \
      ok_ = true;                                                                  \
    } catch (...) {                                                                \
    }                                                                              \
    doctest::detail::report(ok_, "throws " #type ": " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, type)                                           \
  do {                                                                                      \
    bool ok_ = false;                                                                       \
    try {                                                                                   \
      (void)(expr);                                                                         \
    } catch (const type& e_) {                                                              \
      ok_ = doctest::detail::messageMatches(e_, matcher);                                   \
    } catch (...) {                                                                         \
    }                                                                                       \
    doctest::detail::report(ok_, "throws-with " #type ": " #expr, __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int cases_failed = 0;
  for (const auto& c : doctest::detail::registry()) {
    const int before = doctest::detail::failures();
    try {
      c.fn();
    } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++doctest::detail::failures();
      std::fprintf(stderr, "TEST CASE \"%s\" threw: %s\n", c.name, e.what());
    }
    if (doctest::detail::failures() != before) ++cases_failed;
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
              doctest::detail::registry().size(), doctest::detail::registry().size() - cases_failed, cases_failed,
              doctest::detail::checks(), doctest::detail::failures());
  return doctest::detail::failures() == 0 ? 0 : 1;
}
#endif
