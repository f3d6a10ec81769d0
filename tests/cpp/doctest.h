// Minimal doctest-compatible test shim (doctest itself is not in the image).
//
// Supports exactly what the reference's proj/tests/test_*.cpp use so that
// those suites compile unchanged against either the reference library
// (oracle/_ref) or this repo's drop-in offsim library: TEST_CASE, flat
// SUBCASE, CHECK / REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// CHECK_NOTHROW, CAPTURE, FAIL and doctest::Approx(..).epsilon(..).
// Approx follows doctest's default: |a-b| < eps * (1 + max(|a|,|b|)) with
// eps = 100 * FLT_EPSILON.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <set>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  bool matches(double x) const {
    return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};
template <typename T> bool operator==(const T& x, const Approx& a) { return a.matches(static_cast<double>(x)); }
template <typename T> bool operator==(const Approx& a, const T& x) { return a.matches(static_cast<double>(x)); }
template <typename T> bool operator!=(const T& x, const Approx& a) { return !a.matches(static_cast<double>(x)); }

namespace detail {

struct Abort {};  // thrown by REQUIRE / FAIL to leave the current test case

struct Registry {
  struct Case { const char* name; void (*fn)(); };
  std::vector<Case> cases;
  int failures = 0, checks = 0;
  const char* current = "";
  // flat SUBCASE bookkeeping for the current test case
  std::set<int> done;
  int entered = -1;
  bool pending = false;
  static Registry& get() { static Registry r; return r; }
};

inline int add_case(const char* name, void (*fn)()) {
  Registry::get().cases.push_back({name, fn});
  return 0;
}
inline void fail(const char* file, int line, const std::string& what) {
  Registry& r = Registry::get();
  ++r.failures;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, r.current, what.c_str());
}
inline bool note(bool ok, const char* file, int line, const char* expr) {
  ++Registry::get().checks;
  if (!ok) fail(file, line, expr);
  return ok;
}
inline bool enter_subcase(int line) {
  Registry& r = Registry::get();
  if (r.done.count(line)) return false;
  if (r.entered >= 0) { r.pending = true; return false; }
  r.entered = line;
  r.done.insert(line);
  return true;
}

inline int run_all() {
  Registry& r = Registry::get();
  for (const auto& c : r.cases) {
    r.current = c.name;
    r.done.clear();
    do {
      r.entered = -1;
      r.pending = false;
      try {
        c.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        fail(__FILE__, __LINE__, std::string("unexpected exception: ") + e.what());
      }
    } while (r.pending);
  }
  std::printf("[doctest-shim] test cases: %zu | checks: %d | failed: %d\n", r.cases.size(), r.checks,
              r.failures);
  return r.failures == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                        \
  static void fn();                                                                  \
  static const int DOCTEST_CAT(fn, _reg) = doctest::detail::add_case(name, &fn);     \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define SUBCASE(name) if (doctest::detail::enter_subcase(__LINE__))
#define CAPTURE(x) ((void)0)
#define CHECK(...) ((void)doctest::detail::note(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__))
#define REQUIRE(...)                                                                   \
  do {                                                                                 \
    if (!doctest::detail::note(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)) \
      throw doctest::detail::Abort{};                                                  \
  } while (0)
#define FAIL(msg)                                                                      \
  do {                                                                                 \
    doctest::detail::fail(__FILE__, __LINE__, msg);                                    \
    throw doctest::detail::Abort{};                                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                    \
  do {                                                                                 \
    bool caught_ = false;                                                              \
    try { (void)(expr); } catch (const type&) { caught_ = true; } catch (...) {}       \
    doctest::detail::note(caught_, __FILE__, __LINE__, "throws " #type ": " #expr);    \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, type)                                          \
  do {                                                                                 \
    bool ok_ = false;                                                                  \
    try { (void)(expr); } catch (const type& e_) { ok_ = std::string(e_.what()) == (msg); } catch (...) {} \
    doctest::detail::note(ok_, __FILE__, __LINE__, "throws " #type " with " #msg ": " #expr); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                            \
  do {                                                                                 \
    bool ok_ = true;                                                                   \
    try { (void)(expr); } catch (...) { ok_ = false; }                                 \
    doctest::detail::note(ok_, __FILE__, __LINE__, "nothrow: " #expr);                 \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
