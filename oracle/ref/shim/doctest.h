// ORACLE SHIM — TEST INFRASTRUCTURE ONLY. A minimal stand-in for the doctest
// single header (absent: proj/.gitignore:2 ignores vendor/) covering what the
// reference suites under /root/reference/proj/tests use: TEST_CASE, SUBCASE
// (one leaf per re-run of the test body, as doctest does), CHECK, REQUIRE,
// CHECK_THROWS_AS, CHECK_NOTHROW and doctest::Approx (doctest's comparison
// rule: |a - b| < eps * (scale + max(|a|, |b|))). With
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN the TU gets a main() that runs every case
// and exits non-zero on any failure. Optional argv[1]: substring filter.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v), eps_((double)std::numeric_limits<float>::epsilon() * 100), scale_(1.0) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool eq(double a) const { return std::fabs(a - v_) < eps_ * (scale_ + std::max(std::fabs(a), std::fabs(v_))); }
  double value() const { return v_; }

 private:
  double v_, eps_, scale_;
};
template <class T>
inline bool operator==(const T& a, const Approx& b) { return b.eq((double)a); }
template <class T>
inline bool operator==(const Approx& b, const T& a) { return b.eq((double)a); }
template <class T>
inline bool operator!=(const T& a, const Approx& b) { return !b.eq((double)a); }
template <class T>
inline bool operator<=(const T& a, const Approx& b) { return (double)a < b.value() || b.eq((double)a); }
template <class T>
inline bool operator>=(const T& a, const Approx& b) { return (double)a > b.value() || b.eq((double)a); }

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
inline int reg(const char* name, const char* file, int line, void (*fn)()) {
  registry().push_back({name, file, line, fn});
  return 0;
}
struct State {
  long checks = 0, failures = 0;
  const char* current = "";
  std::set<std::string> done;  // leaf subcases already run for the current case
  bool entered = false;        // a subcase was entered on this pass
  bool skipped = false;        // a not-yet-run subcase was skipped on this pass
};
inline State& st() {
  static State s;
  return s;
}
struct RequireFailed {};
inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  ++st().checks;
  if (ok) return;
  ++st().failures;
  std::fprintf(stderr, "%s:%d: ERROR in \"%s\": %s( %s ) failed\n", file, line, st().current, kind, expr);
}
struct Subcase {
  std::string key;
  bool run = false;
  Subcase(const char* name, int line) : key(std::string(name) + "#" + std::to_string(line)) {
    State& s = st();
    if (s.done.count(key)) return;
    if (s.entered) {
      s.skipped = true;
      return;
    }
    s.entered = true;
    run = true;
  }
  ~Subcase() {
    if (run) st().done.insert(key);
  }
  explicit operator bool() const { return run; }
};

inline int run_all(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  long cases = 0, failed_cases = 0;
  for (const Case& c : registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    ++cases;
    State& s = st();
    s.current = c.name;
    s.done.clear();
    const long f0 = s.failures;
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
      s.entered = s.skipped = false;
      try {
        c.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        ++s.failures;
        std::fprintf(stderr, "%s:%d: ERROR in \"%s\": unexpected exception: %s\n", c.file, c.line, c.name, e.what());
      } catch (...) {
        ++s.failures;
        std::fprintf(stderr, "%s:%d: ERROR in \"%s\": unexpected non-std exception\n", c.file, c.line, c.name);
      }
      if (!s.skipped) break;
    }
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const bool ok = s.failures == f0;
    failed_cases += !ok;
    std::printf("[%s] %s (%.2f s)\n", ok ? "PASS" : "FAIL", c.name, secs);
  }
  std::printf("[doctest-shim] test cases: %ld | %ld passed | %ld failed | assertions: %ld | %ld failed\n", cases,
              cases - failed_cases, failed_cases, st().checks, st().failures);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                           \
  static void fn();                                                                     \
  [[maybe_unused]] static const int DOCTEST_CAT(fn, _reg) =                             \
      doctest::detail::reg(name, __FILE__, __LINE__, &fn);                              \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define SUBCASE(name) if (const doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name, __LINE__})

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                               \
  do {                                                                                             \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                       \
    doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);             \
    if (!doctest_ok_) throw doctest::detail::RequireFailed{};                                      \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                 \
  do {                                                                                             \
    bool doctest_ok_ = false;                                                                      \
    try {                                                                                          \
      expr;                                                                                        \
    } catch (const __VA_ARGS__&) {                                                                 \
      doctest_ok_ = true;                                                                          \
    } catch (...) {                                                                                \
    }                                                                                              \
    doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(...)                                                                         \
  do {                                                                                             \
    bool doctest_ok_ = true;                                                                       \
    try {                                                                                          \
      __VA_ARGS__;                                                                                 \
    } catch (...) {                                                                                \
      doctest_ok_ = false;                                                                         \
    }                                                                                              \
    doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__);       \
  } while (0)
#define MESSAGE(...) ((void)0)
#define INFO(...) ((void)0)
#define CAPTURE(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::detail::run_all(argc, argv); }
#endif
