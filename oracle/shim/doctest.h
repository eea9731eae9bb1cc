// TEST INFRASTRUCTURE. A minimal doctest-compatible test framework -- only what
// the reference's unit suite (proj/tests/test_*.cpp) uses: TEST_CASE, SUBCASE
// (each leaf path run in its own pass over the test case), CHECK, REQUIRE,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS (exact text or doctest::Contains),
// CHECK_NOTHROW, FAIL, doctest::Approx
// (doctest's own comparison rule) and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN. The
// real doctest.h is not vendored in /root/reference; this stand-in lets
// oracle/Makefile compile those test sources UNMODIFIED, where they lie,
// against include/gpfilter/*.h + libgpfilter_b200.so (oracle/_ref/gpf_unit_b200)
// and against the reference library (oracle/_ref/gpf_unit_ref).
// Output: one "FAILED file:line: expression" line per failed assertion, one
// "[case] name: ok|FAILED" line per test case, and a summary line
//   "test cases: N | P passed | F failed; assertions: A | AF failed".
#ifndef ORACLE_SHIM_DOCTEST_H
#define ORACLE_SHIM_DOCTEST_H

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <type_traits>
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
  bool eq(double lhs) const {
    return std::fabs(lhs - value_) < eps_ * (scale_ + std::fmax(std::fabs(lhs), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
  double scale_ = 1.0;
};
inline bool operator==(double l, const Approx& r) { return r.eq(l); }
inline bool operator==(const Approx& l, double r) { return l.eq(r); }
inline bool operator!=(double l, const Approx& r) { return !r.eq(l); }
inline bool operator!=(const Approx& l, double r) { return !l.eq(r); }
inline bool operator<=(double l, const Approx& r) { return l < r.value() || r.eq(l); }
inline bool operator>=(double l, const Approx& r) { return l > r.value() || r.eq(l); }
inline bool operator<(double l, const Approx& r) { return l < r.value() && !r.eq(l); }
inline bool operator>(double l, const Approx& r) { return l > r.value() && !r.eq(l); }

// CHECK_THROWS_WITH_AS(expr, doctest::Contains("text"), type): substring match
struct Contains {
  std::string text;
  explicit Contains(const char* t) : text(t) {}
};

namespace detail {

inline bool message_matches(const char* what, const char* expected) { return std::strcmp(what, expected) == 0; }
inline bool message_matches(const char* what, const Contains& c) {
  return std::string(what).find(c.text) != std::string::npos;
}

struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& cases() {
  static std::vector<Case> v;
  return v;
}
struct Registrar {
  Registrar(const char* name, void (*fn)()) { cases().push_back({name, fn}); }
};

struct AbortCase {};  // REQUIRE / FAIL

struct State {
  long long assertions = 0, failed_assertions = 0;
  bool case_failed = false;
  // subcases of the running test case
  std::set<std::string> done;      // paths fully executed
  std::vector<std::string> stack;  // path being executed
  std::vector<bool> ran_at_depth;  // a subcase at this depth was entered in this pass
  int pending = 0;                 // subcases skipped in this pass that still have to run
};
inline State& state() {
  static State s;
  return s;
}

inline void report(bool ok, const char* file, int line, const char* what) {
  State& s = state();
  ++s.assertions;
  if (ok) return;
  ++s.failed_assertions;
  s.case_failed = true;
  std::printf("FAILED %s:%d: %s\n", file, line, what);
}

struct Subcase {
  bool entered = false;
  int pending_before = 0;
  explicit Subcase(const char* name) {
    State& s = state();
    const size_t depth = s.stack.size();
    std::string path;
    for (const auto& p : s.stack) path += p + "\x1f";
    path += name;
    if (s.done.count(path)) return;
    if (s.ran_at_depth.size() <= depth) s.ran_at_depth.resize(depth + 1, false);
    if (s.ran_at_depth[depth]) {  // a sibling ran in this pass: this one waits for the next
      ++s.pending;
      return;
    }
    s.ran_at_depth[depth] = true;
    s.stack.push_back(name);
    pending_before = s.pending;
    entered = true;
  }
  ~Subcase() {
    if (!entered) return;
    State& s = state();
    std::string path;
    for (size_t i = 0; i < s.stack.size(); ++i) path += (i ? "\x1f" : "") + s.stack[i];
    const size_t depth = s.stack.size();
    if (s.ran_at_depth.size() > depth) s.ran_at_depth.resize(depth);  // deeper levels start afresh
    s.stack.pop_back();
    if (s.pending == pending_before || std::uncaught_exceptions() > 0) s.done.insert(path);
  }
  explicit operator bool() const { return entered; }
};

inline int run_all() {
  State& s = state();
  int failed_cases = 0;
  for (const Case& c : cases()) {
    s.done.clear();
    bool failed = false;
    for (int pass = 0; pass < 10000; ++pass) {
      s.stack.clear();
      s.ran_at_depth.clear();
      s.pending = 0;
      s.case_failed = false;
      try {
        c.fn();
      } catch (const AbortCase&) {
        s.case_failed = true;
      } catch (const std::exception& e) {
        s.case_failed = true;
        std::printf("FAILED test case threw: %s\n", e.what());
      } catch (...) {
        s.case_failed = true;
        std::printf("FAILED test case threw an unknown exception\n");
      }
      failed = failed || s.case_failed;
      if (s.pending == 0) break;
    }
    std::printf("[case] %s: %s\n", c.name, failed ? "FAILED" : "ok");
    std::fflush(stdout);
    if (failed) ++failed_cases;
  }
  const int n = static_cast<int>(cases().size());
  std::printf("test cases: %d | %d passed | %d failed; assertions: %lld | %lld failed\n", n,
              n - failed_cases, failed_cases, s.assertions, s.failed_assertions);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)

#define DOCTEST_SHIM_TEST_CASE(fn, name)                                              \
  static void fn();                                                                   \
  static ::doctest::detail::Registrar DOCTEST_SHIM_CAT(fn, _reg)(name, &fn);          \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TEST_CASE(DOCTEST_SHIM_CAT(doctest_shim_case_, __COUNTER__), name)

#define SUBCASE(name) if (::doctest::detail::Subcase DOCTEST_SHIM_CAT(doctest_shim_sub_, __LINE__){name})

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK(" #__VA_ARGS__ ")")
#define REQUIRE(...)                                                                             \
  do {                                                                                           \
    const bool doctest_shim_ok = static_cast<bool>(__VA_ARGS__);                                 \
    ::doctest::detail::report(doctest_shim_ok, __FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")"); \
    if (!doctest_shim_ok) throw ::doctest::detail::AbortCase{};                                  \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                      \
  do {                                                                                                  \
    bool doctest_shim_ok = false;                                                                       \
    try {                                                                                               \
      static_cast<void>(expr);                                                                          \
    } catch (const std::remove_cv_t<std::remove_reference_t<__VA_ARGS__>>&) {                           \
      doctest_shim_ok = true;                                                                           \
    } catch (...) {                                                                                     \
    }                                                                                                   \
    ::doctest::detail::report(doctest_shim_ok, __FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")"); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, ...)                                                            \
  do {                                                                                                  \
    bool doctest_shim_ok = false;                                                                       \
    try {                                                                                               \
      static_cast<void>(expr);                                                                          \
    } catch (const std::remove_cv_t<std::remove_reference_t<__VA_ARGS__>>& doctest_shim_e) {            \
      doctest_shim_ok = ::doctest::detail::message_matches(doctest_shim_e.what(), msg);                 \
    } catch (...) {                                                                                     \
    }                                                                                                   \
    ::doctest::detail::report(doctest_shim_ok, __FILE__, __LINE__, "CHECK_THROWS_WITH_AS(" #expr ", " #msg ", " #__VA_ARGS__ ")"); \
  } while (0)
#define CHECK_NOTHROW(...)                                                                       \
  do {                                                                                           \
    bool doctest_shim_ok = true;                                                                 \
    try {                                                                                        \
      static_cast<void>(__VA_ARGS__);                                                            \
    } catch (...) {                                                                              \
      doctest_shim_ok = false;                                                                   \
    }                                                                                            \
    ::doctest::detail::report(doctest_shim_ok, __FILE__, __LINE__, "CHECK_NOTHROW(" #__VA_ARGS__ ")"); \
  } while (0)
#define FAIL(...)                                                                     \
  do {                                                                                \
    std::ostringstream doctest_shim_os;                                               \
    doctest_shim_os << "FAIL(" << __VA_ARGS__ << ")";                                 \
    ::doctest::detail::report(false, __FILE__, __LINE__, doctest_shim_os.str().c_str()); \
    throw ::doctest::detail::AbortCase{};                                             \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif

#endif  // ORACLE_SHIM_DOCTEST_H
