// TEST INFRASTRUCTURE ONLY -- a minimal stand-in for the doctest single-header framework,
// which the reference's unit tests include (proj/tests/*.cpp, `#include <doctest.h>`) but
// does not vendor (proj/README.md:29).  Implements exactly the subset those tests use:
// TEST_CASE, one level of SUBCASE (each subcase runs in a fresh pass of its test case, as
// doctest does), CHECK / CHECK_FALSE / CHECK_MESSAGE / CHECK_NOTHROW / CHECK_THROWS_AS /
// CHECK_THROWS_WITH_AS, REQUIRE, FAIL, doctest::Approx (default epsilon
// float_eps * 100, doctest's rule) and doctest::Contains.  Written for this repo.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) <
           b.eps_ * (b.scale_ + std::max(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  friend bool operator!=(const Approx& b, double a) { return !(a == b); }

 private:
  double v_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double scale_ = 1.0;
};

struct Contains {
  std::string s;
  explicit Contains(const char* x) : s(x) {}
  explicit Contains(std::string x) : s(std::move(x)) {}
};
inline bool msg_matches(const std::string& what, const char* want) { return what == want; }
inline bool msg_matches(const std::string& what, const std::string& want) { return what == want; }
inline bool msg_matches(const std::string& what, const Contains& c) {
  return what.find(c.s) != std::string::npos;
}

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
struct Reg {
  Reg(const char* n, void (*f)(), const char* file, int line) {
    registry().push_back({n, f, file, line});
  }
};
struct State {
  long checks = 0, failures = 0;
  const char* test = "";
  // subcases: the set of (file:line) already run, and whether this pass entered one
  std::set<std::string> done;
  bool entered = false, pending = false;
};
inline State& st() {
  static State s;
  return s;
}
struct RequireAbort {};
inline void fail(const char* file, int line, const std::string& what) {
  ++st().failures;
  std::fprintf(stderr, "%s:%d: FAILED in TEST_CASE(\"%s\"): %s\n", file, line, st().test,
               what.c_str());
}
inline void check(bool ok, const char* file, int line, const char* expr, bool require) {
  ++st().checks;
  if (ok) return;
  fail(file, line, expr);
  if (require) throw RequireAbort{};
}
struct Subcase {
  bool run = false;
  Subcase(const char* file, int line) {
    const std::string key = std::string(file) + ":" + std::to_string(line);
    State& s = st();
    if (s.entered || s.done.count(key)) {
      if (!s.done.count(key)) s.pending = true;
      return;
    }
    s.done.insert(key);
    s.entered = true;
    run = true;
  }
  explicit operator bool() const { return run; }
};
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                   \
  static void fn();                                                                 \
  static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) \
  if (::doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){__FILE__, __LINE__})

#define DOCTEST_CHECK_IMPL(cond, text, req) \
  ::doctest::detail::check(static_cast<bool>(cond), __FILE__, __LINE__, text, req)
#define CHECK(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), #__VA_ARGS__, false)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", false)
#define CHECK_MESSAGE(cond, msg) DOCTEST_CHECK_IMPL((cond), #cond, false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), #__VA_ARGS__, true)
#define FAIL(msg)                                                         \
  do {                                                                    \
    std::ostringstream doctest_os_;                                       \
    doctest_os_ << msg;                                                   \
    ::doctest::detail::fail(__FILE__, __LINE__, "FAIL: " + doctest_os_.str()); \
    throw ::doctest::detail::RequireAbort{};                              \
  } while (0)
#define CHECK_NOTHROW(...)                                                        \
  do {                                                                            \
    bool doctest_ok_ = true;                                                      \
    try { (void)(__VA_ARGS__); } catch (...) { doctest_ok_ = false; }             \
    DOCTEST_CHECK_IMPL(doctest_ok_, "nothrow: " #__VA_ARGS__, false);             \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                \
  do {                                                                            \
    bool doctest_ok_ = false;                                                     \
    try { (void)(expr); } catch (const __VA_ARGS__&) { doctest_ok_ = true; } catch (...) {} \
    DOCTEST_CHECK_IMPL(doctest_ok_, "throws " #__VA_ARGS__ ": " #expr, false);    \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                     \
  do {                                                                            \
    bool doctest_ok_ = false;                                                     \
    std::string doctest_what_ = "<no exception>";                                 \
    try { (void)(expr); } catch (const __VA_ARGS__& e_) {                         \
      doctest_what_ = e_.what();                                                  \
      doctest_ok_ = ::doctest::msg_matches(doctest_what_, with);                  \
    } catch (...) { doctest_what_ = "<other exception type>"; }                   \
    DOCTEST_CHECK_IMPL(doctest_ok_, ("throws with: " #expr " -> " + doctest_what_).c_str(), false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  using namespace doctest::detail;
  int failed_cases = 0, n = 0;
  for (const TestCase& tc : registry()) {
    State& s = st();
    s.test = tc.name;
    s.done.clear();
    const long before = s.failures;
    do {  // one pass per subcase (plus the first)
      s.entered = s.pending = false;
      try {
        tc.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        fail(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
      } catch (...) {
        fail(tc.file, tc.line, "unexpected exception");
      }
    } while (s.pending);
    ++n;
    if (s.failures != before) ++failed_cases;
  }
  std::printf("[doctest-lite] test cases: %d | %d passed | %d failed; assertions: %ld | %ld failed\n",
              n, n - failed_cases, failed_cases, st().checks, st().failures);
  return failed_cases ? 1 : 0;
}
#endif
