// doctest.h — minimal from-scratch stand-in for the subset of the doctest
// testing framework the reference's own test files use (TEST INFRASTRUCTURE:
// doctest is vendored-but-absent in /root/reference).  It lets
// the UNMODIFIED /root/reference/proj/tests/*.cpp compile and run here, against
// the literal reference build and against the B200 library (tests/cpp/refsuite).
//
// Supported: TEST_CASE, SUBCASE (doctest semantics: the test case is re-run
// once per leaf subcase path, code outside subcases runs every time), CHECK,
// REQUIRE, FAIL, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, doctest::Approx
// (.epsilon), doctest::Contains, DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
// The runner prints one line per failed assertion and a summary; the exit code
// is the number of failed test cases (capped at 255).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <set>
#include <sstream>
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
  friend bool operator==(double a, const Approx& b) { return b.eq(a); }
  friend bool operator==(const Approx& b, double a) { return b.eq(a); }
  friend bool operator!=(double a, const Approx& b) { return !b.eq(a); }
  friend bool operator!=(const Approx& b, double a) { return !b.eq(a); }
  friend bool operator<=(double a, const Approx& b) { return a < b.v_ || b.eq(a); }
  friend bool operator>=(double a, const Approx& b) { return a > b.v_ || b.eq(a); }
  double value() const { return v_; }

 private:
  bool eq(double a) const {
    // doctest: |a - v| < eps * (scale + max(|a|, |v|)), scale = 1
    return std::fabs(a - v_) < eps_ * (1.0 + std::fmax(std::fabs(a), std::fabs(v_)));
  }
  double v_;
  double eps_ = 1.19209290e-07 * 100;  // float epsilon * 100, doctest's default
};

class Contains {
 public:
  explicit Contains(const char* s) : s_(s) {}
  bool matches(const std::string& what) const { return what.find(s_) != std::string::npos; }
  const std::string& str() const { return s_; }

 private:
  std::string s_;
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

// Subcase bookkeeping: a path is the sequence of (file:line) of the subcases
// entered.  In one run, at most one not-yet-finished subcase is entered per
// nesting level; a subcase is finished once it ran without skipping a child.
struct State {
  std::set<std::string> done;
  std::vector<std::string> stack;         // entered subcases of this run
  std::vector<bool> entered_at_depth;     // a sibling at this depth was entered this run
  std::vector<bool> child_skipped;        // per stack level: a child was skipped this run
  bool skipped_any = false;
  int failed_asserts = 0;
  int passed_asserts = 0;
  const char* current = "";
};
inline State& st() {
  static State s;
  return s;
}

struct RequireFailed {};

inline std::string path_key() {
  std::string k;
  for (const auto& p : st().stack) k += p + "/";
  return k;
}

class Subcase {
 public:
  Subcase(const char* name, const char* file, int line) {
    State& s = st();
    const size_t depth = s.stack.size();
    if (s.entered_at_depth.size() <= depth) s.entered_at_depth.resize(depth + 1, false);
    key_ = path_key() + std::string(file) + ":" + std::to_string(line) + ":" + name;
    if (s.done.count(key_)) return;
    if (s.entered_at_depth[depth]) {  // a sibling ran this time: come back later
      s.skipped_any = true;
      if (!s.child_skipped.empty()) s.child_skipped.back() = true;
      return;
    }
    s.entered_at_depth[depth] = true;
    s.stack.push_back(std::string(file) + ":" + std::to_string(line) + ":" + name);
    s.child_skipped.push_back(false);
    if (s.entered_at_depth.size() <= depth + 1) s.entered_at_depth.resize(depth + 2, false);
    s.entered_at_depth[depth + 1] = false;
    entered_ = true;
  }
  ~Subcase() {
    if (!entered_) return;
    State& s = st();
    const bool skipped_child = s.child_skipped.back();
    s.child_skipped.pop_back();
    s.stack.pop_back();
    if (!skipped_child) s.done.insert(key_);
    else if (!s.child_skipped.empty()) s.child_skipped.back() = true;
  }
  explicit operator bool() const { return entered_; }

 private:
  std::string key_;
  bool entered_ = false;
};

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  State& s = st();
  if (ok) {
    ++s.passed_asserts;
    return;
  }
  ++s.failed_asserts;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s ) in TEST_CASE \"%s\"\n", file, line,
               require ? "REQUIRE" : "CHECK", expr, s.current);
  if (require) throw RequireFailed{};
}

template <typename F>
bool throws_with(F&& f, const std::string& expect, bool substring) {
  try {
    f();
  } catch (const std::exception& e) {
    return substring ? std::string(e.what()).find(expect) != std::string::npos
                     : expect == e.what();
  } catch (...) {
  }
  return false;
}

inline int run_all() {
  int failed_cases = 0, cases = 0;
  for (const TestCase& tc : registry()) {
    ++cases;
    State& s = st();
    s = State{};
    s.current = tc.name;
    bool case_failed = false;
    for (int run = 0; run < 100000; ++run) {
      s.stack.clear();
      s.entered_at_depth.assign(1, false);
      s.child_skipped.clear();
      s.skipped_any = false;
      const int before = s.failed_asserts;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        std::fprintf(stderr, "%s:%d: TEST_CASE \"%s\" threw: %s\n", tc.file, tc.line, tc.name,
                     e.what());
        ++s.failed_asserts;
      }
      if (s.failed_asserts > before) case_failed = true;
      if (!s.skipped_any) break;
    }
    if (case_failed) ++failed_cases;
    std::printf("[%s] %s (%d assertions)\n", case_failed ? "FAIL" : " ok ", tc.name,
                s.passed_asserts + s.failed_asserts);
  }
  std::printf("test cases: %d | %d passed | %d failed\n", cases, cases - failed_cases,
              failed_cases);
  return failed_cases > 255 ? 255 : failed_cases;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                        \
  static void fn();                                                                  \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, \
                                                           &fn);                     \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name)                                                                  \
  if (const ::doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name, __FILE__, \
                                                                          __LINE__})
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, \
                                             __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, \
                                               __FILE__, __LINE__, true)
#define FAIL(msg)                                                                  \
  do {                                                                             \
    std::ostringstream doctest_os_;                                                \
    doctest_os_ << msg;                                                            \
    ::doctest::detail::report(false, doctest_os_.str().c_str(), __FILE__, __LINE__, true); \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                   \
  do {                                                                                \
    bool doctest_ok_ = false;                                                         \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (const type&) {                                                           \
      doctest_ok_ = true;                                                             \
    } catch (...) {                                                                   \
    }                                                                                 \
    ::doctest::detail::report(doctest_ok_, #expr " throws " #type, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, type)                                        \
  do {                                                                                \
    bool doctest_ok_ = false;                                                         \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (const type& e) {                                                         \
      doctest_ok_ = ::doctest::detail::matches_with(e.what(), with);                  \
    } catch (...) {                                                                   \
    }                                                                                 \
    ::doctest::detail::report(doctest_ok_, #expr " throws " #type " with " #with, __FILE__, \
                              __LINE__, false);                                       \
  } while (0)

namespace doctest {
namespace detail {
inline bool matches_with(const char* what, const char* s) { return std::string(what) == s; }
inline bool matches_with(const char* what, const std::string& s) { return s == what; }
inline bool matches_with(const char* what, const Contains& c) { return c.matches(what); }
}  // namespace detail
}  // namespace doctest

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
