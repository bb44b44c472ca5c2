// doctest.h -- TEST INFRASTRUCTURE: a minimal stand-in for the doctest
// framework (absent from this image), so that the
// reference's OWN unit-test sources (/root/reference/proj/tests/test_*.cpp)
// compile unchanged against this repo's drop-in headers (include/swe/*.hpp)
// and run on the B200 path.  It implements the subset those files use:
// TEST_SUITE, TEST_CASE, SUBCASE (re-run per leaf, as doctest), CHECK,
// REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, FAIL, doctest::Approx,
// doctest::Contains, and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.  Written from
// doctest's documented semantics; no doctest source is used.
//
// Command line of the built binary: [-tc=<substring>] [-ts=<substring>]
// [-tce=<substring>] (filters on test-case / suite names); exit code 0 iff
// every executed check passed.  Prints one "[doctest] ..." summary line.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

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
  bool matches(double lhs) const {
    // doctest: |lhs - rhs| < eps * (scale + max(|lhs|, |rhs|))
    return std::fabs(lhs - value_) <
           eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;  // doctest default
};
inline bool operator==(double l, const Approx& r) { return r.matches(l); }
inline bool operator==(const Approx& l, double r) { return l.matches(r); }
inline bool operator!=(double l, const Approx& r) { return !r.matches(l); }
inline bool operator!=(const Approx& l, double r) { return !l.matches(r); }
inline bool operator<=(double l, const Approx& r) { return l < r.value() || r.matches(l); }
inline bool operator>=(double l, const Approx& r) { return l > r.value() || r.matches(l); }

struct Contains {
  explicit Contains(const char* s) : s(s) {}
  std::string s;
  bool check(const std::string& what) const { return what.find(s) != std::string::npos; }
};

namespace detail {

struct TestCase {
  const char* name;
  const char* suite;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct State {
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
  // SUBCASE traversal (one leaf path per run of the test case)
  std::set<std::string> done;
  std::vector<std::string> stack;
  std::vector<char> pending_child;  // per level of the stack
  std::vector<char> entered;        // a subcase at this depth ran in this run
  bool pending = false;
  const char* current = "";
};
inline State& st() {
  static State s;
  return s;
}

struct Abort {};  // REQUIRE / FAIL: leave the test case

inline void report(bool ok, const char* file, int line, const std::string& what) {
  State& s = st();
  ++s.checks;
  if (ok) return;
  ++s.failed_checks;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, s.current, what.c_str());
}

struct Reg {
  Reg(const char* name, const char* suite, const char* file, int line, void (*fn)()) {
    registry().push_back({name, suite, file, line, fn});
  }
};

class Subcase {
 public:
  Subcase(const char* name, const char* file, int line) {
    State& s = st();
    const size_t depth = s.stack.size();
    key_ = (depth ? s.stack.back() : std::string()) + "/" + file + ":" + std::to_string(line) + ":" +
           name;
    if (s.entered.size() <= depth) s.entered.resize(depth + 1, 0);
    const bool done = s.done.count(key_) > 0;
    if (done) return;
    if (s.entered[depth]) {  // a sibling ran in this run: come back later
      s.pending = true;
      for (auto& p : s.pending_child) p = 1;
      return;
    }
    entered_ = true;
    s.entered[depth] = 1;
    if (s.entered.size() <= depth + 1) s.entered.resize(depth + 2, 0);
    s.entered[depth + 1] = 0;
    s.stack.push_back(key_);
    s.pending_child.push_back(0);
  }
  ~Subcase() {
    if (!entered_) return;
    State& s = st();
    const bool child_left = s.pending_child.back() != 0;
    s.stack.pop_back();
    s.pending_child.pop_back();
    if (!child_left) s.done.insert(key_);
  }
  Subcase(const Subcase&) = delete;
  explicit operator bool() const { return entered_; }

 private:
  std::string key_;
  bool entered_ = false;
};

inline bool filter_ok(const std::string& v, const std::vector<std::string>& inc,
                      const std::vector<std::string>& exc) {
  for (const auto& e : exc)
    if (v.find(e) != std::string::npos) return false;
  if (inc.empty()) return true;
  for (const auto& i : inc)
    if (v.find(i) != std::string::npos) return true;
  return false;
}

inline int run_all(int argc, char** argv) {
  std::vector<std::string> tc, ts, tce;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    if (a.rfind("-tc=", 0) == 0) tc.push_back(a.substr(4));
    else if (a.rfind("-ts=", 0) == 0) ts.push_back(a.substr(4));
    else if (a.rfind("-tce=", 0) == 0) tce.push_back(a.substr(5));
  }
  State& s = st();
  int cases = 0, failed_cases = 0;
  for (const TestCase& t : registry()) {
    if (!filter_ok(t.name, tc, tce) || !filter_ok(t.suite, ts, {})) continue;
    ++cases;
    s.case_failed = false;
    s.done.clear();
    s.current = t.name;
    int runs = 0;
    do {
      s.pending = false;
      s.stack.clear();
      s.pending_child.clear();
      s.entered.assign(1, 0);
      ++runs;
      try {
        t.fn();
      } catch (const Abort&) {
        s.stack.clear();
        s.pending_child.clear();
      } catch (const std::exception& e) {
        report(false, t.file, t.line, std::string("unexpected exception: ") + e.what());
      } catch (...) {
        report(false, t.file, t.line, "unexpected unknown exception");
      }
    } while (s.pending && runs < 1000);
    if (s.case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "[doctest] test case FAILED: %s (%s:%d)\n", t.name, t.file, t.line);
    }
  }
  std::printf("[doctest] test cases: %d | %d passed | %d failed | assertions: %ld | %ld passed | "
              "%ld failed\n",
              cases, cases - failed_cases, failed_cases, s.checks, s.checks - s.failed_checks,
              s.failed_checks);
  return failed_cases == 0 && s.failed_checks == 0 ? 0 : 1;
}

inline bool matches(const std::string& what, const Contains& c) { return c.check(what); }
inline bool matches(const std::string& what, const char* exact) { return what == exact; }
inline bool matches(const std::string& what, const std::string& exact) { return what == exact; }

}  // namespace detail
}  // namespace doctest

namespace { [[maybe_unused]] constexpr const char* doctest_suite_name_ = ""; }

#define DOCTEST_TEST_SUITE_IMPL_(ns, name)                                  \
  namespace ns {                                                           \
  [[maybe_unused]] constexpr const char* doctest_suite_name_ = name;       \
  }                                                                        \
  namespace ns
#define TEST_SUITE(name) DOCTEST_TEST_SUITE_IMPL_(DOCTEST_CAT(doctest_suite_, __COUNTER__), name)

#define DOCTEST_TEST_CASE_IMPL_(fn, reg, name)                                         \
  static void fn();                                                                     \
  static ::doctest::detail::Reg reg(name, doctest_suite_name_, __FILE__, __LINE__, &fn); \
  static void fn()

#define TEST_CASE(name)                                                                 \
  DOCTEST_TEST_CASE_IMPL_(DOCTEST_CAT(doctest_tc_, __COUNTER__),                        \
                          DOCTEST_CAT(doctest_reg_, __COUNTER__), name)

#define SUBCASE(name)                                                               \
  if (const ::doctest::detail::Subcase& DOCTEST_CAT(doctest_sc_, __COUNTER__) =    \
          ::doctest::detail::Subcase(name, __FILE__, __LINE__))

#define CHECK(...)                                                                       \
  do {                                                                                   \
    bool doctest_ok_ = false;                                                            \
    try {                                                                                \
      doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                      \
    } catch (const std::exception& e) {                                                  \
      ::doctest::detail::report(false, __FILE__, __LINE__,                               \
                                std::string("CHECK(" #__VA_ARGS__ ") threw ") + e.what()); \
      break;                                                                             \
    }                                                                                    \
    ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "CHECK(" #__VA_ARGS__ ")"); \
  } while (0)

#define REQUIRE(...)                                                                        \
  do {                                                                                      \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                \
    ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")"); \
    if (!doctest_ok_) throw ::doctest::detail::Abort{};                                     \
  } while (0)

#define FAIL(msg)                                                                          \
  do {                                                                                     \
    std::ostringstream doctest_os_;                                                        \
    doctest_os_ << msg;                                                                    \
    ::doctest::detail::report(false, __FILE__, __LINE__, "FAIL: " + doctest_os_.str());    \
    throw ::doctest::detail::Abort{};                                                      \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                          \
  do {                                                                                      \
    bool doctest_ok_ = false;                                                               \
    std::string doctest_msg_ = "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ") did not throw"; \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
    } catch (const __VA_ARGS__&) {                                                          \
      doctest_ok_ = true;                                                                   \
    } catch (const std::exception& e) {                                                     \
      doctest_msg_ = std::string("CHECK_THROWS_AS(" #expr ") threw another type: ") + e.what(); \
    } catch (...) {                                                                         \
      doctest_msg_ = "CHECK_THROWS_AS(" #expr ") threw another type";                       \
    }                                                                                       \
    ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, doctest_msg_);               \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                  \
  do {                                                                                         \
    bool doctest_ok_ = false;                                                                  \
    std::string doctest_msg_ = "CHECK_THROWS_WITH_AS(" #expr ") did not throw";                \
    try {                                                                                      \
      static_cast<void>(expr);                                                                 \
    } catch (const __VA_ARGS__& e) {                                                           \
      doctest_ok_ = ::doctest::detail::matches(e.what(), with);                                \
      if (!doctest_ok_)                                                                        \
        doctest_msg_ = std::string("CHECK_THROWS_WITH_AS(" #expr "): message \"") + e.what() + \
                       "\" does not match " #with;                                              \
    } catch (const std::exception& e) {                                                        \
      doctest_msg_ = std::string("CHECK_THROWS_WITH_AS(" #expr ") threw another type: ") +    \
                     e.what();                                                                 \
    } catch (...) {                                                                            \
      doctest_msg_ = "CHECK_THROWS_WITH_AS(" #expr ") threw another type";                     \
    }                                                                                          \
    ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, doctest_msg_);                  \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run_all(argc, argv); }
#endif
