// Minimal doctest-compatible test harness (own code, NOT doctest).
//
// doctest is vendored-but-absent in the reference (proj/.gitignore:2), so
// this header provides just the macros the reference's unit tests use
// (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, REQUIRE_FALSE, CHECK_NOTHROW,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, CAPTURE, doctest::Approx,
// doctest::Contains) so those test sources compile unmodified against the
// C++ drop-in layer (oracle/dropin.mk).  Semantics follow doctest's
// documented behaviour: CHECK records a failure and continues, REQUIRE aborts
// the test case, Approx compares |a - b| < eps (scale + max(|a|, |b|)) with scale = 1 and
// eps = 100 * FLT_EPSILON by default.  Command line: -tc=<patterns> /
// -tce=<patterns> (comma-separated, '*' wildcards) select / exclude test
// cases by name; -s prints every test case name.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
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
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double x) const {
    return std::fabs(x - value_) < eps_ * (scale_ + std::fmax(std::fabs(x), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};
inline bool operator==(double x, const Approx& a) { return a.matches(x); }
inline bool operator==(const Approx& a, double x) { return a.matches(x); }
inline bool operator!=(double x, const Approx& a) { return !a.matches(x); }
inline bool operator!=(const Approx& a, double x) { return !a.matches(x); }

struct Contains {
  explicit Contains(const char* s) : text(s) {}
  std::string text;
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

struct Reg {
  Reg(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct State {
  int failed_asserts = 0;
  int asserts = 0;
  bool current_failed = false;
  const char* current = "";
};
inline State& state() {
  static State s;
  return s;
}

struct RequireAbort {};

inline void report(bool ok, const char* file, int line, const char* macro, const char* expr,
                   const std::string& extra = std::string()) {
  State& s = state();
  ++s.asserts;
  if (ok) return;
  ++s.failed_asserts;
  s.current_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s( %s )%s%s\n", file, line, s.current, macro, expr,
               extra.empty() ? "" : " -- ", extra.c_str());
}

inline bool message_matches(const std::string& what, const char* expected) {
  return what == expected;
}
inline bool message_matches(const std::string& what, const std::string& expected) {
  return what == expected;
}
inline bool message_matches(const std::string& what, const Contains& c) {
  return what.find(c.text) != std::string::npos;
}

inline bool wildcard(const char* pat, const char* str) {
  if (*pat == 0) return *str == 0;
  if (*pat == '*') return wildcard(pat + 1, str) || (*str && wildcard(pat, str + 1));
  return *str && (*pat == *str) && wildcard(pat + 1, str + 1);
}

inline bool any_match(const std::string& patterns, const char* name) {
  std::stringstream ss(patterns);
  std::string p;
  while (std::getline(ss, p, ','))
    if (!p.empty() && wildcard(p.c_str(), name)) return true;
  return false;
}

inline int run(int argc, char** argv) {
  std::string include, exclude;
  bool verbose = false;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    if (a.rfind("-tc=", 0) == 0) include = a.substr(4);
    else if (a.rfind("--test-case=", 0) == 0) include = a.substr(12);
    else if (a.rfind("-tce=", 0) == 0) exclude = a.substr(5);
    else if (a.rfind("--test-case-exclude=", 0) == 0) exclude = a.substr(20);
    else if (a == "-s" || a == "--success") verbose = true;
  }
  int run_n = 0, failed_n = 0, skipped = 0;
  for (const TestCase& tc : registry()) {
    if ((!include.empty() && !any_match(include, tc.name)) ||
        (!exclude.empty() && any_match(exclude, tc.name))) {
      ++skipped;
      continue;
    }
    State& s = state();
    s.current = tc.name;
    s.current_failed = false;
    ++run_n;
    try {
      tc.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& ex) {
      report(false, tc.file, tc.line, "TEST_CASE", tc.name,
             std::string("unexpected exception: ") + ex.what());
    } catch (...) {
      report(false, tc.file, tc.line, "TEST_CASE", tc.name, "unexpected exception");
    }
    if (s.current_failed) ++failed_n;
    if (verbose || s.current_failed)
      std::printf("[doctest] %s: %s\n", s.current_failed ? "FAILED" : "passed", tc.name);
  }
  const State& s = state();
  std::printf("[doctest] test cases: %d | %d passed | %d failed | %d skipped\n", run_n,
              run_n - failed_n, failed_n, skipped);
  std::printf("[doctest] assertions: %d | %d passed | %d failed |\n", s.asserts,
              s.asserts - s.failed_asserts, s.failed_asserts);
  std::printf("[doctest] Status: %s!\n", failed_n ? "FAILURE" : "SUCCESS");
  return failed_n ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_I(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_I(a, b)
#define DOCTEST_TC_I(name, fn)                                                         \
  static void fn();                                                                    \
  static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn);   \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_I(name, DOCTEST_CAT(doctest_tc_, __COUNTER__))

#define DOCTEST_ASSERT_I(macro, ok, text, abort)                                     \
  do {                                                                               \
    const bool doctest_ok_ = (ok);                                                   \
    ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, macro, text);         \
    if (!doctest_ok_ && (abort)) throw ::doctest::detail::RequireAbort();            \
  } while (0)

#define CHECK(...) DOCTEST_ASSERT_I("CHECK", static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, false)
#define CHECK_FALSE(...) DOCTEST_ASSERT_I("CHECK_FALSE", !(__VA_ARGS__), #__VA_ARGS__, false)
#define REQUIRE(...) DOCTEST_ASSERT_I("REQUIRE", static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, true)
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_I("REQUIRE_FALSE", !(__VA_ARGS__), #__VA_ARGS__, true)

#define CHECK_NOTHROW(...)                                                                  \
  do {                                                                                      \
    bool doctest_ok_ = true;                                                                \
    std::string doctest_msg_;                                                               \
    try {                                                                                   \
      (void)(__VA_ARGS__);                                                                  \
    } catch (const std::exception& doctest_ex_) {                                           \
      doctest_ok_ = false;                                                                  \
      doctest_msg_ = doctest_ex_.what();                                                    \
    } catch (...) {                                                                         \
      doctest_ok_ = false;                                                                  \
    }                                                                                       \
    ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "CHECK_NOTHROW", #__VA_ARGS__, \
                              doctest_msg_);                                                \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                          \
  do {                                                                                      \
    bool doctest_ok_ = false;                                                               \
    std::string doctest_msg_ = "no exception";                                              \
    try {                                                                                   \
      (void)(expr);                                                                         \
    } catch (const __VA_ARGS__&) {                                                          \
      doctest_ok_ = true;                                                                   \
    } catch (const std::exception& doctest_ex_) {                                           \
      doctest_msg_ = std::string("wrong exception type: ") + doctest_ex_.what();            \
    } catch (...) {                                                                         \
      doctest_msg_ = "wrong exception type";                                                \
    }                                                                                       \
    ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_AS", #expr,     \
                              doctest_ok_ ? std::string() : doctest_msg_);                  \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                \
  do {                                                                                       \
    bool doctest_ok_ = false;                                                                \
    std::string doctest_msg_ = "no exception";                                               \
    try {                                                                                    \
      (void)(expr);                                                                          \
    } catch (const __VA_ARGS__& doctest_ex_) {                                               \
      doctest_ok_ = ::doctest::detail::message_matches(doctest_ex_.what(), with);            \
      doctest_msg_ = std::string("message: ") + doctest_ex_.what();                          \
    } catch (const std::exception& doctest_ex_) {                                            \
      doctest_msg_ = std::string("wrong exception type: ") + doctest_ex_.what();             \
    } catch (...) {                                                                          \
      doctest_msg_ = "wrong exception type";                                                 \
    }                                                                                        \
    ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_WITH_AS", #expr, \
                              doctest_ok_ ? std::string() : doctest_msg_);                   \
  } while (0)

#define CAPTURE(...) (void)(__VA_ARGS__)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
