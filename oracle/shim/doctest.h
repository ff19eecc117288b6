// TEST INFRASTRUCTURE ONLY — a small stand-in for the doctest single header
// (the reference vendors doctest under proj/vendor/, which is absent here,
// SURVEY §0.5). It lets the reference's own unit suites
// (/root/reference/proj/tests/test_*.cpp) compile unmodified and run as the
// gate that pins oracle/_ref. Semantics kept from doctest: one TEST_CASE body
// is re-run once per SUBCASE (one nesting level, which is all those suites
// use); CHECK* records and continues; REQUIRE* aborts the test case;
// Approx compares |a-b| < eps * (1 + max(|a|, |b|)).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <set>
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
    return std::fabs(x - value_) <
           eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
  }

 private:
  double value_;
  double eps_ = 1.1920928955078125e-07 * 100;
  double scale_ = 1.0;
};
inline bool operator==(double x, const Approx& a) { return a.matches(x); }
inline bool operator==(const Approx& a, double x) { return a.matches(x); }
inline bool operator!=(double x, const Approx& a) { return !a.matches(x); }
inline bool operator!=(const Approx& a, double x) { return !a.matches(x); }

struct Contains {
  explicit Contains(std::string s) : needle(std::move(s)) {}
  bool check(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
  std::string needle;
};

namespace shim {

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

struct Stats {
  long checks = 0;
  long failed_checks = 0;
  int failed_cases = 0;
  bool current_failed = false;
};
inline Stats& stats() {
  static Stats s;
  return s;
}

struct SubcaseState {
  std::set<int> done;
  int entered = -1;
  bool pending = false;
};
inline SubcaseState*& subcase_state() {
  static SubcaseState* s = nullptr;
  return s;
}

struct RequireFailure {};

inline void record(bool ok, const char* what, const char* file, int line) {
  Stats& s = stats();
  ++s.checks;
  if (!ok) {
    ++s.failed_checks;
    s.current_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
  }
}

struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};

class Subcase {
 public:
  Subcase(const char* /*name*/, int line) : line_(line) {
    SubcaseState* st = subcase_state();
    if (st->done.count(line) == 0) {
      if (st->entered == -1) {
        st->entered = line;
        active_ = true;
      } else {
        st->pending = true;
      }
    }
  }
  ~Subcase() {
    if (active_) subcase_state()->done.insert(line_);
  }
  explicit operator bool() const { return active_; }

 private:
  int line_;
  bool active_ = false;
};

inline int run_all() {
  for (const TestCase& tc : registry()) {
    SubcaseState st;
    subcase_state() = &st;
    stats().current_failed = false;
    do {
      st.entered = -1;
      st.pending = false;
      try {
        tc.fn();
      } catch (const RequireFailure&) {
      } catch (const std::exception& e) {
        record(false, e.what(), tc.file, tc.line);
      }
    } while (st.pending);
    if (stats().current_failed) {
      ++stats().failed_cases;
      std::fprintf(stderr, "  in TEST_CASE \"%s\"\n", tc.name);
    }
  }
  const Stats& s = stats();
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n",
              registry().size(), registry().size() - s.failed_cases, s.failed_cases);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", s.checks,
              s.checks - s.failed_checks, s.failed_checks);
  std::printf("[doctest-shim] Status: %s\n", s.failed_cases ? "FAILURE!" : "SUCCESS!");
  return s.failed_cases;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)

#define DOCTEST_SHIM_TEST_CASE(name, fn)                                              \
  static void fn();                                                                   \
  static ::doctest::shim::Registrar DOCTEST_SHIM_CAT(fn, _reg)(name, &fn, __FILE__, \
                                                               __LINE__);             \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TEST_CASE(name, DOCTEST_SHIM_CAT(doctest_shim_tc_, __COUNTER__))

#define SUBCASE(name) \
  if (const ::doctest::shim::Subcase DOCTEST_SHIM_CAT(doctest_shim_sc_, __LINE__){name, __LINE__})

#define CHECK(...) ::doctest::shim::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::shim::record(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define CHECK_EQ(a, b) ::doctest::shim::record((a) == (b), #a " == " #b, __FILE__, __LINE__)
#define CHECK_NE(a, b) ::doctest::shim::record((a) != (b), #a " != " #b, __FILE__, __LINE__)
#define CHECK_LT(a, b) ::doctest::shim::record((a) < (b), #a " < " #b, __FILE__, __LINE__)
#define CHECK_LE(a, b) ::doctest::shim::record((a) <= (b), #a " <= " #b, __FILE__, __LINE__)
#define CHECK_GT(a, b) ::doctest::shim::record((a) > (b), #a " > " #b, __FILE__, __LINE__)
#define CHECK_GE(a, b) ::doctest::shim::record((a) >= (b), #a " >= " #b, __FILE__, __LINE__)
#define CHECK_UNARY(...) CHECK(__VA_ARGS__)

#define DOCTEST_SHIM_REQUIRE_IMPL(ok, text)                                 \
  do {                                                                      \
    const bool doctest_shim_ok_ = (ok);                                     \
    ::doctest::shim::record(doctest_shim_ok_, text, __FILE__, __LINE__);    \
    if (!doctest_shim_ok_) throw ::doctest::shim::RequireFailure{};         \
  } while (0)
#define REQUIRE(...) DOCTEST_SHIM_REQUIRE_IMPL(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__)
#define REQUIRE_FALSE(...) DOCTEST_SHIM_REQUIRE_IMPL(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__)
#define REQUIRE_EQ(a, b) DOCTEST_SHIM_REQUIRE_IMPL((a) == (b), #a " == " #b)

#define CHECK_THROWS_AS(expr, type)                                          \
  do {                                                                       \
    bool doctest_shim_caught_ = false;                                       \
    try {                                                                    \
      static_cast<void>(expr);                                               \
    } catch (const type&) {                                                  \
      doctest_shim_caught_ = true;                                           \
    } catch (...) {                                                          \
    }                                                                        \
    ::doctest::shim::record(doctest_shim_caught_, "throws " #type ": " #expr, \
                            __FILE__, __LINE__);                             \
  } while (0)
#define CHECK_THROWS(expr)                                                   \
  do {                                                                       \
    bool doctest_shim_caught_ = false;                                       \
    try {                                                                    \
      static_cast<void>(expr);                                               \
    } catch (...) {                                                          \
      doctest_shim_caught_ = true;                                           \
    }                                                                        \
    ::doctest::shim::record(doctest_shim_caught_, "throws: " #expr, __FILE__, \
                            __LINE__);                                       \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, type)                             \
  do {                                                                        \
    bool doctest_shim_ok_ = false;                                            \
    try {                                                                     \
      static_cast<void>(expr);                                                \
    } catch (const type& e) {                                                 \
      doctest_shim_ok_ = ::doctest::Contains(matcher).check(e.what());        \
    } catch (...) {                                                           \
    }                                                                         \
    ::doctest::shim::record(doctest_shim_ok_, "throws " #type " with " #matcher \
                            ": " #expr, __FILE__, __LINE__);                  \
  } while (0)
#define CHECK_NOTHROW(expr)                                                  \
  do {                                                                       \
    bool doctest_shim_ok_ = true;                                            \
    try {                                                                    \
      static_cast<void>(expr);                                               \
    } catch (...) {                                                          \
      doctest_shim_ok_ = false;                                              \
    }                                                                        \
    ::doctest::shim::record(doctest_shim_ok_, "nothrow: " #expr, __FILE__,    \
                            __LINE__);                                       \
  } while (0)

#if defined(DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN)
int main() { return ::doctest::shim::run_all(); }
#endif
