// doctest.h -- TEST INFRASTRUCTURE ONLY.
//
// The handful of doctest (https://github.com/doctest/doctest) macros the
// reference's tests use (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, FAIL, SUBCASE, doctest::Approx), restated so that
// proj/tests/*.cpp compile unchanged against oracle/ref_shim.  doctest is a
// git-ignored vendor dependency of the reference (proj/.gitignore), absent
// here.  Semantics kept: a failed CHECK records the failure and continues, a
// failed REQUIRE / FAIL ends the test case; an exception escaping a test case
// fails it; Approx compares |a - b| < eps * (scale + max(|a|, |b|)) with the
// default eps = 100 * float epsilon and scale 1.  The main() (defined where
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN is set) runs every registered case (or
// those whose name contains the -tc= filter) and prints one summary line.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
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
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool eq(double a) const {
    return std::fabs(a - v_) < eps_ * (scale_ + std::fmax(std::fabs(a), std::fabs(v_)));
  }
  friend bool operator==(double a, const Approx& b) { return b.eq(a); }
  friend bool operator==(const Approx& b, double a) { return b.eq(a); }
  friend bool operator!=(double a, const Approx& b) { return !b.eq(a); }
  friend bool operator!=(const Approx& b, double a) { return !b.eq(a); }
  friend bool operator<=(double a, const Approx& b) { return a < b.v_ || b.eq(a); }
  friend bool operator>=(double a, const Approx& b) { return a > b.v_ || b.eq(a); }

 private:
  double v_;
  double eps_ = 1.1920928955078125e-05;  // 100 * FLT_EPSILON
  double scale_ = 1.0;
};

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

struct Reg {
  Reg(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct Abort {};  // REQUIRE / FAIL: leave the current test case

inline int& failures() {
  static int n = 0;
  return n;
}
inline long long& assertions() {
  static long long n = 0;
  return n;
}

inline void fail(const char* file, int line, const std::string& what) {
  ++failures();
  std::printf("%s:%d: ERROR: %s\n", file, line, what.c_str());
}

inline void check(bool ok, const char* expr, const char* file, int line, bool require) {
  ++assertions();
  if (ok) return;
  fail(file, line, std::string(require ? "REQUIRE( " : "CHECK( ") + expr + " ) is NOT correct!");
  if (require) throw Abort{};
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)

#define TEST_CASE(name)                                                                 \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                     \
  static ::doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(                    \
      name, __FILE__, __LINE__, &DOCTEST_CAT(doctest_fn_, __LINE__));                   \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define DOCTEST_ASSERT_IMPL(expr, require)                                              \
  do {                                                                                  \
    bool doctest_ok_ = false;                                                           \
    try {                                                                               \
      doctest_ok_ = static_cast<bool>(expr);                                            \
    } catch (const std::exception& e) {                                                 \
      ::doctest::detail::fail(__FILE__, __LINE__,                                       \
                              std::string("exception in " #expr ": ") + e.what());      \
      if (require) throw ::doctest::detail::Abort{};                                    \
      break;                                                                            \
    }                                                                                   \
    ::doctest::detail::check(doctest_ok_, #expr, __FILE__, __LINE__, require);          \
  } while (0)

#define CHECK(...) DOCTEST_ASSERT_IMPL((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_ASSERT_IMPL((__VA_ARGS__), true)
#define CHECK_FALSE(...) DOCTEST_ASSERT_IMPL(!(__VA_ARGS__), false)
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_IMPL(!(__VA_ARGS__), true)

#define CHECK_THROWS_AS(expr, ...)                                                      \
  do {                                                                                  \
    ++::doctest::detail::assertions();                                                  \
    bool doctest_thrown_ = false;                                                       \
    try {                                                                               \
      static_cast<void>(expr);                                                          \
    } catch (const __VA_ARGS__&) {                                                      \
      doctest_thrown_ = true;                                                           \
    } catch (...) {                                                                     \
      ::doctest::detail::fail(__FILE__, __LINE__,                                       \
                              "CHECK_THROWS_AS( " #expr " ): wrong exception type");    \
      break;                                                                            \
    }                                                                                   \
    if (!doctest_thrown_)                                                               \
      ::doctest::detail::fail(__FILE__, __LINE__,                                       \
                              "CHECK_THROWS_AS( " #expr " ): did not throw");           \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, message, ...)                                        \
  do {                                                                                  \
    ++::doctest::detail::assertions();                                                  \
    bool doctest_ok_ = false;                                                           \
    try {                                                                               \
      static_cast<void>(expr);                                                          \
    } catch (const __VA_ARGS__& e) {                                                    \
      doctest_ok_ = std::string(e.what()) == std::string(message);                      \
    } catch (...) {                                                                     \
    }                                                                                   \
    if (!doctest_ok_)                                                                   \
      ::doctest::detail::fail(__FILE__, __LINE__,                                       \
                              "CHECK_THROWS_WITH_AS( " #expr " ) failed");              \
  } while (0)

#define FAIL(msg)                                                                       \
  do {                                                                                  \
    ::doctest::detail::fail(__FILE__, __LINE__, std::string("FAIL: ") + (msg));         \
    throw ::doctest::detail::Abort{};                                                   \
  } while (0)

// The reference's tests use at most one SUBCASE per test case, which runs
// exactly once with the enclosing code.
#define SUBCASE(name) if (true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  const char* filter = nullptr;
  for (int i = 1; i < argc; ++i)
    if (std::strncmp(argv[i], "-tc=", 4) == 0) filter = argv[i] + 4;
  int run = 0, failed_cases = 0;
  for (const auto& c : ::doctest::detail::registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    ++run;
    const int before = ::doctest::detail::failures();
    try {
      c.fn();
    } catch (const ::doctest::detail::Abort&) {
    } catch (const std::exception& e) {
      ::doctest::detail::fail(c.file, c.line, std::string("exception: ") + e.what());
    } catch (...) {
      ::doctest::detail::fail(c.file, c.line, "unknown exception");
    }
    const bool ok = ::doctest::detail::failures() == before;
    if (!ok) ++failed_cases;
    std::printf("[case] %s: %s\n", ok ? "passed" : "FAILED", c.name);
  }
  std::printf("[doctest] test cases: %d | %d passed | %d failed | assertions: %lld\n", run,
              run - failed_cases, failed_cases, ::doctest::detail::assertions());
  return failed_cases ? 1 : 0;
}
#endif
