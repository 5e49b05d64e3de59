// doctest.h — a minimal doctest-compatible test shim (this repo's own code).
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) are written
// against doctest, which the reference does not vendor (proj/.gitignore:2) and
// which is not installable offline.  This header implements just the subset
// those files use — TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, REQUIRE_MESSAGE,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, doctest::Approx and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN — so the reference's test files compile
// UNMODIFIED against the B200 drop-in and run as plain executables
// (exit code = number of failed test cases).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

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

struct State {
  int checks = 0;
  int failed_checks = 0;
  bool current_failed = false;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireFailure {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   const char* extra = nullptr) {
  State& st = state();
  ++st.checks;
  if (!ok) {
    ++st.failed_checks;
    st.current_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s )%s%s\n", file, line, kind, expr, extra ? " -- " : "",
                 extra ? extra : "");
  }
}

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
  friend bool operator==(double lhs, const Approx& rhs) { return rhs.eq(lhs); }
  friend bool operator==(const Approx& lhs, double rhs) { return lhs.eq(rhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.eq(lhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.eq(rhs); }

 private:
  bool eq(double x) const {
    const double m = std::fmax(std::fabs(x), std::fabs(value_));
    return std::fabs(x - value_) < eps_ * (scale_ + m);
  }
  double value_;
  double eps_ = 1.1920929e-07 * 100;  // doctest's default: float epsilon * 100
  double scale_ = 1.0;
};

inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    state().current_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailure&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: test case \"%s\" threw: %s\n", tc.file, tc.line, tc.name, e.what());
      state().current_failed = true;
    } catch (...) {
      std::fprintf(stderr, "%s:%d: test case \"%s\" threw an unknown exception\n", tc.file, tc.line, tc.name);
      state().current_failed = true;
    }
    if (state().current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "[doctest-shim] FAILED: %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - failed_cases, failed_cases);
  std::printf("[doctest-shim] assertions: %d | %d passed | %d failed\n", state().checks,
              state().checks - state().failed_checks, state().failed_checks);
  return failed_cases;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                                   \
  static void fn();                                                                             \
  static doctest::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);               \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  doctest::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                          \
  do {                                                                                        \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                  \
    doctest::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                \
    if (!doctest_ok_) throw doctest::RequireFailure{};                                        \
  } while (0)
#define REQUIRE_MESSAGE(cond, msg)                                                            \
  do {                                                                                        \
    const bool doctest_ok_ = static_cast<bool>(cond);                                         \
    doctest::report(doctest_ok_, "REQUIRE_MESSAGE", #cond, __FILE__, __LINE__);               \
    if (!doctest_ok_) throw doctest::RequireFailure{};                                        \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                            \
  do {                                                                                        \
    bool doctest_ok_ = false;                                                                 \
    try {                                                                                     \
      static_cast<void>(expr);                                                                \
    } catch (const __VA_ARGS__&) {                                                            \
      doctest_ok_ = true;                                                                     \
    } catch (...) {                                                                           \
    }                                                                                         \
    doctest::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, ...)                                                  \
  do {                                                                                        \
    bool doctest_ok_ = false;                                                                 \
    try {                                                                                     \
      static_cast<void>(expr);                                                                \
    } catch (const __VA_ARGS__& e) {                                                          \
      doctest_ok_ = std::string(e.what()).find(msg) != std::string::npos;                     \
    } catch (...) {                                                                           \
    }                                                                                         \
    doctest::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__);          \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::run_all(); }
#endif
