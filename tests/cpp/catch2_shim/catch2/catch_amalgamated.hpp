// Minimal stand-in for <catch2/catch_amalgamated.hpp> (Catch2 v3 is not installed in
// this image; the reference's proj/tests/CMakeLists.txt:3-4 expects it under
// /usr/local/include).  It implements exactly the subset the reference's unit tests
// use -- TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH,
// FAIL and Catch::Approx(..).margin(..)/.epsilon(..) -- so that those test files can be
// compiled UNMODIFIED against this repo's drop-in headers (include/chunklab/*.hpp) and
// run on the B200 (oracle/Makefile target `reftests`).  Test infrastructure only.
#pragma once

// the real amalgamated header pulls these in transitively; test files rely on it
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <set>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

namespace Catch {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  bool matches(double x) const {
    const double d = std::fabs(x - value_);
    if (d <= margin_) return true;
    // Catch2 v3: relative part scaled by |value| (Approx::equalityComparisonImpl)
    return d <= epsilon_ * (std::isinf(value_) ? 0.0 : std::fabs(value_));
  }
  friend bool operator==(double x, const Approx& a) { return a.matches(x); }
  friend bool operator==(const Approx& a, double x) { return a.matches(x); }
  friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
  friend bool operator!=(const Approx& a, double x) { return !a.matches(x); }
  double value() const { return value_; }

 private:
  double value_;
  double margin_ = 0.0;
  // Catch2's default: float epsilon * 100
  double epsilon_ = 1.1920928955078125e-07 * 100.0;
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

struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};

struct State {
  long checks = 0;
  long failed_checks = 0;
  bool case_failed = false;
};

inline State& state() {
  static State s;
  return s;
}

struct RequireFailure {};

inline void report(bool ok, const char* file, int line, const char* what, bool fatal) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failed_checks;
  s.case_failed = true;
  std::printf("  %s:%d: FAILED: %s\n", file, line, what);
  if (fatal) throw RequireFailure{};
}

inline int run_all() {
  int failed = 0, passed = 0;
  for (const TestCase& tc : registry()) {
    State& s = state();
    s.case_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailure&) {
    } catch (const std::exception& e) {
      s.case_failed = true;
      std::printf("  %s:%d: unexpected exception: %s\n", tc.file, tc.line, e.what());
    } catch (...) {
      s.case_failed = true;
      std::printf("  %s:%d: unexpected non-std exception\n", tc.file, tc.line);
    }
    if (s.case_failed) {
      ++failed;
      std::printf("FAILED test case: %s\n", tc.name);
    } else {
      ++passed;
    }
  }
  std::printf("test cases: %d passed, %d failed | assertions: %ld passed, %ld failed\n", passed,
              failed, state().checks - state().failed_checks, state().failed_checks);
  return failed == 0 ? 0 : 1;
}

}  // namespace shim
}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_TEST_CASE2(fn, name, ...)                                               \
  static void fn();                                                                       \
  static const ::Catch::shim::Registrar CATCH_SHIM_CAT(fn, _reg){name, &fn, __FILE__,     \
                                                                 __LINE__};               \
  static void fn()
#define TEST_CASE(...) CATCH_SHIM_TEST_CASE2(CATCH_SHIM_CAT(catch_shim_case_, __LINE__), __VA_ARGS__)

#define CHECK(...) ::Catch::shim::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) ::Catch::shim::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) ::Catch::shim::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define FAIL(msg)                                                                          \
  do {                                                                                     \
    std::ostringstream catch_shim_os;                                                      \
    catch_shim_os << msg;                                                                  \
    ::Catch::shim::report(false, __FILE__, __LINE__, catch_shim_os.str().c_str(), true);   \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                        \
  do {                                                                                     \
    bool catch_shim_ok = false;                                                            \
    try {                                                                                  \
      static_cast<void>(expr);                                                             \
    } catch (const type&) {                                                                \
      catch_shim_ok = true;                                                                \
    } catch (...) {                                                                        \
    }                                                                                      \
    ::Catch::shim::report(catch_shim_ok, __FILE__, __LINE__, "throws " #type ": " #expr,   \
                          false);                                                          \
  } while (0)
#define CHECK_THROWS_WITH(expr, msg)                                                       \
  do {                                                                                     \
    bool catch_shim_ok = false;                                                            \
    std::string catch_shim_got = "(no exception)";                                         \
    try {                                                                                  \
      static_cast<void>(expr);                                                             \
    } catch (const std::exception& e) {                                                    \
      catch_shim_got = e.what();                                                           \
      catch_shim_ok = catch_shim_got == std::string(msg);                                  \
    } catch (...) {                                                                        \
      catch_shim_got = "(non-std exception)";                                              \
    }                                                                                      \
    if (!catch_shim_ok) std::printf("  got: %s\n", catch_shim_got.c_str());                \
    ::Catch::shim::report(catch_shim_ok, __FILE__, __LINE__, "throws with: " #expr, false); \
  } while (0)

// The amalgamated Catch2 distribution links main() from catch_amalgamated.cpp
// (proj/tests/CMakeLists.txt:3); the shim provides it when CATCH_SHIM_MAIN is defined.
#ifdef CATCH_SHIM_MAIN
int main() { return ::Catch::shim::run_all(); }
#endif
