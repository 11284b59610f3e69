// Minimal doctest-compatible test shim (test infrastructure, not product).
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) include
// "doctest.h", which the reference never vendored (proj/.gitignore:2 ignores
// /vendor/). This header implements only the subset those suites use —
// TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, REQUIRE_MESSAGE, CHECK_THROWS,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, doctest::Approx(..).epsilon(..),
// doctest::Contains — so the UNMODIFIED reference test sources compile and
// run against either the reference engine (oracle/_ref) or the B200 engine.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  double value;
  double eps = 1.1920928955078125e-05 * 100;  // doctest default: FLT_EPSILON * 100
};
inline bool approx_eq(double lhs, const Approx& a) {
  return std::fabs(lhs - a.value) <
         a.eps * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.value)));
}
inline bool operator==(double lhs, const Approx& rhs) { return approx_eq(lhs, rhs); }
inline bool operator==(const Approx& lhs, double rhs) { return approx_eq(rhs, lhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !approx_eq(lhs, rhs); }
inline bool operator!=(const Approx& lhs, double rhs) { return !approx_eq(rhs, lhs); }

struct Contains {
  explicit Contains(std::string s) : needle(std::move(s)) {}
  bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
  std::string needle;
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

struct State {
  long checks = 0;
  long failures = 0;
  bool current_failed = false;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireAbort {};

inline void report(bool ok, bool require, const char* file, int line, const char* what,
                   const char* msg = nullptr) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  s.current_failed = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED%s%s\n", file, line, require ? "REQUIRE" : "CHECK",
               what, msg ? " — " : "", msg ? msg : "");
  if (require) throw RequireAbort{};
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

inline bool message_matches(const std::string& what, const Contains& c) { return c.matches(what); }
inline bool message_matches(const std::string& what, const char* s) { return what == s; }
inline bool message_matches(const std::string& what, const std::string& s) { return what == s; }

inline int run_all(int argc, char** argv) {
  const char* filter = nullptr;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("--test-case=", 0) == 0) filter = argv[i] + 12;
  }
  State& s = state();
  int cases = 0, failed_cases = 0;
  for (const auto& tc : registry()) {
    if (filter && std::string(tc.name).find(filter) == std::string::npos) continue;
    ++cases;
    s.current_failed = false;
    try {
      tc.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      ++s.failures;
      s.current_failed = true;
      std::fprintf(stderr, "%s:%d: TEST CASE '%s' threw: %s\n", tc.file, tc.line, tc.name, e.what());
    } catch (...) {
      ++s.failures;
      s.current_failed = true;
      std::fprintf(stderr, "%s:%d: TEST CASE '%s' threw a non-std exception\n", tc.file, tc.line,
                   tc.name);
    }
    if (s.current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "[doctest-shim] FAILED: %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %ld | %ld failed\n",
              cases, cases - failed_cases, failed_cases, s.checks, s.failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                              \
  static void DOCTEST_ANON(doctest_fn_)();                                           \
  static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(                    \
      name, __FILE__, __LINE__, &DOCTEST_ANON(doctest_fn_));                         \
  static void DOCTEST_ANON(doctest_fn_)()

#define DOCTEST_EVAL_(expr, req, msg)                                                \
  do {                                                                               \
    bool doctest_ok_ = false;                                                        \
    try {                                                                            \
      doctest_ok_ = static_cast<bool>(expr);                                         \
    } catch (const ::doctest::detail::RequireAbort&) {                               \
      throw;                                                                         \
    } catch (const std::exception& e) {                                              \
      ::doctest::detail::report(false, req, __FILE__, __LINE__, #expr, e.what());    \
      break;                                                                         \
    }                                                                                \
    ::doctest::detail::report(doctest_ok_, req, __FILE__, __LINE__, #expr, msg);     \
  } while (0)

#define CHECK(...) DOCTEST_EVAL_((__VA_ARGS__), false, nullptr)
#define CHECK_FALSE(...) DOCTEST_EVAL_(!(__VA_ARGS__), false, nullptr)
#define REQUIRE(...) DOCTEST_EVAL_((__VA_ARGS__), true, nullptr)
#define REQUIRE_MESSAGE(cond, msg) DOCTEST_EVAL_((cond), true, msg)
#define FAIL(msg) ::doctest::detail::report(false, true, __FILE__, __LINE__, "FAIL", msg)

#define CHECK_THROWS(...)                                                            \
  do {                                                                               \
    bool doctest_threw_ = false;                                                     \
    try {                                                                            \
      (void)(__VA_ARGS__);                                                           \
    } catch (...) {                                                                  \
      doctest_threw_ = true;                                                         \
    }                                                                                \
    ::doctest::detail::report(doctest_threw_, false, __FILE__, __LINE__,             \
                              "THROWS " #__VA_ARGS__);                               \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                   \
  do {                                                                               \
    bool doctest_threw_ = false;                                                     \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const __VA_ARGS__&) {                                                   \
      doctest_threw_ = true;                                                         \
    } catch (...) {                                                                  \
    }                                                                                \
    ::doctest::detail::report(doctest_threw_, false, __FILE__, __LINE__,             \
                              "THROWS_AS " #expr ", " #__VA_ARGS__);                 \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, with, ...)                                        \
  do {                                                                               \
    bool doctest_ok_ = false;                                                        \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const __VA_ARGS__& e) {                                                 \
      doctest_ok_ = ::doctest::detail::message_matches(e.what(), with);              \
    } catch (...) {                                                                  \
    }                                                                                \
    ::doctest::detail::report(doctest_ok_, false, __FILE__, __LINE__,                \
                              "THROWS_WITH_AS " #expr);                              \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run_all(argc, argv); }
#endif
