// Minimal doctest-compatible test harness (our code, not doctest): just the
// constructs the reference's unit suites use (proj/tests/*.cpp): TEST_CASE,
// CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, FAIL, doctest::Approx(..).epsilon(..).
// The reference vendors real doctest under proj/vendor/ (git-ignored and absent),
// so this lets its test sources compile unchanged against the B200 drop-in.
#pragma once

#include <cmath>
#include <cstdio>
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
  double eps = 1.1920928955078125e-05;  // doctest's default: float epsilon * 100
  double scale = 1.0;
};
inline bool operator==(double lhs, const Approx& a) {
  return std::fabs(lhs - a.value) < a.eps * (a.scale + std::fmax(std::fabs(lhs), std::fabs(a.value)));
}
inline bool operator==(const Approx& a, double rhs) { return rhs == a; }
inline bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

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
struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) { registry().push_back({name, fn, file, line}); }
};
struct State {
  int assertions = 0, failed_assertions = 0;
  bool current_failed = false;
};
inline State& state() {
  static State s;
  return s;
}
struct Abort {};  // REQUIRE / FAIL stop the current test case
inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  ++state().assertions;
  if (ok) return;
  ++state().failed_assertions;
  state().current_failed = true;
  std::printf("%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, kind, expr);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                             \
  static void fn();                                                                                  \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);          \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_test_fn_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                   \
  do {                                                                                                 \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                           \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);               \
    if (!doctest_ok_) throw ::doctest::detail::Abort{};                                                \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                     \
  do {                                                                                                 \
    bool doctest_ok_ = false;                                                                          \
    try {                                                                                              \
      static_cast<void>(expr);                                                                         \
    } catch (const __VA_ARGS__&) {                                                                     \
      doctest_ok_ = true;                                                                              \
    } catch (...) {                                                                                    \
    }                                                                                                  \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__,      \
                              __LINE__);                                                               \
  } while (0)
#define FAIL(msg)                                                                                      \
  do {                                                                                                 \
    ::doctest::detail::report(false, "FAIL", msg, __FILE__, __LINE__);                                 \
    throw ::doctest::detail::Abort{};                                                                  \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  const char* only = nullptr;
  for (int i = 1; i < argc; ++i)
    if (std::string(argv[i]).rfind("--test-case=", 0) == 0) only = argv[i] + 12;
  int cases = 0, failed = 0;
  for (const auto& tc : ::doctest::detail::registry()) {
    if (only && std::string(tc.name).find(only) == std::string::npos) continue;
    ++cases;
    ::doctest::detail::state().current_failed = false;
    try {
      tc.fn();
    } catch (const ::doctest::detail::Abort&) {
    } catch (const std::exception& e) {
      std::printf("%s:%d: ERROR: test case THREW exception: %s\n", tc.file, tc.line, e.what());
      ::doctest::detail::state().current_failed = true;
    } catch (...) {
      std::printf("%s:%d: ERROR: test case THREW an unknown exception\n", tc.file, tc.line);
      ::doctest::detail::state().current_failed = true;
    }
    if (::doctest::detail::state().current_failed) {
      ++failed;
      std::printf("  in TEST_CASE: %s\n", tc.name);
    }
  }
  const auto& st = ::doctest::detail::state();
  std::printf("[doctest] test cases: %d | %d passed | %d failed\n", cases, cases - failed, failed);
  std::printf("[doctest] assertions: %d | %d passed | %d failed |\n", st.assertions,
              st.assertions - st.failed_assertions, st.failed_assertions);
  std::printf("[doctest] Status: %s!\n", failed ? "FAILURE" : "SUCCESS");
  return failed ? 1 : 0;
}
#endif
