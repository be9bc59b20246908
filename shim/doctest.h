// doctest.h -- minimal stand-in for the doctest subset the reference's unit
// tests use (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// CHECK_NOTHROW, FAIL, doctest::Approx, doctest::Contains).  doctest itself is
// not vendored in the reference (proj/.gitignore:2) nor installed here; this
// header lets /root/reference/proj/tests/*.cpp compile UNCHANGED against the
// GPU-backed shim (shim/dvs_gpu.cpp).  Define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
// in exactly one translation unit.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <stdexcept>  // the reference tests rely on doctest pulling these in
#include <ostream>
#include <sstream>
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
  int failed_checks = 0;
  int checks = 0;
};

inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* what, const char* file, int line, bool require) {
  ++state().checks;
  if (!ok) {
    ++state().failed_checks;
    std::fprintf(stderr, "%s:%d: %s FAILED: %s\n", file, line, require ? "REQUIRE" : "CHECK", what);
    if (require) throw RequireFailed{};
  }
}

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    // doctest: |lhs - v| < eps * (scale + max(|lhs|, |v|)), scale = 1
    const double margin = rhs.eps_ * (1.0 + std::fmax(std::fabs(lhs), std::fabs(rhs.value_)));
    return std::fabs(lhs - rhs.value_) < margin || lhs == rhs.value_;
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }

 private:
  double value_;
  double eps_ = 1.1920929e-07 * 100;  // doctest's default: float epsilon * 100
};

struct Contains {
  explicit Contains(const char* s) : needle(s) {}
  std::string needle;
};

inline bool matches(const std::string& msg, const Contains& c) {
  return msg.find(c.needle) != std::string::npos;
}
inline bool matches(const std::string& msg, const char* s) { return msg == s; }

inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    const int before = state().failed_checks;
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++state().failed_checks;
      std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw: %s\n", tc.file, tc.line, tc.name, e.what());
    } catch (...) {
      ++state().failed_checks;
      std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw an unknown exception\n", tc.file, tc.line,
                   tc.name);
    }
    if (state().failed_checks != before) {
      ++failed_cases;
      std::fprintf(stderr, "  -> FAILED: %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - static_cast<size_t>(failed_cases), failed_cases);
  std::printf("[doctest-shim] assertions: %d | %d passed | %d failed\n", state().checks,
              state().checks - state().failed_checks, state().failed_checks);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(p) DOCTEST_CAT(p, __LINE__)

#define TEST_CASE(name)                                                                   \
  static void DOCTEST_ANON(doctest_fn_)();                                                \
  static doctest::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__,          \
                                                       &DOCTEST_ANON(doctest_fn_));       \
  static void DOCTEST_ANON(doctest_fn_)()

#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(msg) doctest::report(false, msg, __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, ...)                                                        \
  do {                                                                                    \
    bool ok_ = false;                                                                     \
    try {                                                                                 \
      static_cast<void>(expr);                                                            \
    } catch (const __VA_ARGS__&) {                                                        \
      ok_ = true;                                                                         \
    } catch (...) {                                                                       \
    }                                                                                     \
    doctest::report(ok_, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")", __FILE__, __LINE__, false); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, with, ...)                                             \
  do {                                                                                    \
    bool ok_ = false;                                                                     \
    try {                                                                                 \
      static_cast<void>(expr);                                                            \
    } catch (const __VA_ARGS__& e_) {                                                     \
      ok_ = doctest::matches(e_.what(), with);                                            \
    } catch (...) {                                                                       \
    }                                                                                     \
    doctest::report(ok_, "CHECK_THROWS_WITH_AS(" #expr ")", __FILE__, __LINE__, false);   \
  } while (0)

#define CHECK_NOTHROW(expr)                                                               \
  do {                                                                                    \
    bool ok_ = true;                                                                      \
    try {                                                                                 \
      static_cast<void>(expr);                                                            \
    } catch (...) {                                                                       \
      ok_ = false;                                                                        \
    }                                                                                     \
    doctest::report(ok_, "CHECK_NOTHROW(" #expr ")", __FILE__, __LINE__, false);          \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::run_all(); }
#endif
