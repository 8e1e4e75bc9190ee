// TEST INFRASTRUCTURE — stand-in for the few Catch2 v3 macros the reference's own test files for the hot
// path use (proj/tests/test_core.cpp, test_blas.cpp: TEST_CASE, SECTION incl. nesting, CHECK, REQUIRE,
// CHECK_THROWS_AS, Catch::Approx with epsilon / margin).  Catch2 is not installed in this image; with this
// header the reference's test sources compile unchanged (oracle/Makefile, target _ref/ref_tests_*) and run
// against the reference headers + oracle/eigen_standin.  Written for this repository; header-only, main()
// included.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

namespace Catch {

class Approx {
public:
  explicit Approx(double v) : v_(v) {}
  Approx &epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx &margin(double m) {
    margin_ = m;
    return *this;
  }
  bool matches(double x) const {
    const double d = std::fabs(x - v_);
    return d <= margin_ || d <= eps_ * (std::isinf(v_) ? 0.0 : std::fabs(v_));
  }
  double value() const { return v_; }

private:
  double v_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double margin_ = 0.0;
};
inline bool operator==(double x, const Approx &a) { return a.matches(x); }
inline bool operator==(const Approx &a, double x) { return a.matches(x); }
inline bool operator!=(double x, const Approx &a) { return !a.matches(x); }
inline bool operator!=(const Approx &a, double x) { return !a.matches(x); }
inline bool operator<=(double x, const Approx &a) { return x < a.value() || a.matches(x); }
inline bool operator>=(double x, const Approx &a) { return x > a.value() || a.matches(x); }

namespace standin {

struct TestCase {
  const char *name;
  void (*fn)();
};
inline std::vector<TestCase> &registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Registrar {
  Registrar(const char *name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct AbortTestCase {};
inline const char *first_arg(const char *name, const char * = nullptr) { return name; }

struct State {
  std::vector<int> target;   // section index to enter at each depth on this pass
  std::vector<int> seen;     // sections met so far at each depth (under the entered parent)
  std::vector<char> entered; // a section was already entered at this depth on this pass
  int depth = 0;
  int checks = 0, failures = 0;
  std::string current;
  bool taken(int d) const { return d < static_cast<int>(entered.size()) && entered[d]; }
  void mark_taken(int d) {
    if (static_cast<int>(entered.size()) <= d)
      entered.resize(d + 1, 0);
    entered[d] = 1;
  }
};
inline State &state() {
  static State s;
  return s;
}

class Section {
public:
  // Sections at depth d + 1 are only met inside the entered section of depth d, so one counter per depth
  // is enough: seen[d] ends the pass as the number of siblings along the path taken.
  explicit Section(const char *) {
    State &s = state();
    const int d = s.depth;
    if (static_cast<int>(s.seen.size()) <= d)
      s.seen.resize(d + 1, 0);
    const int idx = s.seen[d]++;
    if (static_cast<int>(s.target.size()) == d && idx == 0) {
      s.target.push_back(0);  // first visit of this depth: take the first section
      entered_ = true;
    } else {
      entered_ = static_cast<int>(s.target.size()) > d && s.target[d] == idx && !s.taken(d);
    }
    if (entered_) {
      s.mark_taken(d);
      ++s.depth;
    }
  }
  ~Section() {
    if (entered_)
      --state().depth;
  }
  explicit operator bool() const { return entered_; }

private:
  bool entered_ = false;
};

inline void report_failure(const char *kind, const char *expr, const char *file, int line) {
  State &s = state();
  ++s.failures;
  std::printf("FAILED %s:%d: %s( %s )   [test case: %s]\n", file, line, kind, expr, s.current.c_str());
}

inline int run_all() {
  State &s = state();
  int cases = 0, failed_cases = 0;
  for (const TestCase &tc : registry()) {
    ++cases;
    const int before = s.failures;
    s.current = tc.name;
    s.target.clear();
    for (;;) {  // one pass per leaf section
      s.seen.clear();
      s.entered.clear();
      s.depth = 0;
      try {
        tc.fn();
      } catch (const AbortTestCase &) {
      } catch (const std::exception &e) {
        ++s.failures;
        std::printf("FAILED [test case: %s]: unexpected exception: %s\n", tc.name, e.what());
      }
      bool advanced = false;
      while (!s.target.empty()) {
        const size_t d = s.target.size() - 1;
        const int siblings = d < s.seen.size() ? s.seen[d] : 0;
        if (s.target[d] + 1 < siblings) {
          ++s.target[d];
          advanced = true;
          break;
        }
        s.target.pop_back();
      }
      if (!advanced)
        break;
    }
    if (s.failures != before)
      ++failed_cases;
  }
  std::printf("%s: %d test cases, %d assertions, %d failures\n", failed_cases ? "FAILED" : "ok", cases, s.checks,
              s.failures);
  return failed_cases ? 1 : 0;
}

} // namespace standin
} // namespace Catch

#define CATCH_STANDIN_CAT2(a, b) a##b
#define CATCH_STANDIN_CAT(a, b) CATCH_STANDIN_CAT2(a, b)
#define TEST_CASE(...)                                                                                              \
  static void CATCH_STANDIN_CAT(catch_standin_case_, __LINE__)();                                                   \
  static ::Catch::standin::Registrar CATCH_STANDIN_CAT(catch_standin_reg_, __LINE__)(                               \
      ::Catch::standin::first_arg(__VA_ARGS__), &CATCH_STANDIN_CAT(catch_standin_case_, __LINE__));                 \
  static void CATCH_STANDIN_CAT(catch_standin_case_, __LINE__)()
#define SECTION(...) if (::Catch::standin::Section CATCH_STANDIN_CAT(catch_standin_sec_, __LINE__){""})
#define CHECK(...)                                                                                                  \
  do {                                                                                                              \
    ++::Catch::standin::state().checks;                                                                             \
    if (!(__VA_ARGS__))                                                                                             \
      ::Catch::standin::report_failure("CHECK", #__VA_ARGS__, __FILE__, __LINE__);                                  \
  } while (0)
#define REQUIRE(...)                                                                                                \
  do {                                                                                                              \
    ++::Catch::standin::state().checks;                                                                             \
    if (!(__VA_ARGS__)) {                                                                                           \
      ::Catch::standin::report_failure("REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                                \
      throw ::Catch::standin::AbortTestCase{};                                                                      \
    }                                                                                                               \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                                                 \
  do {                                                                                                              \
    ++::Catch::standin::state().checks;                                                                             \
    bool catch_standin_ok = false;                                                                                  \
    try {                                                                                                           \
      static_cast<void>(expr);                                                                                      \
    } catch (const type &) {                                                                                        \
      catch_standin_ok = true;                                                                                      \
    } catch (...) {                                                                                                 \
    }                                                                                                               \
    if (!catch_standin_ok)                                                                                          \
      ::Catch::standin::report_failure("CHECK_THROWS_AS", #expr ", " #type, __FILE__, __LINE__);                    \
  } while (0)

#ifndef CATCH_STANDIN_NO_MAIN
int main() { return ::Catch::standin::run_all(); }
#endif
