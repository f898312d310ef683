// Minimal doctest-compatible shim (TEST_CASE / SUBCASE / CHECK / REQUIRE /
// CHECK_THROWS_AS / Approx) so doctest-style suites build without the doctest
// dependency (absent here).  Each TEST_CASE body is re-run once per
// SUBCASE, entering exactly one subcase per run, as doctest does.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace shim {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}
struct SubcaseState {
  int target = 0;  // which subcase to enter this run
  int seen = 0;    // subcases encountered this run
};
inline SubcaseState& sub() {
  static SubcaseState s;
  return s;
}
inline bool enter_subcase() { return sub().seen++ == sub().target; }
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  checks()++;
  if (ok) return;
  failures()++;
  std::fprintf(stderr, "%s:%d: check failed: %s\n", file, line, expr);
  if (require) throw RequireFailed{};
}
}  // namespace shim

namespace doctest {
struct Approx {
  explicit Approx(double v) : value(v) {}
  double value;
  double eps = 1e-5;
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value) <= a.eps * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.value)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
};
}  // namespace doctest

#define SHIM_CAT2(a, b) a##b
#define SHIM_CAT(a, b) SHIM_CAT2(a, b)
#define TEST_CASE(name)                                                              \
  static void SHIM_CAT(shim_case_, __LINE__)();                                      \
  static shim::Registrar SHIM_CAT(shim_reg_, __LINE__)(name, SHIM_CAT(shim_case_, __LINE__)); \
  static void SHIM_CAT(shim_case_, __LINE__)()
#define SUBCASE(name) if (shim::enter_subcase())
#define CHECK(...) shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                        \
  do {                                                                     \
    bool thrown_ = false;                                                  \
    try {                                                                  \
      (void)(expr);                                                        \
    } catch (const type&) {                                                \
      thrown_ = true;                                                      \
    } catch (...) {                                                        \
    }                                                                      \
    shim::report(thrown_, "throws " #type ": " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define FAIL(msg) shim::report(false, msg, __FILE__, __LINE__, true)

#ifdef SHIM_MAIN
int main() {
  int cases = 0;
  for (const auto& c : shim::registry()) {
    shim::sub().target = 0;
    do {
      shim::sub().seen = 0;
      try {
        c.fn();
      } catch (const shim::RequireFailed&) {
      } catch (const std::exception& e) {
        shim::failures()++;
        std::fprintf(stderr, "%s: unexpected exception: %s\n", c.name, e.what());
      }
      shim::sub().target++;
    } while (shim::sub().target < shim::sub().seen);
    cases++;
  }
  std::printf("%d test cases, %d checks, %d failures\n", cases, shim::checks(), shim::failures());
  return shim::failures() ? 1 : 0;
}
#endif
