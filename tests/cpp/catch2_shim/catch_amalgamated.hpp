// Minimal stand-in for Catch2's amalgamated header (TEST INFRASTRUCTURE).
//
// Catch2 is not installed in this image, so the reference's own
// unit test files (e.g. /root/reference/proj/tests/test_sidecar.cpp) are
// compiled UNMODIFIED against this shim plus the fsx drop-in sidecar header,
// and run on the GPU.  Supports the subset those files use: TEST_CASE, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS.  main() lives in shim_main.cpp.
#pragma once
#include <iostream>

#include <cstdio>
#include <exception>
#include <string>
#include <vector>

namespace catch_shim {

struct Case {
  const char* name;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> cases;
  return cases;
}

struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct State {
  int checks = 0;
  int failed = 0;
  const char* current = "";
};

inline State& state() {
  static State s;
  return s;
}

struct RequireFailure {};

inline void check(bool ok, const char* expr, const char* file, int line, bool require) {
  ++state().checks;
  if (ok) return;
  ++state().failed;
  std::fprintf(stderr, "  FAILED %s: %s (%s:%d)\n", require ? "REQUIRE" : "CHECK", expr, file, line);
  if (require) throw RequireFailure{};
}

}  // namespace catch_shim

namespace Catch {
// Catch2's Approx: relative epsilon (default 100 * float epsilon) or absolute margin.
class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    const double d = lhs > a.value_ ? lhs - a.value_ : a.value_ - lhs;
    const double scale = (lhs > 0 ? lhs : -lhs) > (a.value_ > 0 ? a.value_ : -a.value_)
                             ? (lhs > 0 ? lhs : -lhs)
                             : (a.value_ > 0 ? a.value_ : -a.value_);
    return d <= a.margin_ || d <= a.eps_ * scale;
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

 private:
  double value_;
  double eps_ = 1.1920929e-07 * 100;
  double margin_ = 0.0;
};
}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_CASE(fn, name)                                   \
  static void fn();                                                 \
  static catch_shim::Registrar CATCH_SHIM_CAT(fn, _reg)(name, &fn); \
  static void fn()
#define TEST_CASE(name, ...) CATCH_SHIM_CASE(CATCH_SHIM_CAT(catch_shim_case_, __LINE__), name)
#define CHECK(...) catch_shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) \
  catch_shim::check(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) catch_shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_FALSE(...) \
  catch_shim::check(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)
#define FAIL(msg) catch_shim::check(false, msg, __FILE__, __LINE__, true)
#define WARN(msg) (std::cerr << "WARN: " << msg << "\n")
#define CHECK_NOTHROW(expr)                                                          \
  do {                                                                               \
    bool catch_shim_ok = true;                                                       \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (...) {                                                                  \
      catch_shim_ok = false;                                                         \
    }                                                                                \
    catch_shim::check(catch_shim_ok, #expr " does not throw", __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                   \
  do {                                                                                \
    bool catch_shim_thrown = false;                                                   \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (const type&) {                                                           \
      catch_shim_thrown = true;                                                       \
    } catch (...) {                                                                   \
    }                                                                                 \
    catch_shim::check(catch_shim_thrown, #expr " throws " #type, __FILE__, __LINE__, false); \
  } while (0)
