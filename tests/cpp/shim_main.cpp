// Runner for test files written against the Catch2 shim (TEST INFRASTRUCTURE).
// Usage: <binary> [substring filter]
#include <chrono>
#include <cstring>

#include "catch_amalgamated.hpp"

int main(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int cases = 0, failed_cases = 0;
  for (const auto& c : catch_shim::registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    ++cases;
    const int before = catch_shim::state().failed;
    const auto t0 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[ RUN  ] %s\n", c.name);
    bool threw = false;
    try {
      c.fn();
    } catch (const catch_shim::RequireFailure&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "  FAILED: unexpected exception: %s\n", e.what());
      threw = true;
    }
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    const bool bad = threw || catch_shim::state().failed != before;
    failed_cases += bad;
    std::fprintf(stderr, "[ %s ] %s (%.1f ms)\n", bad ? "FAIL" : " OK ", c.name, ms);
  }
  std::printf("%d test cases, %d failed, %d checks, %d failed checks\n", cases, failed_cases,
              catch_shim::state().checks, catch_shim::state().failed);
  return failed_cases == 0 && cases > 0 ? 0 : 1;
}
