// Runner for test files written against the Catch2 shim (TEST INFRASTRUCTURE).
// Usage: <binary> [substring filter]
#include <execinfo.h>
#include <pthread.h>
#include <signal.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "catch_amalgamated.hpp"

namespace {

// Per-case watchdog: a case that runs longer than FSX_CASE_TIMEOUT_S (default
// 180 s) gets the main thread's backtrace printed (SIGUSR1 handler; resolve
// the addresses with addr2line -e <binary>) and the process exits with 3,
// instead of hanging until the caller's timeout with no trace of where.
std::atomic<const char*> g_case{nullptr};
std::atomic<int64_t> g_case_start_ms{0};

int64_t now_ms() {
  return std::chrono::duration_cast<std::chrono::milliseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

void dump_and_exit(int) {
  void* frames[64];
  const int n = backtrace(frames, 64);
  const char* c = g_case.load();
  const char hdr[] = "\n[ HANG ] backtrace of the main thread:\n";
  (void)!write(2, hdr, sizeof hdr - 1);
  if (c) {
    (void)!write(2, c, std::strlen(c));
    (void)!write(2, "\n", 1);
  }
  backtrace_symbols_fd(frames, n, 2);
  _exit(3);
}

void start_watchdog() {
  const char* e = std::getenv("FSX_CASE_TIMEOUT_S");
  const int64_t limit_ms = (e ? std::atoll(e) : 180) * 1000;
  if (limit_ms <= 0) return;
  signal(SIGUSR1, dump_and_exit);
  const pthread_t main_thread = pthread_self();
  std::thread([=] {
    for (;;) {
      std::this_thread::sleep_for(std::chrono::milliseconds(500));
      const int64_t t0 = g_case_start_ms.load();
      if (g_case.load() && t0 > 0 && now_ms() - t0 > limit_ms) {
        pthread_kill(main_thread, SIGUSR1);
        std::this_thread::sleep_for(std::chrono::seconds(5));
        _exit(3);
      }
    }
  }).detach();
}

}  // namespace

int main(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  start_watchdog();
  int cases = 0, failed_cases = 0;
  for (const auto& c : catch_shim::registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    ++cases;
    const int before = catch_shim::state().failed;
    const auto t0 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[ RUN  ] %s\n", c.name);
    g_case_start_ms.store(now_ms());
    g_case.store(c.name);
    bool threw = false;
    try {
      c.fn();
    } catch (const catch_shim::RequireFailure&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "  FAILED: unexpected exception: %s\n", e.what());
      threw = true;
    }
    g_case.store(nullptr);
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    const bool bad = threw || catch_shim::state().failed != before;
    failed_cases += bad;
    std::fprintf(stderr, "[ %s ] %s (%.1f ms)\n", bad ? "FAIL" : " OK ", c.name, ms);
  }
  std::printf("%d test cases, %d failed, %d checks, %d failed checks\n", cases, failed_cases,
              catch_shim::state().checks, catch_shim::state().failed);
  std::fflush(stdout);
  // the watchdog also covers process exit (static destructors)
  g_case_start_ms.store(now_ms());
  g_case.store("<process exit>");
  return failed_cases == 0 && cases > 0 ? 0 : 1;
}
