// Acceptance criterion 4 of the reference ("sidecar integrity, soak, and
// forwarding envelope", tests/acceptance_test.cpp:229-334) re-expressed for the
// drop-in fissim::SidecarFabric (include/fsx/dropin/fissim/sidecar.hpp) on the
// reference's own SimKernel, including its RealTime kernel thread.  The
// acceptance binary itself cannot run on the GPU box (its other criteria read
// reference fixture files), so this harness restates criterion 4 only.
//
//   usage: dropin_criterion4 [soak_seconds=60]
#include <atomic>
#include <chrono>
#include <cstdio>
#include <future>
#include <random>
#include <thread>

#include "fissim/sidecar.hpp"

using namespace fissim;

namespace {

int failures = 0;

void check(bool ok, const std::string& what) {
  if (!ok) {
    ++failures;
    std::printf("  FAILED: %s\n", what.c_str());
  }
}

std::map<int, int> topo() {
  std::map<int, int> t;
  for (int g = 0; g < 8; ++g) t[g] = g < 4 ? 0 : 1;
  return t;
}

DataRef ref_of(const std::string& id, size_t bytes) {
  DataRef r;
  r.ref_id = id;
  r.producer = "p";
  r.desc = {{static_cast<int64_t>(bytes)}, 1};
  return r;
}

void byte_exact_sweep() {
  SimKernel kernel(ClockMode::Virtual);
  SidecarConfig cfg;
  cfg.arena_bytes = 192 * 1024 * 1024;
  SidecarFabric fabric(kernel, topo(), cfg);
  std::mt19937_64 rng(4040);
  for (int i = 0; i < 24; ++i) {
    size_t size = i < 2 ? (i + 1) : size_t(1) << (rng() % 27);
    if (i % 5 == 0) size = (size_t(1) << 26) - (rng() % 1000);
    const int dst = (i % 2 == 0) ? 2 : 6;
    const std::string id = "acc4/r" + std::to_string(i);
    auto payload = synth_payload(rng(), size);
    std::vector<uint8_t> got;
    bool final_seen = false;
    fabric.register_interest(dst, id, [&](const ForwardEnvelope& env, std::vector<uint8_t> b) {
      got = std::move(b);
      final_seen = env.final;
    });
    kernel.post("send", [&, id, dst, size] { fabric.send_payload("acc4", ref_of(id, size), 0, dst, payload); });
    kernel.run_until_idle();
    check(final_seen, "transfer did not complete");
    check(got == payload, "bytes differ after transfer of size " + std::to_string(size));
  }
  auto s = fabric.stats();
  check(s.integrity_errors == 0, "integrity errors in byte-exactness sweep");
  check(s.segments_in_use == 0, "arena leak in byte-exactness sweep");
}

void soak(double seconds) {
  SimKernel kernel(ClockMode::RealTime);
  SidecarFabric fabric(kernel, topo());  // default 1 GiB slab per destination gpu
  const int total = static_cast<int>(15 * seconds);
  const size_t bytes = 32 * 1024 * 1024;
  std::atomic<int> delivered{0};
  auto base = synth_payload(99, bytes);
  for (int i = 0; i < total; ++i)
    fabric.register_interest(1, "soak/r" + std::to_string(i),
                             [&](const ForwardEnvelope&, std::vector<uint8_t> got) {
                               if (got.size() == bytes && got == base) delivered.fetch_add(1);
                             });
  for (int i = 0; i < total; ++i)
    kernel.schedule(i * (1000.0 / 15.0), "soak.send", [&fabric, &base, i] {
      fabric.send_payload("soak", ref_of("soak/r" + std::to_string(i), base.size()), 0, 1, base);
    });
  kernel.start();
  auto deadline = std::chrono::steady_clock::now() +
                  std::chrono::milliseconds(static_cast<int64_t>(seconds * 1000) + 40000);
  while (delivered.load() < total && std::chrono::steady_clock::now() < deadline)
    std::this_thread::sleep_for(std::chrono::milliseconds(20));
  kernel.stop();
  auto s = fabric.stats();
  check(delivered.load() == total, "soak lost transfers: " + std::to_string(delivered.load()) + "/" +
                                       std::to_string(total));
  check(s.integrity_errors == 0, "soak integrity errors");
  check(s.segments_in_use == 0, "soak arena leak");
}

void latency_envelope() {
  SimKernel kernel(ClockMode::RealTime);
  SidecarFabric fabric(kernel, topo());
  kernel.start();
  const size_t bytes = 8 * 1024 * 1024;
  auto payload = synth_payload(7, bytes);
  std::vector<double> ms;
  for (int i = 0; i < 5; ++i) {
    const std::string id = "lat/r" + std::to_string(i);
    std::promise<void> done;
    fabric.register_interest(1, id, [&done](const ForwardEnvelope&, std::vector<uint8_t>) { done.set_value(); });
    auto t0 = std::chrono::steady_clock::now();
    kernel.post("lat.send", [&fabric, &payload, id] {
      fabric.send_payload("lat", ref_of(id, payload.size()), 0, 1, payload);
    });
    done.get_future().wait();
    ms.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
  kernel.stop();
  std::sort(ms.begin(), ms.end());
  std::printf("  8 MiB forward median %.3f ms (modeled latency %.3f ms included by the RealTime kernel)\n",
              ms[ms.size() / 2], SidecarConfig{}.latency_ms(Transport::LocalBuffer, bytes));
  check(ms[ms.size() / 2] <= 50.0, "8 MB forwarding took too long");
}

}  // namespace

int main(int argc, char** argv) {
  const double soak_s = argc > 1 ? std::atof(argv[1]) : 60.0;
  auto t0 = std::chrono::steady_clock::now();
  byte_exact_sweep();
  std::printf("byte-exactness sweep done (%d failures)\n", failures);
  soak(soak_s);
  std::printf("soak %.0f s done (%d failures)\n", soak_s, failures);
  latency_envelope();
  std::printf("criterion 4 on the drop-in: %s in %.1f s\n", failures ? "FAILED" : "PASSED",
              std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  return failures ? 1 : 0;
}
