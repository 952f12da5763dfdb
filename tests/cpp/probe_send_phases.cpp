// Host-overhead probe of the drop-in engine's small-message path (config C:
// 32 host-span rows per decode step into ChunkCallback consumers): the
// FSX_PHASE hooks of include/fsx/fabric.hpp record the time between
// consecutive hook points; one JSON line per transition, ns per message.
#include <cuda_runtime.h>
#include <x86intrin.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <map>
#include <string>
#include <utility>

static uint64_t g_last_t = 0;
static int g_last_i = -1;
static std::map<std::pair<int, int>, std::pair<uint64_t, uint64_t>> g_acc;  // (from,to) -> (ticks, count)
static bool g_on = false;
static inline void phase_mark(int i) {
  const uint64_t t = __rdtsc();
  if (g_on && g_last_i >= 0) {
    auto& a = g_acc[{g_last_i, i}];
    a.first += t - g_last_t;
    a.second += 1;
  }
  g_last_t = t;
  g_last_i = i;
}
#define FSX_PHASE(i) phase_mark(i)

#include "fsx/fabric.hpp"

extern "C" {
#include "fsx_oracle.h"
}

using namespace fsx;

int main(int argc, char** argv) {
  const int row = argc > 1 ? std::atoi(argv[1]) : 7168;
  const bool device = argc > 2 && std::string(argv[2]) == "device";  // device rows -> raw consumers
  const int batch = 32, steps = 400;
  std::map<int, int> topo{{0, 0}, {1, 0}};
  EventLoop k;
  SidecarConfig cfg;
  cfg.async_borrowed_sources = device;
  SidecarFabric f(k, topo, cfg);
  std::vector<uint8_t> rowbuf(row);
  or_synth_payload_into(7, rowbuf.data(), row);
  void* drow = nullptr;
  if (device) {
    if (cudaMalloc(&drow, (size_t)row * batch) != cudaSuccess) return 2;
    for (int r = 0; r < batch; ++r)
      cudaMemcpy(static_cast<uint8_t*>(drow) + (size_t)r * row, rowbuf.data(), row, cudaMemcpyHostToDevice);
    cudaDeviceSynchronize();  // pageable-source copies may return before their DMA lands
  }
  int64_t got = 0;
  for (int r = 0; r < batch; ++r) {
    if (device)
      f.register_interest_raw(1, "req-" + std::to_string(100000 + r) + "/r0001",
                              [&](const ForwardEnvelope& env, int64_t off) {
                                FSX_PHASE(15);
                                got += env.chunk_bytes;
                                f.ack_raw(1, off);
                              });
    else
      f.register_interest(1, "req-" + std::to_string(100000 + r) + "/r0001",
                          [&](const ForwardEnvelope&, std::vector<uint8_t> b) {
                            FSX_PHASE(15);
                            got += (int64_t)b.size();
                          });
  }
  auto step = [&](int s) {
    for (int r = 0; r < batch; ++r)
      f.send("req-" + std::to_string(100000 + r),
             DataRef{"req-" + std::to_string(100000 + r) + "/r0001", 0, true}, 0, 1,
             std::span<const uint8_t>(device ? static_cast<const uint8_t*>(drow) + (size_t)r * row
                                             : rowbuf.data(), row),
             s, false);
    FSX_PHASE(16);
    k.run_until_idle();
    FSX_PHASE(17);
  };
  for (int s = 0; s < 20; ++s) step(s);
  const auto a = std::chrono::steady_clock::now();
  const uint64_t t0 = __rdtsc();
  g_on = true;
  for (int s = 20; s < 20 + steps; ++s) step(s);
  g_on = false;
  const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
  const double ns_per_tick = sec * 1e9 / double(__rdtsc() - t0);
  std::printf("{\"row_bytes\": %d, \"source\": \"%s\", \"us_per_step\": %.1f}\n", row,
              device ? "device rows, raw interest" : "host span, ChunkCallback", sec / steps * 1e6);
  for (auto& [k2, v] : g_acc)
    std::printf("{\"from\": %d, \"to\": %d, \"ns_per_msg\": %.1f, \"count_per_step\": %.1f}\n", k2.first, k2.second,
                v.first * ns_per_tick / (batch * steps), double(v.second) / steps);
  return 0;
}
