// Throughput of the C++ SidecarFabric engine (include/fsx/fabric.hpp) through
// the reference-facing API: SidecarFabric::send_payload (sidecar.hpp:367-370)
// of config-B video embeddings (117,440,512 B each) that already live on the
// producer GPU, delivered to
//   raw   -- register_interest_raw + ack_raw (zero copy: the consumer reads
//            the slab in place, sidecar.hpp:276-290), and
//   chunk -- register_interest with a ChunkCallback (owned host vector:
//            D2H copy + dg64 verification, sidecar.hpp:527-563).
// Virtual event loop; every send waits for its bytes to land (reference
// semantics).  Prints one JSON line per mode.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <vector>

#include "fsx/fabric.hpp"

extern "C" {
#include "fsx_oracle.h"
}

using namespace fsx;

int main(int argc, char** argv) {
  const int64_t n = 117440512;
  const int items = argc > 1 ? std::atoi(argv[1]) : 16;
  std::map<int, int> topo{{0, 0}, {1, 0}};
  void* d = nullptr;
  if (cudaMalloc(&d, n) != cudaSuccess) return 2;
  std::vector<uint8_t> host(n);
  or_synth_payload_into(or_payload_seed("req-000000/r0000", 16, 0), host.data(), n);
  cudaMemcpy(d, host.data(), n, cudaMemcpyHostToDevice);
  // modes: 0 device payload -> raw interest (zero copy), 1 device payload ->
  // ChunkCallback (owned vector), 2 HOST span (the reference executors' own
  // send of a std::vector, pageable) -> raw interest, 3 host span -> ChunkCallback
  // 4 device payload -> early-start interest (segment + chunk flags handed
  // over inside the send event; the consumer waits on the flags itself)
  static const char* kModes[] = {"raw_zero_copy", "chunk_callback_owned_vector", "host_span_raw",
                                 "host_span_chunk_callback", "early_start_interest"};
  for (int mode = 0; mode < 5; ++mode) {
    EventLoop k;
    SidecarConfig cfg;
    cfg.arena_bytes = 2 * n + 4096;
    cfg.device_chunk_bytes = 7340032;
    SidecarFabric f(k, topo, cfg);
    int64_t delivered = 0;
    double send_s = 0;  // event-thread time inside send()
    auto one = [&](int i) {
      const std::string id = "req-" + std::to_string(i) + "/r0000";
      if (mode == 4) {
        f.register_interest_early(1, id, [&](const ForwardEnvelope& env, int64_t off,
                                             const SidecarFabric::ChunkFlags& c) {
          if (c.n_chunks > 0) fsx_wait(f.handle(), 1, c.flag_base, c.n_chunks, c.token, -1);
          delivered += env.chunk_bytes;
          f.ack_raw(1, off);
        });
      } else if (mode % 2 == 0) {
        f.register_interest_raw(1, id, [&](const ForwardEnvelope& env, int64_t off) {
          delivered += env.chunk_bytes;
          f.ack_raw(1, off);
        });
      } else {
        f.register_interest(1, id, [&](const ForwardEnvelope& env, std::vector<uint8_t> b) {
          delivered += static_cast<int64_t>(b.size());
        });
      }
      k.post("send", [&, id] {
        const auto a = std::chrono::steady_clock::now();
        f.send_payload("req", DataRef{id, n, false}, 0, 1,
                       std::span<const uint8_t>((mode < 2 || mode == 4) ? static_cast<const uint8_t*>(d)
                                                                         : host.data(), n));
        send_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
      });
      k.run_until_idle();
    };
    one(-1);  // warm-up
    delivered = 0;
    send_s = 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < items; ++i) one(i);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("{\"mode\": \"%s\", \"items\": %d, \"bytes\": %lld, \"gbs\": %.2f, \"ms_per_item\": %.3f,"
                " \"send_ms_per_item\": %.3f, \"integrity_errors\": %lld}\n",
                kModes[mode], items,
                (long long)delivered, delivered / s / 1e9, s / items * 1e3, send_s / items * 1e3,
                (long long)f.stats().integrity_errors);
  }
  cudaFree(d);

  // Config C through the same API: per decode step every active request's
  // thinker sends one hidden-state row (host span, streaming ref, seq = step)
  // and the talker's ChunkCallback receives it (executor_sim.hpp:370-381,
  // 556-562).  Reported as microseconds per step and messages per second.
  // device mode: the thinker's rows already on its GPU (the real deployment),
  // sent from device memory to raw (zero-copy) talker consumers, the producer
  // keeping each step's rows until delivery (async_borrowed_sources)
  for (int mode = 0; mode < 3; ++mode) {
    const int row = mode == 1 ? 2048 : 7168;
    const bool device = mode == 2;
    const int batch = 32, steps = 200;
    EventLoop k;
    SidecarConfig cfg;
    cfg.async_borrowed_sources = device;
    SidecarFabric f(k, topo, cfg);
    void* drow = nullptr;
    if (device && cudaMalloc(&drow, (size_t)row * batch) != cudaSuccess) return 2;
    std::vector<uint8_t> rowbuf(row);
    or_synth_payload_into(7, rowbuf.data(), row);
    for (int r = 0; r < batch && device; ++r)
      cudaMemcpy(static_cast<uint8_t*>(drow) + (size_t)r * row, rowbuf.data(), row, cudaMemcpyHostToDevice);
    // a pageable-source cudaMemcpy may return before its DMA lands: the rows
    // must be complete before a send hands them to the (unordered) lane kernel
    if (device) cudaDeviceSynchronize();
    int64_t got = 0;
    for (int r = 0; r < batch; ++r) {
      if (device)
        f.register_interest_raw(1, "req-" + std::to_string(r) + "/r0001",
                                [&](const ForwardEnvelope& env, int64_t off) {
                                  got += env.chunk_bytes;
                                  f.ack_raw(1, off);
                                });
      else
        f.register_interest(1, "req-" + std::to_string(r) + "/r0001",
                            [&](const ForwardEnvelope&, std::vector<uint8_t> b) { got += (int64_t)b.size(); });
    }
    double send_s = 0, deliver_s = 0;  // host time split: the sends, then the deliveries
    auto step = [&](int s) {
      const auto a = std::chrono::steady_clock::now();
      for (int r = 0; r < batch; ++r)
        f.send("req-" + std::to_string(r), DataRef{"req-" + std::to_string(r) + "/r0001", 0, true}, 0, 1,
               std::span<const uint8_t>(device ? static_cast<const uint8_t*>(drow) + (size_t)r * row
                                               : rowbuf.data(),
                                        row),
               s, false);
      const auto b = std::chrono::steady_clock::now();
      k.run_until_idle();
      send_s += std::chrono::duration<double>(b - a).count();
      deliver_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - b).count();
    };
    for (int s = 0; s < 10; ++s) step(s);
    got = 0;
    send_s = deliver_s = 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (int s = 10; s < 10 + steps; ++s) step(s);
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("{\"mode\": \"%s\", \"rows_per_step\": %d, \"row_bytes\": %d, "
                "\"us_per_step\": %.1f, \"send_us_per_step\": %.1f, \"deliver_us_per_step\": %.1f, "
                "\"msgs_per_s\": %.0f, \"bytes_ok\": %s}\n",
                device ? "stream_device_rows_raw_interest" : "stream_host_span_chunk_callback", batch, row,
                sec / steps * 1e6, send_s / steps * 1e6, deliver_s / steps * 1e6,
                batch * steps / sec,
                got == (int64_t)batch * steps * row ? "true" : "false");
    if (drow) cudaFree(drow);
  }
  return 0;
}
