// Probe: host memcpy bandwidth of a 112 MiB pageable span (the reference
// executors' send of a std::vector) into pinned staging memory, by thread
// count -- the bound on how fast a borrowed pageable span can be copied out
// before send() returns (sidecar.hpp:302 borrows the span for the call only).
// Diagnostic only.
//   g++ -O2 -std=c++17 -I/usr/local/cuda/include -o build/probe_host_copy scripts/probe_host_copy.cpp \
//       -L/usr/local/cuda/lib64 -lcudart -lpthread
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

int main() {
  const size_t n = 117440512;
  std::vector<uint8_t> src(n);
  for (size_t i = 0; i < n; ++i) src[i] = (uint8_t)(i * 131);
  uint8_t* pinned = nullptr;
  if (cudaHostAlloc(&pinned, n, cudaHostAllocDefault) != cudaSuccess) return 2;
  std::vector<uint8_t> pageable(n, 1);
  const unsigned hw = std::thread::hardware_concurrency();
  for (int dst_kind = 0; dst_kind < 2; ++dst_kind) {
    uint8_t* dst = dst_kind ? pageable.data() : pinned;
    for (unsigned t : {1u, 2u, 4u, 8u, 12u, 16u, 24u, 32u}) {
      if (t > hw) break;
      double best = 1e30;
      for (int rep = 0; rep < 5; ++rep) {
        const auto a = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        const size_t per = (n / t + 63) / 64 * 64;
        for (unsigned k = 0; k < t; ++k)
          th.emplace_back([&, k] {
            const size_t b = k * per, e = std::min(n, b + per);
            if (e > b) std::memcpy(dst + b, src.data() + b, e - b);
          });
        for (auto& x : th) x.join();
        best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count());
      }
      std::printf("{\"dst\": \"%s\", \"threads\": %u, \"hw_threads\": %u, \"ms\": %.3f, \"gbs\": %.1f}\n",
                  dst_kind ? "pageable" : "pinned", t, hw, best * 1e3, n / best / 1e9);
    }
  }
  cudaFreeHost(pinned);
  return 0;
}
