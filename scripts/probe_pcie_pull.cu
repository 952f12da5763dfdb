// Probe: how fast can an SM pull small messages out of mapped pinned host
// memory (the small-message lane's data path)?  Diagnostic only.
//   latency     one thread, 64 dependent 8-byte volatile loads (PCIe round trip)
//   regs C x T  C CTAs x T threads, each lane 4 x 16 B volatile loads per round,
//               pulling `bytes` (contiguous) into device memory
//   bulk        one CTA, one elected thread: cp.async.bulk host->shared in
//               16 KiB pieces (mbarrier complete_tx), up to 192 KiB in flight,
//               then cp.async.bulk shared->global
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/probe_pcie_pull scripts/probe_pcie_pull.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void latency_kernel(const uint64_t* h, int n, uint64_t* out) {
  uint64_t idx = 0;
  const uint64_t t0 = gtime();
  for (int i = 0; i < n; ++i) {
    uint64_t v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(h + idx) : "memory");
    idx = (v + i) & 7;
  }
  out[0] = gtime() - t0;
  out[1] = idx;
}

__global__ void regs_kernel(const uint4* __restrict__ h, uint4* __restrict__ d, int nv) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int stride = gridDim.x * blockDim.x;
  for (int base = tid; base < nv; base += 4 * stride) {
    uint4 r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (base + k * stride < nv)
        asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[k].x), "=r"(r[k].y), "=r"(r[k].z), "=r"(r[k].w)
                     : "l"(h + base + k * stride));
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (base + k * stride < nv) d[base + k * stride] = r[k];
  }
}

__global__ void bulk_kernel(const uint8_t* h, uint8_t* d, int bytes) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[12];
  if (threadIdx.x != 0) return;
  constexpr int kPiece = 16384, kMax = 12;
  const int pieces = (bytes + kPiece - 1) / kPiece;
  for (int p0 = 0; p0 < pieces; p0 += kMax) {
    const int np = min(kMax, pieces - p0);
    for (int i = 0; i < np; ++i) {
      const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[i]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < np; ++i) {
      const int off = (p0 + i) * kPiece;
      const uint32_t len = (uint32_t)min(kPiece, bytes - off);
      const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[i]);
      const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm + i * kPiece);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(len) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s),
          "l"(h + off), "r"(len), "r"(b)
          : "memory");
    }
    for (int i = 0; i < np; ++i) {
      const int off = (p0 + i) * kPiece;
      const uint32_t len = (uint32_t)min(kPiece, bytes - off);
      const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[i]);
      const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm + i * kPiece);
      asm volatile(
          "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(b)
          : "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d + off), "r"(s), "r"(len)
                   : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    for (int i = 0; i < np; ++i) {
      const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[i]);
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(b));
    }
  }
}

int main() {
  uint8_t* h = nullptr;
  cudaHostAlloc(&h, 8 << 20, cudaHostAllocMapped | cudaHostAllocPortable);
  for (int i = 0; i < (8 << 20); ++i) h[i] = (uint8_t)i;
  uint8_t* d = nullptr;
  uint64_t* out = nullptr;
  cudaMalloc(&d, 8 << 20);
  cudaMalloc(&out, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  latency_kernel<<<1, 1>>>(reinterpret_cast<uint64_t*>(h), 64, out);
  latency_kernel<<<1, 1>>>(reinterpret_cast<uint64_t*>(h), 64, out);
  uint64_t lat[2];
  cudaMemcpy(lat, out, 16, cudaMemcpyDeviceToHost);
  std::printf("{\"case\": \"latency\", \"ns_per_dependent_load\": %.1f}\n", lat[0] / 64.0);
  cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384);
  auto time_it = [&](auto&& launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int t = 0; t < 20; ++t) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    return best * 1e3;
  };
  const float empty = time_it([&] { regs_kernel<<<1, 32>>>(nullptr, nullptr, 0); });
  std::printf("{\"case\": \"empty launch\", \"us\": %.2f}\n", empty);
  for (int bytes : {7168, 65536, 229376, 1048576}) {
    const int nv = bytes / 16;
    for (int ctas : {1, 2, 4, 8}) {
      for (int thr : {512, 1024}) {
        const float us = time_it([&] {
          regs_kernel<<<ctas, thr>>>(reinterpret_cast<const uint4*>(h), reinterpret_cast<uint4*>(d), nv);
        });
        std::printf("{\"case\": \"regs\", \"bytes\": %d, \"ctas\": %d, \"threads\": %d, \"us\": %.2f, \"gbs\": %.1f}\n",
                    bytes, ctas, thr, us, bytes / (us * 1e3));
      }
    }
    const float us = time_it([&] { bulk_kernel<<<1, 32, 12 * 16384>>>(h, d, bytes); });
    std::printf("{\"case\": \"bulk\", \"bytes\": %d, \"us\": %.2f, \"gbs\": %.1f}\n", bytes, us, bytes / (us * 1e3));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) std::printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
  }
  return 0;
}
