// Probe: how fast can an SM kernel copy HBM->HBM on this B200, next to
// cudaMemcpyAsync D2D?  Plain grid (one CTA per tile, no persistence, no flags)
// with 16-byte and 32-byte vectors and several unrolls.  Diagnostic only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/probe_sm_copy scripts/probe_sm_copy.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

template <int U>
__global__ void __launch_bounds__(256) copy16(const uint4* __restrict__ s, uint4* __restrict__ d, int64_t n) {
  const int64_t base = (int64_t)blockIdx.x * 256 * U;
  uint4 r[U];
#pragma unroll
  for (int k = 0; k < U; ++k) {
    const int64_t i = base + k * 256 + threadIdx.x;
    if (i < n) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                            : "=r"(r[k].x), "=r"(r[k].y), "=r"(r[k].z), "=r"(r[k].w) : "l"(s + i));
  }
#pragma unroll
  for (int k = 0; k < U; ++k) {
    const int64_t i = base + k * 256 + threadIdx.x;
    if (i < n) asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(d + i),
                            "r"(r[k].x), "r"(r[k].y), "r"(r[k].z), "r"(r[k].w) : "memory");
  }
}

template <int U>
__global__ void __launch_bounds__(256) copy_persist(const uint4* __restrict__ s, uint4* __restrict__ d, int64_t n) {
  for (int64_t base = (int64_t)blockIdx.x * 256 * U; base < n; base += (int64_t)gridDim.x * 256 * U) {
    uint4 r[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t i = base + k * 256 + threadIdx.x;
      if (i < n) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                              : "=r"(r[k].x), "=r"(r[k].y), "=r"(r[k].z), "=r"(r[k].w) : "l"(s + i));
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t i = base + k * 256 + threadIdx.x;
      if (i < n) asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(d + i),
                              "r"(r[k].x), "r"(r[k].y), "r"(r[k].z), "r"(r[k].w) : "memory");
    }
  }
}

template <typename F>
float time_it(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  const int64_t bytes = int64_t{469762048};
  void *s, *d;
  cudaMalloc(&s, bytes);
  cudaMalloc(&d, bytes);
  cudaMemset(s, 1, bytes);
  const int64_t nv = bytes / 16;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto gbs = [&](float ms) { return 2.0 * bytes / (ms * 1e-3) / 1e9; };
  printf("{\"memcpy_d2d\": %.1f", gbs(time_it([&] { cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice); }, 20)));
  printf(", \"grid_u4\": %.1f", gbs(time_it([&] { copy16<4><<<(nv + 1023) / 1024, 256>>>((const uint4*)s, (uint4*)d, nv); }, 20)));
  printf(", \"grid_u8\": %.1f", gbs(time_it([&] { copy16<8><<<(nv + 2047) / 2048, 256>>>((const uint4*)s, (uint4*)d, nv); }, 20)));
  printf(", \"grid_u16\": %.1f", gbs(time_it([&] { copy16<16><<<(nv + 4095) / 4096, 256>>>((const uint4*)s, (uint4*)d, nv); }, 20)));
  for (int per : {2, 4, 8}) {
    printf(", \"persist_u8_%d\": %.1f", per,
           gbs(time_it([&] { copy_persist<8><<<sms * per, 256>>>((const uint4*)s, (uint4*)d, nv); }, 20)));
  }
  printf("}\n");
  return 0;
}
