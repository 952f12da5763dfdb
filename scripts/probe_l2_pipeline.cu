// Probe: does a consumer that follows a producer copy chunk by chunk on the
// same B200 read the producer's fresh writes from L2, and does discarding
// them after the read save their write-back?  Diagnostic for the N=1
// colocated pass.  A writer (32 KiB tiles, chunk counters and
// flags like K1) copies src -> slab; a follower (one 256-thread CTA per SM,
// warp w takes 7 KiB rows w, w+W, ...; flag acquire per chunk) copies
// slab rows -> out, optionally discarding them from L2, concurrently on a
// high-priority stream.  Cases:
//   writer alone | follower alone on a cold slab | pass (hot slab) | pass
//   with discard | pass with the follower reading a COLD buffer instead
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/probe_l2_pipeline scripts/probe_l2_pipeline.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int64_t kRow = 7168;
constexpr int64_t kChunkRows = 1024;
constexpr int64_t kChunk = kRow * kChunkRows;  // 7 MiB
constexpr int kTile = 32768;

__device__ __forceinline__ uint64_t ld_acq(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ int g_store_policy = 0;  // 0 plain stores, 1 L2::evict_last, 2 L2::evict_first

__global__ void __launch_bounds__(256) writer(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                              unsigned* counters, uint64_t* flags, uint64_t token) {
  uint64_t pol;
  if (g_store_policy == 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const int64_t tile = blockIdx.x;
  const int64_t base = tile * (kTile / 16);
  uint4 r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k)
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[k].x), "=r"(r[k].y), "=r"(r[k].z), "=r"(r[k].w)
                 : "l"(src + base + k * 256 + threadIdx.x));
  if (g_store_policy == 0) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst + base + k * 256 + threadIdx.x),
                   "r"(r[k].x), "r"(r[k].y), "r"(r[k].z), "r"(r[k].w)
                   : "memory");
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(
                       dst + base + k * 256 + threadIdx.x),
                   "r"(r[k].x), "r"(r[k].y), "r"(r[k].z), "r"(r[k].w), "l"(pol)
                   : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int64_t c = tile * kTile / kChunk;
    unsigned prev;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(counters + c) : "memory");
    if (prev == kChunk / kTile - 1) {
      counters[c] = 0;
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flags + c), "l"(token) : "memory");
    }
  }
}

__global__ void __launch_bounds__(256) follower(const uint8_t* slab, uint8_t* out, int64_t rows,
                                                const uint64_t* flags, uint64_t token, int discard) {
  const int lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * 8;
  for (int64_t g = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); g < rows; g += W) {
    if (flags) {
      if (lane == 0)
        while (ld_acq(flags + g / kChunkRows) != token) __nanosleep(64);
      __syncwarp();
    }
    const uint4* s = reinterpret_cast<const uint4*>(slab + g * kRow);
    uint4* d = reinterpret_cast<uint4*>(out + g * kRow);
    uint4 r[14];
#pragma unroll
    for (int k = 0; k < 14; ++k)
      asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(r[k].x), "=r"(r[k].y), "=r"(r[k].z), "=r"(r[k].w)
                   : "l"(s + k * 32 + lane));
#pragma unroll
    for (int k = 0; k < 14; ++k)
      asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(d + k * 32 + lane), "r"(r[k].x),
                   "r"(r[k].y), "r"(r[k].z), "r"(r[k].w)
                   : "memory");
    if (discard)
      for (int64_t a = lane; a < kRow / 128; a += 32)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(slab + g * kRow + a * 128) : "memory");
  }
}

int main() {
  const int64_t chunks = 64;  // 448 MiB
  const int64_t bytes = chunks * kChunk, rows = chunks * kChunkRows;
  uint8_t *src, *slab, *cold, *out;
  unsigned* counters;
  uint64_t* flags;
  cudaMalloc(&src, bytes);
  cudaMalloc(&slab, bytes);
  cudaMalloc(&cold, bytes);
  cudaMalloc(&out, bytes);
  cudaMalloc(&counters, chunks * 4);
  cudaMalloc(&flags, chunks * 8);
  cudaMemset(src, 1, bytes);
  cudaMemset(cold, 2, bytes);
  cudaMemset(counters, 0, chunks * 4);
  cudaMemset(flags, 0, chunks * 8);
  int lo, hi, sms;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaStream_t sw, sf;
  cudaStreamCreateWithPriority(&sw, cudaStreamNonBlocking, lo);
  cudaStreamCreateWithPriority(&sf, cudaStreamNonBlocking, hi);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  uint64_t token = 1;
  const int tiles = (int)(bytes / kTile);
  auto run = [&](const char* name, bool w, int mode /*0 none,1 hot,2 hot+discard,3 cold*/, int reps) {
    float best = 1e9f;
    for (int it = 0; it < reps; ++it) {
      ++token;
      cudaDeviceSynchronize();
      cudaEventRecord(e0, sw);
      cudaStreamWaitEvent(sf, e0, 0);
      if (w) writer<<<tiles, 256, 0, sw>>>(reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(slab),
                                           counters, flags, token);
      if (mode)
        follower<<<sms, 256, 0, sf>>>(mode == 3 ? cold : slab, out, rows, w ? flags : nullptr, token,
                                      mode == 2);
      cudaEvent_t ef;
      cudaEventCreate(&ef);
      cudaEventRecord(ef, sf);
      cudaStreamWaitEvent(sw, ef, 0);
      cudaEventRecord(e1, sw);
      cudaEventSynchronize(e1);
      cudaEventDestroy(ef);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it > 0 && ms < best) best = ms;
    }
    std::printf("{\"case\": \"%s\", \"ms\": %.4f, \"payload_gbs\": %.1f}\n", name, best, bytes / (best * 1e-3) / 1e9);
  };
  for (int pol : {0, 1}) {
    cudaMemcpyToSymbol(g_store_policy, &pol, sizeof(pol));
    std::printf("{\"writer_stores\": \"%s\"}\n", pol ? "L2::evict_last" : "plain");
    run("writer alone (src -> slab)", true, 0, 6);
    run("follower alone, cold slab (slab -> out)", false, 3, 6);
    run("pass: writer || follower on the hot slab", true, 1, 6);
    run("pass: writer || follower on the hot slab + discard", true, 2, 6);
    run("pass: writer || follower reading a cold buffer", true, 3, 6);
  }
  // stream-ordered: does a reader right after the writer hit L2 at all?
  // (once with plain stores, once with L2::evict_last stores)
  for (int pol : {0, 1})
  for (int64_t nch : {2, 8, 16}) {
    cudaMemcpyToSymbol(g_store_policy, &pol, sizeof(pol));
    const int64_t b = nch * kChunk, r = nch * kChunkRows;
    for (int hot = 1; hot >= 0; --hot) {
      float best = 1e9f;
      for (int it = 0; it < 6; ++it) {
        cudaMemsetAsync(cold + bytes - (int64_t{256} << 20), 3, int64_t{256} << 20, sw);  // flush L2
        writer<<<(int)(b / kTile), 256, 0, sw>>>(reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(slab),
                                                  counters, flags, ++token);
        cudaEventRecord(e0, sw);
        follower<<<sms, 256, 0, sw>>>(hot ? slab : cold, out, r, nullptr, 0, 0);
        cudaEventRecord(e1, sw);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it > 0 && ms < best) best = ms;
      }
      std::printf("{\"case\": \"serial read of %lld MiB right after the write (%s stores), %s\", \"ms\": %.4f, \"payload_gbs\": %.1f}\n",
                  (long long)(b >> 20), pol ? "evict_last" : "plain", hot ? "same (hot) buffer" : "cold buffer", best,
                  b / (best * 1e-3) / 1e9);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  std::printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
