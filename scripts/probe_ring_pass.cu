// Probe: the N=1 colocated pass through an L2-sized receive RING instead of a
// whole-item slab.  A persistent writer (K1 analogue: 32 KiB
// tiles, chunk counters, a ready generation per ring slot) copies src -> ring
// slot g % R for chunk g, waiting until the follower has released the slot's
// previous use; a persistent follower (merge analogue: one CTA per SM, warp per
// 7 KiB row, rows in order) waits for the chunk, copies ring rows -> out and
// releases the slot once all of the chunk's rows are out.  Rewritten dirty
// lines of a slot that stays in L2 never go back to DRAM, so the pass should
// move ~src + out only.  Compared with the same writer/follower over a full
// slab (no reuse, today's layout).  Every spin has a %globaltimer timeout: a
// stuck pass reports "timeout" instead of hanging.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/probe_ring_pass scripts/probe_ring_pass.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int64_t kRow = 7168;
constexpr int64_t kChunkRows = 1024;
constexpr int64_t kChunk = kRow * kChunkRows;  // 7 MiB
constexpr int kTile = 32768;
constexpr int kTilesPerChunk = (int)(kChunk / kTile);  // 224
constexpr uint64_t kTimeoutNs = 2000000000ull;        // 2 s

__device__ __forceinline__ uint64_t now_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ int g_timeout = 0;

// wait until *p >= want; false on timeout
__device__ bool wait_ge(const uint32_t* p, uint32_t want) {
  const uint64_t t0 = now_ns();
  while (ld_acq(p) < want) {
    if (now_ns() - t0 > kTimeoutNs || *(volatile int*)&g_timeout) {
      atomicExch(&g_timeout, 1);
      return false;
    }
    __nanosleep(64);
  }
  return true;
}

// ring == nullptr: full slab (chunk g at g * kChunk, no backpressure)
__global__ void __launch_bounds__(256) writer(const uint4* __restrict__ src, uint8_t* slab, int ring_slots,
                                              int64_t chunks, unsigned* counters, uint32_t* ready_gen,
                                              const uint32_t* released_gen) {
  __shared__ int ok;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const int64_t tiles = chunks * kTilesPerChunk;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t g = t / kTilesPerChunk;
    const int64_t slot = ring_slots ? g % ring_slots : g;
    if (threadIdx.x == 0) {
      ok = 1;
      if (ring_slots && g >= ring_slots) ok = wait_ge(released_gen + slot, (uint32_t)(g / ring_slots));
    }
    __syncthreads();
    if (!ok) return;
    const int64_t in_chunk = (t % kTilesPerChunk) * kTile;
    const uint4* s = src + (g * kChunk + in_chunk) / 16;
    uint4* d = reinterpret_cast<uint4*>(slab + slot * kChunk + in_chunk);
    uint4 r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                   : "=r"(r[k].x), "=r"(r[k].y), "=r"(r[k].z), "=r"(r[k].w)
                   : "l"(s + k * 256 + threadIdx.x), "l"(pol));
#pragma unroll
    for (int k = 0; k < 8; ++k) d[k * 256 + threadIdx.x] = r[k];
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned prev;
      asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(counters + g) : "memory");
      if (prev == kTilesPerChunk - 1) st_rel(ready_gen + slot, (uint32_t)(ring_slots ? g / ring_slots + 1 : 1));
    }
  }
}

__global__ void __launch_bounds__(256) follower(const uint8_t* slab, int ring_slots, uint8_t* out, int64_t chunks,
                                                const uint32_t* ready_gen, uint32_t* released_gen,
                                                unsigned* merged) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const int lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * 8;
  const int64_t rows = chunks * kChunkRows;
  int64_t waited = -1;
  for (int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); r < rows; r += W) {
    const int64_t g = r / kChunkRows;
    const int64_t slot = ring_slots ? g % ring_slots : g;
    if (g != waited) {
      int ok = 1;
      if (lane == 0) ok = wait_ge(ready_gen + slot, (uint32_t)(ring_slots ? g / ring_slots + 1 : 1));
      ok = __shfl_sync(0xffffffffu, ok, 0);
      if (!ok) return;
      waited = g;
    }
    const uint4* s = reinterpret_cast<const uint4*>(slab + slot * kChunk + (r % kChunkRows) * kRow);
    uint4* d = reinterpret_cast<uint4*>(out + r * kRow);
    uint4 v[14];
#pragma unroll
    for (int k = 0; k < 14; ++k) v[k] = s[k * 32 + lane];
#pragma unroll
    for (int k = 0; k < 14; ++k)
      asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(
                       d + k * 32 + lane),
                   "r"(v[k].x), "r"(v[k].y), "r"(v[k].z), "r"(v[k].w), "l"(pol)
                   : "memory");
    __syncwarp();
    if (ring_slots && lane == 0) {
      unsigned prev;
      asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(merged + g) : "memory");
      if (prev == kChunkRows - 1) st_rel(released_gen + slot, (uint32_t)(g / ring_slots + 1));
    }
  }
}

int main() {
  const int64_t chunks = 64;  // 448 MiB: the config-B pass is 64 chunks of 7 MiB
  const int64_t bytes = chunks * kChunk;
  uint8_t *src, *slab, *out;
  unsigned *counters, *merged;
  uint32_t *ready, *released;
  cudaMalloc(&src, bytes);
  cudaMalloc(&slab, bytes);
  cudaMalloc(&out, bytes);
  cudaMalloc(&counters, chunks * 4);
  cudaMalloc(&merged, chunks * 4);
  cudaMalloc(&ready, chunks * 4);
  cudaMalloc(&released, chunks * 4);
  cudaMemset(src, 7, bytes);
  int lo, hi, sms;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaStream_t sw, sf;
  cudaStreamCreateWithPriority(&sw, cudaStreamNonBlocking, lo);
  cudaStreamCreateWithPriority(&sf, cudaStreamNonBlocking, hi);
  cudaEvent_t e0, e1, ef;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&ef);
  auto run = [&](int ring, int wgrid, int reps) {
    float best = 1e9f, sum = 0;
    int n = 0, timeout = 0;
    for (int it = 0; it < reps; ++it) {
      cudaMemsetAsync(counters, 0, chunks * 4, sw);
      cudaMemsetAsync(merged, 0, chunks * 4, sw);
      cudaMemsetAsync(ready, 0, chunks * 4, sw);
      cudaMemsetAsync(released, 0, chunks * 4, sw);
      cudaStreamSynchronize(sw);
      cudaEventRecord(e0, sw);
      cudaStreamWaitEvent(sf, e0, 0);
      // the follower first: its one CTA per SM is resident before the writer's
      follower<<<sms, 256, 0, sf>>>(slab, ring, out, chunks, ready, released, merged);
      writer<<<wgrid, 256, 0, sw>>>(reinterpret_cast<const uint4*>(src), slab, ring, chunks, counters, ready,
                                    released);
      cudaEventRecord(ef, sf);
      cudaStreamWaitEvent(sw, ef, 0);
      cudaEventRecord(e1, sw);
      cudaEventSynchronize(e1);
      int to = 0;
      cudaMemcpyFromSymbol(&to, g_timeout, sizeof(int));
      if (to) {
        timeout = 1;
        int z = 0;
        cudaMemcpyToSymbol(g_timeout, &z, sizeof(int));
        continue;
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it > 0) {
        best = ms < best ? ms : best;
        sum += ms;
        ++n;
      }
    }
    std::printf("{\"ring_slots\": %d, \"ring_mib\": %lld, \"writer_ctas\": %d, \"best_ms\": %.4f, \"mean_ms\": %.4f, "
                "\"payload_gbs\": %.1f, \"timeout\": %s}\n",
                ring, (long long)(ring * kChunk >> 20), wgrid, best, n ? sum / n : 0.f,
                bytes / (best * 1e-3) / 1e9, timeout ? "true" : "false");
  };
  // full slab (no reuse), writer as a persistent grid of 2 and 3 CTAs per SM
  run(0, sms * 2, 8);
  run(0, sms * 3, 8);
  for (int ring : {4, 8, 12, 16, 24})
    for (int per : {2, 3}) run(ring, sms * per, 8);
  // correctness of the last ring run: out == src (all 7s)
  uint8_t probe[4] = {0};
  cudaMemcpy(probe, out + bytes - 4, 4, cudaMemcpyDeviceToHost);
  cudaError_t e = cudaDeviceSynchronize();
  std::printf("{\"status\": \"%s\", \"last_bytes_ok\": %s}\n", cudaGetErrorString(e),
              probe[0] == 7 && probe[3] == 7 ? "true" : "false");
  return e == cudaSuccess ? 0 : 1;
}
