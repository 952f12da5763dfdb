// Probe: the product K1 (fsx::launch_forward, linked from build/fsx_kernels.o)
// for one small transfer, 200 launches back to back in a CUDA graph, next to
// cudaMemcpyAsync D2D of the same bytes -- the same harness as
// scripts/probe_launch_floor.cu, so the two files' numbers compare directly.
// Diagnostic only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -Ipaper_2603_12118_b200/csrc \
//        -o build/probe_k1_floor scripts/probe_k1_floor.cu build/fsx_kernels.o
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "fsx_kernels.cuh"

// the lean probe kernel of scripts/probe_launch_floor.cu (4 KiB tiles, count +
// release), here with a distinct counter and flag per launch like the product
__global__ void __launch_bounds__(256) lean_tiles(const uint4* __restrict__ s, uint4* __restrict__ d, int64_t nv,
                                                  uint32_t* counter, uint64_t* flag, uint32_t need, uint64_t token) {
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (i < nv) d[i] = __ldg(s + i);
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(counter), "r"(1u) : "memory");
  if (old + 1 != need) return;
  *counter = 0;
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flag), "l"(token) : "memory");
}

// one thread publishes a chunk flag behind a stream-ordered copy
__global__ void flag_kernel(uint64_t* dflag, uint64_t* hflag, uint64_t token) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(dflag), "l"(token) : "memory");
  if (hflag) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(hflag), "l"(token) : "memory");
}

int main() {
  const int reps = 200;
  uint8_t *s = nullptr, *d = nullptr;
  uint32_t* c = nullptr;
  uint64_t* f = nullptr;
  cudaMalloc(&s, 64 << 20);
  cudaMalloc(&d, 64 << 20);
  cudaMalloc(&c, 1 << 20);
  cudaMalloc(&f, 1 << 20);
  cudaMemset(s, 1, 64 << 20);
  cudaMemset(c, 0, 1 << 20);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fsx::preload_kernels();
  using WV = int (*)(cudaStream_t, unsigned long long, unsigned long long, unsigned int);
  void* wvp = nullptr;
  cudaDriverEntryPointQueryResult q{};
  cudaGetDriverEntryPoint("cuStreamWriteValue64", &wvp, cudaEnableDefault, &q);
  const WV wv = reinterpret_cast<WV>(wvp);
  if (!wv) return 1;
  uint64_t* hf = nullptr;
  cudaHostAlloc(&hf, 1 << 20, cudaHostAllocMapped);
  auto time_graph = [&](auto&& body) -> double {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal) != cudaSuccess) return -1;
    for (int i = 0; i < reps; ++i) body(i);
    if (cudaStreamEndCapture(st, &g) != cudaSuccess) return -2;
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) return -3;
    double best = 1e30;
    for (int t = 0; t < 5; ++t) {
      cudaGraphLaunch(ge, st);
      cudaEventRecord(e0, st);
      cudaGraphLaunch(ge, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    if (cudaGetLastError() != cudaSuccess) return -4;
    return best * 1e3 / reps;
  };
  for (int64_t n : {int64_t{64} << 10, int64_t{256} << 10, int64_t{1} << 20, int64_t{4} << 20}) {
    auto k1 = [&](int64_t unit, bool bulk) {
      return time_graph([&](int i) {
        fsx::FwdBatch b{};
        b.n = 1;
        fsx::FwdArgs& a = b.t[0];
        a.src = s;
        a.dst = d;
        a.bytes = n;
        a.chunk_bytes = n;
        a.slice = unit;
        a.chunk_units = (n + unit - 1) / unit;
        a.last_units = a.chunk_units;
        a.total_units = a.chunk_units;
        a.n_chunks = 1;
        a.vec = 16;
        a.peer = 0;
        a.counters = c + i;
        a.dflags = f + i;
        a.hflags = nullptr;
        a.token = 1000 + i;
        a.digest = nullptr;
        b.unit_off[1] = a.total_units;
        b.small = unit == 4096 ? 1 : 0;  // as fsx_forward_batch picks it (batch <= 2 MiB)
        fsx::launch_forward(b, bulk, st);
      });
    };
    const double t4 = k1(4096, false), t32 = k1(32768, false), b4 = k1(4096, true), b32 = k1(32768, true);
    const unsigned g4 = (unsigned)((n / 16 + 255) / 256);
    const double lean_same = time_graph([&](int i) {
      lean_tiles<<<g4, 256, 0, st>>>(reinterpret_cast<const uint4*>(s), reinterpret_cast<uint4*>(d), n / 16, c, f,
                                     g4, 1000 + i);
    });
    const double lean_distinct = time_graph([&](int i) {
      lean_tiles<<<g4, 256, 0, st>>>(reinterpret_cast<const uint4*>(s), reinterpret_cast<uint4*>(d), n / 16, c + 64 * i,
                                     f + 64 * i, g4, 1000 + i);
    });
    std::printf("{\"bytes\": %lld, \"lean_4k_same_counter_us\": %.3f, \"lean_4k_distinct_counters_us\": %.3f}\n",
                (long long)n, lean_same, lean_distinct);
    const double mc = time_graph([&](int) { cudaMemcpyAsync(d, s, n, cudaMemcpyDeviceToDevice, st); });
    // the copy-engine form of K1 (FSX_FWD_DMA): the copy, then the chunk flag
    // by a stream memory operation (device flag; + the mapped host mirror)
    const double dma = time_graph([&](int i) {
      cudaMemcpyAsync(d, s, n, cudaMemcpyDeviceToDevice, st);
      wv(st, reinterpret_cast<uintptr_t>(f + i), 1000 + i, 0);
    });
    const double dma_host = time_graph([&](int i) {
      cudaMemcpyAsync(d, s, n, cudaMemcpyDeviceToDevice, st);
      wv(st, reinterpret_cast<uintptr_t>(f + i), 1000 + i, 0);
      wv(st, reinterpret_cast<uintptr_t>(hf + i), 1000 + i, 0);
    });
    // the copy, then a one-thread flag kernel behind it (stream order)
    const double dma_fk = time_graph([&](int i) {
      cudaMemcpyAsync(d, s, n, cudaMemcpyDeviceToDevice, st);
      flag_kernel<<<1, 1, 0, st>>>(f + i, nullptr, 1000 + i);
    });
    const double dma_fk_host = time_graph([&](int i) {
      cudaMemcpyAsync(d, s, n, cudaMemcpyDeviceToDevice, st);
      flag_kernel<<<1, 1, 0, st>>>(f + i, hf + i, 1000 + i);
    });
    std::printf("{\"bytes\": %lld, \"k1_tile_4k_us\": %.3f, \"k1_tile_32k_us\": %.3f, \"k1_bulk_4k_us\": %.3f, "
                "\"k1_bulk_32k_us\": %.3f, \"dma_memop_flag_us\": %.3f, \"dma_memop_flag_host_us\": %.3f, "
                "\"dma_flag_kernel_us\": %.3f, \"dma_flag_kernel_host_us\": %.3f, \"memcpy_us\": %.3f}\n",
                (long long)n, t4, t32, b4, b32, dma, dma_host, dma_fk, dma_fk_host, mc);
  }
  return 0;
}
