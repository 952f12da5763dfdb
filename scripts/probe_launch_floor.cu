// Probe: where does a small K1 transfer's ~2.7 us go (profiles/k1_sweep_*,
// VERDICT r01 "K1 small-transfer floor")?  Back-to-back launches captured in a
// CUDA graph (200 per replay), CUDA-event timed, per launch:
//   empty          <<<1, 32>>> no work: the graph's kernel-to-kernel floor
//   copy           one CTA per 32 KiB tile (256 thr x 8 x 16 B), no flags
//   copy+count     + __syncthreads + atom.add.acq_rel.gpu + st.release.gpu (K1's protocol)
//   copy+count+pdl the same launched with programmatic stream serialization
//                  (griddepcontrol.wait before the loads, launch_dependents after)
//   small tiles    one CTA per 4 KiB (256 thr x 1 x 16 B) + count
//   memcpy         cudaMemcpyAsync D2D of the same bytes
// Diagnostic only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/probe_launch_floor scripts/probe_launch_floor.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void empty_kernel() {}

template <int V, bool COUNT, bool PDL>
__global__ void __launch_bounds__(256) copy_tiles(const uint4* __restrict__ s, uint4* __restrict__ d, int64_t nv,
                                                  uint32_t* counter, uint64_t* flag, uint32_t need, uint64_t token) {
  if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t base = (int64_t)blockIdx.x * 256 * V;
  uint4 r[V];
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int64_t i = base + k * 256 + threadIdx.x;
    if (i < nv) r[k] = __ldg(s + i);
  }
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int64_t i = base + k * 256 + threadIdx.x;
    if (i < nv) d[i] = r[k];
  }
  if (PDL) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (!COUNT) return;
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(counter), "r"(1u) : "memory");
  if (old + 1 != need) return;
  *counter = 0;
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flag), "l"(token) : "memory");
}

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      std::printf("{\"error\": \"%s at %d\"}\n", cudaGetErrorString(e_), __LINE__); \
      return 1;                                                                \
    }                                                                          \
  } while (0)

template <int V, bool COUNT, bool PDL>
static cudaError_t launch(cudaStream_t st, const uint4* s, uint4* d, int64_t bytes, uint32_t* c, uint64_t* f) {
  const int64_t nv = bytes / 16;
  const unsigned grid = (unsigned)((nv + 256 * V - 1) / (256 * V));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = PDL ? at : nullptr;
  cfg.numAttrs = PDL ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, copy_tiles<V, COUNT, PDL>, s, d, nv, c, f, grid, (uint64_t)1);
}

int main() {
  const int reps = 200;
  uint4 *s = nullptr, *d = nullptr;
  uint32_t* c = nullptr;
  uint64_t* f = nullptr;
  CK(cudaMalloc(&s, 64 << 20));
  CK(cudaMalloc(&d, 64 << 20));
  CK(cudaMalloc(&c, 4096));
  CK(cudaMalloc(&f, 4096));
  CK(cudaMemset(s, 1, 64 << 20));
  CK(cudaMemset(c, 0, 4096));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto time_graph = [&](auto&& body) -> double {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal) != cudaSuccess) return -1;
    for (int i = 0; i < reps; ++i) body();
    if (cudaStreamEndCapture(st, &g) != cudaSuccess) return -1;
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) return -1;
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
    if (cudaGetLastError() != cudaSuccess) return -1;
    return best * 1e3 / reps;
  };
  std::printf("{\"case\": \"empty\", \"us\": %.3f}\n", time_graph([&] { empty_kernel<<<1, 32, 0, st>>>(); }));
  for (int64_t n : {int64_t{64} << 10, int64_t{256} << 10, int64_t{1} << 20, int64_t{4} << 20}) {
    const double cp = time_graph([&] { launch<8, false, false>(st, s, d, n, c, f); });
    const double cc = time_graph([&] { launch<8, true, false>(st, s, d, n, c, f); });
    const double pdl = time_graph([&] { launch<8, true, true>(st, s, d, n, c, f); });
    const double sm = time_graph([&] { launch<1, true, false>(st, s, d, n, c, f); });
    const double smp = time_graph([&] { launch<1, true, true>(st, s, d, n, c, f); });
    const double mc = time_graph([&] { cudaMemcpyAsync(d, s, n, cudaMemcpyDeviceToDevice, st); });
    std::printf("{\"bytes\": %lld, \"copy_us\": %.3f, \"copy_count_us\": %.3f, \"copy_count_pdl_us\": %.3f, "
                "\"tiles4k_count_us\": %.3f, \"tiles4k_count_pdl_us\": %.3f, \"memcpy_us\": %.3f}\n",
                (long long)n, cp, cc, pdl, sm, smp, mc);
  }
  return 0;
}
