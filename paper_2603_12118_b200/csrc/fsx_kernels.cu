// fsx_kernels.cu -- sm_100a kernels of the sidecar data plane.
//
//   K0 synth_kernel      synth_payload_into (common.hpp:247-259) on the device
//   K1 forward_kernel    payload placement of SidecarFabric::send/try_place_local
//                        (sidecar.hpp:302-347, 465-483) as a chunked 16-byte push
//                        into the consumer slab with per-chunk completion flags
//   K3 merge_scan_kernel + merge_copy_kernel
//                        the consumer-side multimodal merge (derived contract,
//                        SURVEY.md 8a-8; record_replay.hpp:404-416 slot order)
//   flag kernels         set / wait on chunk flags (release/acquire, sys scope)
//
// Everything here is integer byte movement: rows are opaque 16-byte vectors,
// never converted through a floating-point type, so bf16 NaN/Inf patterns in the
// synthetic payloads survive bit for bit.  No tensor cores: nothing is a
// contraction.  All kernels are HBM- or NVLink-bound; see DESIGN.md.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "fsx_kernels.cuh"

namespace fsx {
namespace kern {

constexpr int kFwdThreads = 256;
// L2 policy of the follow merge's prompt-row stores (l2_policy: 0 normal,
// 1 evict_first, 2 evict_last); FSX_FOLLOW_OUT_POLICY selects at build time
#ifndef FSX_FOLLOW_OUT_POLICY
#define FSX_FOLLOW_OUT_POLICY 1
#endif
constexpr int kFollowOutPolicy = FSX_FOLLOW_OUT_POLICY;
constexpr int kTmaTileBytes = 32768;  // K1 bulk-copy tile (forward_tma_kernel)
constexpr int kMaxDevices = 64;       // per-device launch attributes
// K1 variants: <vectors per lane per batch, min CTAs per SM>.  0: 16 x 16 B
// (8 KiB per warp batch, 2 CTAs/SM), 1: 8 x 16 B at 4 CTAs/SM (register cap 64).
constexpr int kMergeThreads = 256;
constexpr int kMergeUnroll = 16;  // 32 lanes x 16 x 16 B = 8 KiB of a row per batch
constexpr int kScanThreads = 1024;
constexpr int kScanRounds = 16;  // 1024 threads x 16 = 16384 token ids per round

// ---------------------------------------------------------------------------
// PTX helpers

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Coherent streaming load: used where the data may have been written by a
// peer GPU during this kernel's lifetime (early-start merge).
__device__ __forceinline__ uint4 ld_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// L2 eviction-priority policies (createpolicy) for the .L2::cache_hint forms.
__device__ __forceinline__ uint64_t l2_policy(int which) {
  uint64_t p;
  if (which == 2)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else if (which == 1)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint4 ld_nc_v4_pol(const void* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ void st_v4_pol(void* p, const uint4& v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}

// 32-byte vectors: sm_100 has 256-bit global loads/stores (LDG/STG .256).
struct alignas(32) v8u32 {
  uint4 lo, hi;
};

__device__ __forceinline__ v8u32 ld_nc_v8_pol(const void* p, uint64_t pol) {
  v8u32 r;
  asm volatile(
      "ld.global.nc.L1::no_allocate.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
      : "=r"(r.lo.x), "=r"(r.lo.y), "=r"(r.lo.z), "=r"(r.lo.w), "=r"(r.hi.x), "=r"(r.hi.y),
        "=r"(r.hi.z), "=r"(r.hi.w)
      : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ void st_v8_pol(void* p, const v8u32& v, uint64_t pol) {
  asm volatile(
      "st.global.L1::no_allocate.L2::cache_hint.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8}, %9;" ::"l"(p),
      "r"(v.lo.x), "r"(v.lo.y), "r"(v.lo.z), "r"(v.lo.w), "r"(v.hi.x), "r"(v.hi.y), "r"(v.hi.z),
      "r"(v.hi.w), "l"(pol)
      : "memory");
}

// Loads/stores of one V-byte vector (V = 16 or 32) with L2 policies.
template <int V>
struct VecIO;
template <>
struct VecIO<16> {
  using T = uint4;
  static __device__ __forceinline__ T ld(const void* p, uint64_t pol) { return ld_nc_v4_pol(p, pol); }
  static __device__ __forceinline__ void st(void* p, const T& v, uint64_t pol) { st_v4_pol(p, v, pol); }
};
template <>
struct VecIO<32> {
  using T = v8u32;
  static __device__ __forceinline__ T ld(const void* p, uint64_t pol) { return ld_nc_v8_pol(p, pol); }
  static __device__ __forceinline__ void st(void* p, const T& v, uint64_t pol) { st_v8_pol(p, v, pol); }
};

__device__ __forceinline__ void st_v4(void* p, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void st_release_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Device spin on a completion flag.  A flag that never arrives (a producer
// that died, or a kernel the spinning CTAs keep from being scheduled) would
// hang the GPU, so after FSX_SPIN_TIMEOUT_S seconds the kernel traps: the
// launch fails with an error the host sees instead of a hang.
// (set per device by the runtime from FSX_SPIN_TIMEOUT_S, default 30 s)
__constant__ uint64_t c_spin_timeout_ns = 30ull * 1000000000ull;

__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// gpu-scope wait: producer and consumer on the same GPU (colocated pass)
__device__ __forceinline__ void spin_until_gpu(const uint64_t* flag, uint64_t token) {
  if (ld_acquire_gpu(flag) == token) return;
  const uint64_t t0 = globaltimer_ns();
  uint32_t n = 0;
  while (ld_acquire_gpu(flag) != token) {
    __nanosleep(64);
    if ((++n & 1023u) == 0 && globaltimer_ns() - t0 > c_spin_timeout_ns) asm volatile("trap;");
  }
}

__device__ __forceinline__ void spin_until(const uint64_t* flag, uint64_t token) {
  if (ld_acquire_sys(flag) == token) return;
  const uint64_t t0 = globaltimer_ns();
  uint32_t n = 0;
  while (ld_acquire_sys(flag) != token) {
    __nanosleep(64);
    if ((++n & 1023u) == 0 && globaltimer_ns() - t0 > c_spin_timeout_ns) asm volatile("trap;");
  }
}

// splitmix64 finaliser (common.hpp:203-208): output k (1-based) of a stream
// with state s0 is mix(s0 + k * gamma), which makes every word independent.
__device__ __forceinline__ uint64_t splitmix_word(uint64_t s0, uint64_t k) {
  uint64_t z = s0 + k * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// ---------------------------------------------------------------------------
// K1 forward

// fsx integrity digest dg64 (replaces the serial checksum64 of
// common.hpp:221-241 on the device hop): with w_k the k-th little-endian
// 8-byte word of the payload (the last one zero-padded) and n its length,
//   dg64 = n * 0x9e3779b97f4a7c15 + sum_k f(w_k ^ (k + 1) * 0xbf58476d1ce4e5b9)  (mod 2^64)
//   f(x) = y ^ (y >> 29), y = x * 0x94d049bb133111eb
// Every term is independent (order-free sum, position folded into the word),
// so any partition of the bytes can be digested in parallel and combined with
// one atomic add; a flipped bit, a dropped or a swapped word changes it.
__device__ __forceinline__ uint64_t dg_word(uint64_t w, uint64_t k) {
  const uint64_t y = (w ^ ((k + 1) * 0xbf58476d1ce4e5b9ull)) * 0x94d049bb133111ebull;
  return y ^ (y >> 29);
}

__device__ __forceinline__ uint64_t dg_vec(const uint4& v, uint64_t word) {
  const uint64_t lo = (uint64_t)v.x | ((uint64_t)v.y << 32);
  const uint64_t hi = (uint64_t)v.z | ((uint64_t)v.w << 32);
  return dg_word(lo, word) + dg_word(hi, word + 1);
}

// digest of the words that start in [from, end) of a buffer whose byte 0 is
// word 0 (zero padding past `end`), read byte-wise
__device__ __forceinline__ uint64_t dg_bytes(const uint8_t* p, int64_t from, int64_t end) {
  uint64_t acc = 0;
  for (int64_t w = from >> 3; w * 8 < end; ++w) {
    uint64_t v = 0;
    for (int b = 0; b < 8 && w * 8 + b < end; ++b) v |= (uint64_t)p[w * 8 + b] << (8 * b);
    acc += dg_word(v, (uint64_t)w);
  }
  return acc;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

__device__ __forceinline__ uint64_t dg_any(const uint4& v, uint64_t word) { return dg_vec(v, word); }
__device__ __forceinline__ uint64_t dg_any(const v8u32& v, uint64_t word) {
  return dg_vec(v.lo, word) + dg_vec(v.hi, word + 2);
}

// Copy [beg, end) of src into dst with one warp using V-byte vectors (src, dst
// and beg are 16-byte aligned; V = 32 also needs 32-byte aligned src/dst).  All
// loads of a batch are issued before its stores (U x V bytes per lane in
// flight).  With `dig`, the lane also digests the words it moved (returned per
// lane; lane 0 adds the unvectorised head/tail bytes).
template <int U, int V>
__device__ __forceinline__ uint64_t warp_copy_vec(const uint8_t* __restrict__ src,
                                                  uint8_t* __restrict__ dst, int64_t beg, int64_t end,
                                                  bool dig, int lane, uint64_t ld_pol, uint64_t st_pol) {
  using IO = VecIO<V>;
  using T = typename IO::T;
  uint64_t acc = 0;
  const int64_t vbeg = (beg + V - 1) & ~int64_t{V - 1};
  const int64_t vend = end & ~int64_t{V - 1};
  if (vbeg < vend) {
    const int64_t nv = (vend - vbeg) / V;
    const uint64_t w0 = (uint64_t)(vbeg >> 3);
    for (int64_t base = 0; base < nv; base += 32 * U) {
      T r[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = base + k * 32 + lane;
        if (i < nv) r[k] = IO::ld(src + vbeg + i * V, ld_pol);
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = base + k * 32 + lane;
        if (i < nv) IO::st(dst + vbeg + i * V, r[k], st_pol);
      }
      if (dig) {
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int64_t i = base + k * 32 + lane;
          if (i < nv) acc += dg_any(r[k], w0 + (uint64_t)i * (V / 8));
        }
      }
    }
    for (int64_t i = beg + lane; i < vbeg; i += 32) dst[i] = src[i];
    for (int64_t i = vend + lane; i < end; i += 32) dst[i] = src[i];
    if (dig && lane == 0) {
      if (beg < vbeg) acc += dg_bytes(src, beg, vbeg);
      if (vend < end) acc += dg_bytes(src, vend, end);
    }
    return acc;
  }
  for (int64_t i = beg + lane; i < end; i += 32) dst[i] = src[i];
  if (dig && lane == 0) acc += dg_bytes(src, beg, end);  // unit smaller than a vector
  return acc;
}

// `vec`: 0 = byte path (unaligned; the runtime digests the source
// separately), otherwise the kernel's vector width V (16 or 32; the runtime
// launches the V = 32 instance only when every transfer allows it).
template <int U, int V>
__device__ __forceinline__ uint64_t warp_copy_range(const uint8_t* __restrict__ src,
                                                    uint8_t* __restrict__ dst, int64_t beg,
                                                    int64_t end, int vec, bool dig, int lane,
                                                    uint64_t ld_pol, uint64_t st_pol) {
  if (vec) return warp_copy_vec<U, V>(src, dst, beg, end, dig, lane, ld_pol, st_pol);
  for (int64_t i = beg + lane; i < end; i += 32) dst[i] = src[i];
  return 0;
}

__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t* p, uint32_t v, bool sys) {
  uint32_t old;
  if (sys)
    asm volatile("atom.add.acq_rel.sys.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  else
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Work unit u (kFwdUnitBytes, one warp) covers slice s of chunk c; units are
// chunk-major so chunks complete roughly in order and a consumer can start on
// chunk 0 while later chunks are still in flight.  Warps stream independently
// (no CTA barrier): after its unit a warp counts itself into the chunk counter
// with an acq_rel atomic (release covers the warp's stores via __syncwarp; gpu
// scope for a local slab, system scope when the slab is peer memory), and the
// warp that completes the chunk fences at system scope and publishes the token
// to the consumer-device flag and the host-mapped flag.
template <int U, int MINB, int V>
__global__ void __launch_bounds__(kFwdThreads, MINB) forward_kernel(const __grid_constant__ FwdBatch b) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (kFwdThreads / 32);
  const int64_t total = b.unit_off[b.n];
  // The producer's source is read once (evict first); slab writes may be
  // kept in L2 for a consumer that merges right after on this GPU.
  const uint64_t ld_pol = l2_policy(1);
  const uint64_t st_pol = l2_policy(b.l2_keep_dst ? 2 : 0);
  int i = 0;  // transfer of the current unit; units only grow per warp
  for (int64_t gu = (int64_t)blockIdx.x * (kFwdThreads / 32) + (threadIdx.x >> 5); gu < total;
       gu += warps) {
    while (gu >= b.unit_off[i + 1]) ++i;
    const FwdArgs& a = b.t[i];
    const int64_t u = gu - b.unit_off[i];
    const int64_t c = u / a.chunk_units;
    const int64_t s = u - c * a.chunk_units;
    const int64_t cbeg = c * a.chunk_bytes;
    const int64_t cend = min(cbeg + a.chunk_bytes, a.bytes);
    const int64_t beg = cbeg + s * a.slice;
    const int64_t end = min(beg + a.slice, cend);
    const bool dig = a.digest != nullptr;
    uint64_t acc = warp_copy_range<U, V>(a.src, a.dst, beg, end, a.vec, dig, lane, ld_pol, st_pol);
    if (dig) {  // fused dg64: one atomic per unit, ordered before the counter release
      acc = warp_sum_u64(acc);
      if (lane == 0) {
        if (u == 0) acc += (uint64_t)a.bytes * 0x9e3779b97f4a7c15ull;
        atomicAdd(reinterpret_cast<unsigned long long*>(a.digest), (unsigned long long)acc);
      }
    }
    __syncwarp();
    if (a.counters == nullptr) continue;  // diagnostic only: no completion tracking
    if (lane == 0) {
      const uint32_t units = (c == a.n_chunks - 1) ? (uint32_t)a.last_units : (uint32_t)a.chunk_units;
      const uint32_t prev = atom_add_acq_rel(&a.counters[c], 1u, a.peer != 0);
      if (prev == units - 1) {
        a.counters[c] = 0u;  // slot is clean for the next transfer that draws it
        if (a.peer) {
          // data sits in peer memory: publish at system scope
          __threadfence_system();
          st_release_sys(&a.dflags[c], a.token);
          if (a.hflags) st_relaxed_sys(&a.hflags[c], a.token);
        } else {
          // data sits in this GPU's memory: every counted warp released at gpu
          // scope and the acq_rel bump acquired them, so a gpu-scope release
          // publishes the chunk to device consumers; the host mirror is a
          // posted store issued only after every unit of the chunk is in L2.
          st_release_gpu(&a.dflags[c], a.token);
          if (a.hflags) st_relaxed_sys(&a.hflags[c], a.token);
        }
      }
    }
  }
}

// K1, tile form (default).  One CTA per tile of kTileThreads x U x 16 B, no
// persistence: the hardware CTA scheduler hands tiles to SMs as earlier ones
// retire, which on B200 sustains ~6.7 TB/s for a plain copy where a persistent
// grid-stride loop tops out near 5.9-6.3 (scripts/probe_sm_copy.cu).  Tiles are
// chunk-major in blockIdx order, so chunks complete roughly in order.  After
// its loads and stores the CTA barriers, and one thread counts the tile into
// the chunk counter with an acq_rel atomic (bar.sync makes every thread's
// stores part of that release; gpu scope for a local slab, system scope for
// peer memory); the CTA that completes the chunk publishes the token.
constexpr int kTileThreads = 256;

template <int U>
__global__ void __launch_bounds__(kTileThreads) forward_tile_kernel(const __grid_constant__ FwdBatch b) {
  __shared__ uint64_t red[kTileThreads / 32];
  const int64_t gt = blockIdx.x;
  int i = 0;
  while (gt >= b.unit_off[i + 1]) ++i;
  const FwdArgs& a = b.t[i];
  const int64_t u = gt - b.unit_off[i];
  const int64_t c = u / a.chunk_units;
  const int64_t s = u - c * a.chunk_units;
  const int64_t cbeg = c * a.chunk_bytes;
  const int64_t cend = min(cbeg + a.chunk_bytes, a.bytes);
  const int64_t beg = cbeg + s * a.slice;
  const int64_t end = min(beg + a.slice, cend);
  const uint64_t ld_pol = l2_policy(1);
  const uint64_t st_pol = l2_policy(b.l2_keep_dst ? 2 : 0);
  const bool dig = a.digest != nullptr;
  uint64_t acc = 0;
  if (a.vec) {
    // beg is 16-byte aligned (slices and chunks are multiples of 16)
    const int64_t vend = end & ~int64_t{15};
    const int64_t nv = (vend - beg) >> 4;
    uint4 r[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t v = k * kTileThreads + threadIdx.x;
      if (v < nv) r[k] = ld_nc_v4_pol(a.src + beg + v * 16, ld_pol);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t v = k * kTileThreads + threadIdx.x;
      if (v < nv) st_v4_pol(a.dst + beg + v * 16, r[k], st_pol);
    }
    if (dig) {
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t v = k * kTileThreads + threadIdx.x;
        if (v < nv) acc += dg_vec(r[k], (uint64_t)((beg >> 3) + 2 * v));
      }
      if (threadIdx.x == 0 && vend < end) acc += dg_bytes(a.src, vend, end);
    }
    for (int64_t j = vend + threadIdx.x; j < end; j += kTileThreads) a.dst[j] = a.src[j];
  } else {
    for (int64_t j = beg + threadIdx.x; j < end; j += kTileThreads) a.dst[j] = a.src[j];
  }
  if (dig) {  // block-reduce the digest, one atomic per tile
    acc = warp_sum_u64(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  }
  __syncthreads();
  if (threadIdx.x != 0 || a.counters == nullptr) return;
  if (dig) {
    uint64_t t = 0;
    for (int w = 0; w < kTileThreads / 32; ++w) t += red[w];
    if (u == 0) t += (uint64_t)a.bytes * 0x9e3779b97f4a7c15ull;
    atomicAdd(reinterpret_cast<unsigned long long*>(a.digest), (unsigned long long)t);
  }
  const uint32_t units = (c == a.n_chunks - 1) ? (uint32_t)a.last_units : (uint32_t)a.chunk_units;
  const uint32_t prev = atom_add_acq_rel(&a.counters[c], 1u, a.peer != 0);
  if (prev == units - 1) {
    a.counters[c] = 0u;
    if (a.peer) {
      __threadfence_system();
      st_release_sys(&a.dflags[c], a.token);
    } else {
      st_release_gpu(&a.dflags[c], a.token);
    }
    if (a.hflags) st_relaxed_sys(&a.hflags[c], a.token);
  }
}

// Stand-alone dg64 of n device bytes, accumulated into *out (zeroed by the
// caller): consumer-side verification of a delivered slab segment, and the
// producer digest when K1 ran its unaligned byte path.
__global__ void __launch_bounds__(256) digest_kernel(const uint8_t* __restrict__ p, int64_t n,
                                                     uint64_t* out) {
  uint64_t acc = 0;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t tail_from = 0;
  if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
    const int64_t nv = n >> 4;
    const uint4* v = reinterpret_cast<const uint4*>(p);
    for (int64_t i = tid; i < nv; i += stride) acc += dg_vec(ld_v4(v + i), 2 * (uint64_t)i);
    tail_from = nv << 4;
  } else {
    const int64_t nw = n >> 3;  // whole words, byte-assembled
    for (int64_t w = tid; w < nw; w += stride) acc += dg_bytes(p, w * 8, w * 8 + 8);
    tail_from = nw << 3;
  }
  if (tid == 0) acc += dg_bytes(p, tail_from, n) + (uint64_t)n * 0x9e3779b97f4a7c15ull;
  acc = warp_sum_u64(acc);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(reinterpret_cast<unsigned long long*>(out), (unsigned long long)acc);
}

// Small host messages (fsx_put_small), one CTA per message: copy the staged
// bytes from the mapped pinned mailbox (PCIe reads) into the slab segment,
// then read the landed segment back into the slot while computing its dg64,
// so a ChunkCallback consumer gets the bytes that are in device memory,
// verified on the device.  bar.sync orders the CTA's slab stores before its
// own re-reads (coherent loads, no .nc).
constexpr int kMailThreads = 256;
__global__ void __launch_bounds__(kMailThreads) mailbox_kernel(const __grid_constant__ MailStep m) {
  __shared__ uint64_t red[kMailThreads / 32];
  uint8_t* slot = m.mail + m.slot[blockIdx.x];
  MailHeader* h = reinterpret_cast<MailHeader*>(slot);
  uint8_t* bytes = slot + kMailHeader;
  uint8_t* dst = h->dst;
  const int64_t n = h->n;
  const bool vec = (reinterpret_cast<uintptr_t>(dst) & 15) == 0;  // slots are 64 B aligned
  const int64_t nv = vec ? n >> 4 : 0;
  for (int64_t i = threadIdx.x; i < nv; i += kMailThreads)
    st_v4(dst + 16 * i, ld_v4(bytes + 16 * i));
  for (int64_t j = nv * 16 + threadIdx.x; j < n; j += kMailThreads) dst[j] = bytes[j];
  __syncthreads();
  uint64_t acc = 0;
  for (int64_t i = threadIdx.x; i < nv; i += kMailThreads) {
    const uint4 v = ld_v4(dst + 16 * i);
    *reinterpret_cast<uint4*>(bytes + 16 * i) = v;
    acc += dg_vec(v, 2 * (uint64_t)i);
  }
  __syncthreads();  // every vector store into the slot precedes the tail rewrite below
  if (threadIdx.x == 0) {
    const int64_t from = nv * 16;
    for (int64_t j = from; j < n; ++j) bytes[j] = dst[j];
    acc += dg_bytes(dst, from, n) + (uint64_t)n * 0x9e3779b97f4a7c15ull;
  }
  acc = warp_sum_u64(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int w = 0; w < kMailThreads / 32; ++w) t += red[w];
    h->digest = t;
  }
}

__global__ void set_flags_kernel(FlagSetArgs a) {
  for (int i = threadIdx.x; i < a.n; i += blockDim.x) {
    st_release_sys(&a.dflags[i], a.token);
    if (a.hflags) st_release_sys(&a.hflags[i], a.token);
  }
}

__global__ void wait_flags_kernel(const uint64_t* dflags, int32_t n, uint64_t token) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) spin_until(&dflags[i], token);
  __syncthreads();
}

// ---------------------------------------------------------------------------
// K3 merge, phase 1: per-request placeholder positions.
//
// One CTA per request.  Per round, warp w reads kScanRounds x 32 consecutive
// token ids with coalesced loads (round j, lane l -> token base_w + 32 j + l),
// ballots the placeholder mask of each round, and the CTA scans the per-warp
// totals once in shared memory.  The k-th placeholder row of the request gets
// its row offset inside the request written to
// scratch[item_row_off[first item] + k].
__global__ void __launch_bounds__(kScanThreads) merge_scan_kernel(fsx_merge_batch b) {
  __shared__ int32_t warp_excl[kScanThreads / 32];
  __shared__ int32_t tile_total;
  __shared__ int64_t running;
  const int r = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t t0 = b.d_req_row_off[r], t1 = b.d_req_row_off[r + 1];
  const int64_t i0 = b.d_req_item_off[r], i1 = b.d_req_item_off[r + 1];
  const int64_t kbase = b.d_item_row_off[i0];
  const int64_t want = b.d_item_row_off[i1] - kbase;
  const uint32_t lt_mask = (1u << lane) - 1u;
  if (threadIdx.x == 0) running = 0;
  __syncthreads();
  constexpr int64_t kTile = int64_t{kScanThreads} * kScanRounds;
  for (int64_t t = t0; t < t1; t += kTile) {
    const int64_t wbase = t + int64_t{warp} * 32 * kScanRounds + lane;
    uint32_t m[kScanRounds];
    int wcount = 0;
#pragma unroll
    for (int j = 0; j < kScanRounds; ++j) {
      const int64_t tt = wbase + 32 * j;
      const bool p = tt < t1 && b.d_token_ids[tt] == b.placeholder_id;
      m[j] = __ballot_sync(0xffffffffu, p);
      wcount += __popc(m[j]);
    }
    if (lane == 0) warp_excl[warp] = wcount;
    __syncthreads();
    if (warp == 0) {
      const int v = warp_excl[lane];
      int incl = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += x;
      }
      warp_excl[lane] = incl - v;
      if (lane == 31) tile_total = incl;
    }
    __syncthreads();
    int64_t k = running + warp_excl[warp];
#pragma unroll
    for (int j = 0; j < kScanRounds; ++j) {
      if ((m[j] >> lane) & 1u) {
        const int64_t kk = k + __popc(m[j] & lt_mask);
        if (kk < want) b.d_scratch[kbase + kk] = (int32_t)(wbase + 32 * j - t0);
      }
      k += __popc(m[j]);
    }
    __syncthreads();
    if (threadIdx.x == 0) running += tile_total;
    __syncthreads();
  }
  if (threadIdx.x == 0) b.d_status[r] = (running == want) ? 0 : FSX_E_VALIDATION;
}

__device__ __forceinline__ int64_t upper_index(const int64_t* off, int64_t n, int64_t x) {
  // largest i in [0, n) with off[i] <= x  (off is non-decreasing, off[0] == 0)
  int64_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (off[mid] <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// K3 merge, phase 2: one warp per placeholder row.  Lane 0 resolves the row's
// item (binary search over item row offsets) and request, then the warp moves
// the row as 16-byte vectors, all loads of a batch issued before its stores.
__global__ void __launch_bounds__(kMergeThreads) merge_copy_kernel(fsx_merge_batch b) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (kMergeThreads / 32);
  const int64_t rb = b.row_bytes;
  const bool vec_rows = (rb & 15) == 0;
  // newest rows first (meant for L2 reuse of K1's tail; measured no effect on
  // B200, DESIGN.md §3 -- kept, it costs nothing)
  const bool newest_first = b.d_item_flag == nullptr;
  const bool discard = (b.mode & FSX_MERGE_DISCARD) != 0;
  for (int64_t k = (int64_t)blockIdx.x * (kMergeThreads / 32) + (threadIdx.x >> 5);
       k < b.total_item_rows; k += warps) {
    const int64_t g = newest_first ? b.total_item_rows - 1 - k : k;
    int64_t item = 0, req = 0;
    if (lane == 0) {
      item = upper_index(b.d_item_row_off, b.num_items + 1, g);
      // skip zero-row items sharing the same offset
      while (b.d_item_row_off[item + 1] <= g) ++item;
      req = upper_index(b.d_req_item_off, b.num_requests + 1, item);
      while (b.d_req_item_off[req + 1] <= item) ++req;
    }
    item = __shfl_sync(0xffffffffu, item, 0);
    req = __shfl_sync(0xffffffffu, req, 0);
    if (b.d_status[req] != 0) continue;  // validation failed: request untouched
    const int64_t j = g - b.d_item_row_off[item];
    if (b.d_item_flag) {
      if (lane == 0) {
        const int64_t cr = b.d_item_chunk_rows[item];
        spin_until(b.d_item_flag[item] + (cr > 0 ? j / cr : 0), b.d_item_token[item]);
      }
      __syncwarp();
    }
    const uint8_t* src = static_cast<const uint8_t*>(b.d_item_src[item]) + j * rb;
    const int64_t t = b.d_req_row_off[req] + b.d_scratch[g];
    uint8_t* dst = static_cast<uint8_t*>(b.d_embeds) + t * rb;
    if (vec_rows && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
      const int64_t nv = rb >> 4;
      const uint4* s = reinterpret_cast<const uint4*>(src);
      uint4* d = reinterpret_cast<uint4*>(dst);
      for (int64_t base = 0; base < nv; base += 32 * kMergeUnroll) {
        uint4 r[kMergeUnroll];
#pragma unroll
        for (int k = 0; k < kMergeUnroll; ++k) {
          const int64_t i = base + k * 32 + lane;
          if (i < nv) r[k] = ld_v4(s + i);
        }
#pragma unroll
        for (int k = 0; k < kMergeUnroll; ++k) {
          const int64_t i = base + k * 32 + lane;
          if (i < nv) st_v4(d + i, r[k]);
        }
      }
    } else {
      for (int64_t i = lane; i < rb; i += 32) dst[i] = src[i];
    }
    if (discard) {
      // the row's values are in registers and stored: drop its slab lines
      // from L2 without writing them back (whole 128-byte lines only)
      const uintptr_t lo = (reinterpret_cast<uintptr_t>(src) + 127) & ~uintptr_t{127};
      const uintptr_t hi = (reinterpret_cast<uintptr_t>(src) + rb) & ~uintptr_t{127};
      for (uintptr_t a = lo + 128 * (uintptr_t)lane; a < hi; a += 128 * 32)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
    }
  }
}

// K3 merge, phase 2, early-start form: rows are taken in arrival order in runs
// of kStreamRun consecutive placeholder rows per warp.  The warp resolves the
// run's first row once (binary searches), prefetches the run's placeholder
// positions with one coalesced load (one lane per row), and walks the rows
// keeping item- and request-level values in registers, re-reading them only
// when the run crosses into the next item or request, and spinning on a chunk
// flag only when the run enters a new chunk.  A persistent grid of these warps
// follows the producer's K1 chunk by chunk with far less per-row latency than
// resolving every row from scratch (merge_copy_kernel).
constexpr int kStreamRun = 16;
__global__ void __launch_bounds__(kMergeThreads) merge_stream_kernel(fsx_merge_batch b,
                                                                     unsigned long long* work) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (kMergeThreads / 32);
  const int64_t rb = b.row_bytes;
  const int64_t n = b.total_item_rows;
  const int64_t runs = (n + kStreamRun - 1) / kStreamRun;
  const bool vec_rows = (rb & 15) == 0;
  const bool discard = (b.mode & FSX_MERGE_DISCARD) != 0;
  const bool early = b.d_item_flag != nullptr;
  // runs are claimed from the work counter in arrival order (every warp works
  // on the earliest rows whose chunk has landed), or statically without one
  auto claim = [&](int64_t prev) -> int64_t {
    if (!work) return prev < 0 ? (int64_t)blockIdx.x * (kMergeThreads / 32) + (threadIdx.x >> 5) : prev + warps;
    unsigned long long u = 0;
    if (lane == 0) u = atomicAdd(work, 1ull);
    return (int64_t)__shfl_sync(0xffffffffu, u, 0);
  };
  for (int64_t u = claim(-1); u < runs; u = claim(u)) {
    const int64_t g0 = u * kStreamRun;
    const int64_t g1 = min(g0 + kStreamRun, n);
    const int32_t mypos = (g0 + lane < g1) ? b.d_scratch[g0 + lane] : 0;
    // every lane runs the same (uniform) resolution: same addresses, broadcast loads
    int64_t item = upper_index(b.d_item_row_off, b.num_items + 1, g0);
    while (b.d_item_row_off[item + 1] <= g0) ++item;
    int64_t req = upper_index(b.d_req_item_off, b.num_requests + 1, item);
    while (b.d_req_item_off[req + 1] <= item) ++req;
    int64_t item_beg = b.d_item_row_off[item], item_end = b.d_item_row_off[item + 1];
    const uint8_t* item_src = static_cast<const uint8_t*>(b.d_item_src[item]);
    int64_t req_row = b.d_req_row_off[req];
    int32_t req_ok = b.d_status[req] == 0;
    int64_t chunk_rows = early ? b.d_item_chunk_rows[item] : 0;
    int64_t waited = -1;  // chunk of the current item already waited for
    for (int64_t g = g0; g < g1; ++g) {
      if (g >= item_end) {  // next item (skipping zero-row items), maybe next request
        do {
          ++item;
        } while (b.d_item_row_off[item + 1] <= g);
        item_beg = b.d_item_row_off[item];
        item_end = b.d_item_row_off[item + 1];
        item_src = static_cast<const uint8_t*>(b.d_item_src[item]);
        if (b.d_req_item_off[req + 1] <= item) {
          do {
            ++req;
          } while (b.d_req_item_off[req + 1] <= item);
          req_row = b.d_req_row_off[req];
          req_ok = b.d_status[req] == 0;
        }
        if (early) chunk_rows = b.d_item_chunk_rows[item];
        waited = -1;
      }
      const int32_t pos = __shfl_sync(0xffffffffu, mypos, (int)(g - g0));
      if (!req_ok) continue;  // validation failed: request untouched
      const int64_t j = g - item_beg;
      if (early) {
        const int64_t c = chunk_rows > 0 ? j / chunk_rows : 0;
        if (c != waited) {
          if (lane == 0) spin_until(b.d_item_flag[item] + c, b.d_item_token[item]);
          __syncwarp();
          waited = c;
        }
      }
      const uint8_t* src = item_src + j * rb;
      uint8_t* dst = static_cast<uint8_t*>(b.d_embeds) + (req_row + pos) * rb;
      if (vec_rows && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
        const int64_t nv = rb >> 4;
        const uint4* sv = reinterpret_cast<const uint4*>(src);
        uint4* dv = reinterpret_cast<uint4*>(dst);
        for (int64_t base = 0; base < nv; base += 32 * kMergeUnroll) {
          uint4 r[kMergeUnroll];
#pragma unroll
          for (int k = 0; k < kMergeUnroll; ++k) {
            const int64_t i = base + k * 32 + lane;
            if (i < nv) r[k] = ld_v4(sv + i);
          }
#pragma unroll
          for (int k = 0; k < kMergeUnroll; ++k) {
            const int64_t i = base + k * 32 + lane;
            if (i < nv) st_v4(dv + i, r[k]);
          }
        }
      } else {
        for (int64_t i = lane; i < rb; i += 32) dst[i] = src[i];
      }
      if (discard) {
        const uintptr_t lo = (reinterpret_cast<uintptr_t>(src) + 127) & ~uintptr_t{127};
        const uintptr_t hi = (reinterpret_cast<uintptr_t>(src) + rb) & ~uintptr_t{127};
        for (uintptr_t a = lo + 128 * (uintptr_t)lane; a < hi; a += 128 * 32)
          asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
      }
    }
  }
}

// K3 merge, phase 2, "follow" form for early start: warp w of W moves the
// placeholder rows g = w, w + W, w + 2W, ... in increasing order, so at any
// moment the whole grid works on a window of about W rows right behind the
// producer (one chunk's worth for W ~ chunk rows) instead of some warps
// holding runs many chunks ahead.  Behind K1 on the same GPU that window is
// still in L2 when it is read, and with FSX_MERGE_DISCARD its lines are
// dropped from L2 right after, so the slab never round-trips through HBM.
// Item / request values are re-read only when the warp's row crosses into the
// next item; the row's chunk flag is checked (lane 0, acquire) before its
// loads; the position comes from the scan's scratch.
template <int U>
__global__ void __launch_bounds__(kMergeThreads, 2) merge_follow_kernel(fsx_merge_batch b) {
  const int lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * (kMergeThreads / 32);
  const int64_t w = (int64_t)blockIdx.x * (kMergeThreads / 32) + (threadIdx.x >> 5);
  const int64_t rb = b.row_bytes;
  const int64_t n = b.total_item_rows;
  if (w >= n) return;
  const bool vec_rows = (rb & 15) == 0;
  const bool discard = (b.mode & FSX_MERGE_DISCARD) != 0;
  const bool early = b.d_item_flag != nullptr;
  // the producer's K1 runs on this GPU: a gpu-scope acquire pairs with its
  // gpu-scope release; across GPUs the wait is system scope
#ifndef FSX_COLOCATED_GPU_SCOPE
#define FSX_COLOCATED_GPU_SCOPE 1
#endif
  const bool colocated = FSX_COLOCATED_GPU_SCOPE && (b.mode & FSX_MERGE_COLOCATED) != 0;
  // the prompt rows are written once and not re-read here: evict them from L2
  // first, so they do not push out slab rows K1 has just written
  const uint64_t out_pol = l2_policy(kFollowOutPolicy);
  int64_t item = upper_index(b.d_item_row_off, b.num_items + 1, w);
  while (b.d_item_row_off[item + 1] <= w) ++item;
  int64_t req = upper_index(b.d_req_item_off, b.num_requests + 1, item);
  while (b.d_req_item_off[req + 1] <= item) ++req;
  int64_t item_beg = b.d_item_row_off[item], item_end = b.d_item_row_off[item + 1];
  const uint8_t* item_src = static_cast<const uint8_t*>(b.d_item_src[item]);
  int64_t chunk_rows = early ? b.d_item_chunk_rows[item] : 0;
  int64_t req_row = b.d_req_row_off[req];
  bool req_ok = b.d_status[req] == 0;
  int64_t waited = -1;
  for (int64_t g = w; g < n; g += W) {
    if (g >= item_end) {
      do {
        ++item;
      } while (b.d_item_row_off[item + 1] <= g);
      item_beg = b.d_item_row_off[item];
      item_end = b.d_item_row_off[item + 1];
      item_src = static_cast<const uint8_t*>(b.d_item_src[item]);
      if (early) chunk_rows = b.d_item_chunk_rows[item];
      waited = -1;
      if (b.d_req_item_off[req + 1] <= item) {
        do {
          ++req;
        } while (b.d_req_item_off[req + 1] <= item);
        req_row = b.d_req_row_off[req];
        req_ok = b.d_status[req] == 0;
      }
    }
    if (!req_ok) continue;  // validation failed: request untouched
    const int64_t j = g - item_beg;
    const int32_t pos = b.d_scratch[g];
    if (early) {
      const int64_t c = chunk_rows > 0 ? j / chunk_rows : 0;
      if (c != waited) {
        if (lane == 0) {
          if (colocated) spin_until_gpu(b.d_item_flag[item] + c, b.d_item_token[item]);
          else spin_until(b.d_item_flag[item] + c, b.d_item_token[item]);
        }
        __syncwarp();
        waited = c;
      }
    }
    const uint8_t* src = item_src + j * rb;
    uint8_t* dst = static_cast<uint8_t*>(b.d_embeds) + (req_row + pos) * rb;
    if (vec_rows && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
      const int64_t nv = rb >> 4;
      const uint4* sv = reinterpret_cast<const uint4*>(src);
      uint4* dv = reinterpret_cast<uint4*>(dst);
      for (int64_t base = 0; base < nv; base += 32 * U) {
        uint4 r[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int64_t i = base + k * 32 + lane;
          if (i < nv) r[k] = ld_v4(sv + i);
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int64_t i = base + k * 32 + lane;
          if (i < nv) st_v4_pol(dv + i, r[k], out_pol);
        }
      }
    } else {
      for (int64_t i = lane; i < rb; i += 32) dst[i] = src[i];
    }
    if (discard) {
      const uintptr_t lo = (reinterpret_cast<uintptr_t>(src) + 127) & ~uintptr_t{127};
      const uintptr_t hi = (reinterpret_cast<uintptr_t>(src) + rb) & ~uintptr_t{127};
      for (uintptr_t a = lo + 128 * (uintptr_t)lane; a < hi; a += 128 * 32)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
    }
  }
}

// Follow kernel, software-pipelined (FSX_MERGE_STREAM=4): the same row order
// as merge_follow_kernel, but while a row's loads are in flight the warp
// already resolves its next row (placeholder position, source view) and lane 0
// issues that row's chunk-flag acquire, so the flag and position latencies
// overlap the data instead of preceding it.  lane 0's acquire plus the
// __syncwarp before the next row's loads order them after the flag.
struct FollowRow {
  const uint8_t* src;
  uint8_t* dst;
  const uint64_t* flag;
  uint64_t token;
  bool valid, ok;
};

template <int U>
__global__ void __launch_bounds__(kMergeThreads, 2) merge_follow2_kernel(fsx_merge_batch b) {
  const int lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * (kMergeThreads / 32);
  const int64_t w = (int64_t)blockIdx.x * (kMergeThreads / 32) + (threadIdx.x >> 5);
  const int64_t rb = b.row_bytes;
  const int64_t n = b.total_item_rows;
  if (w >= n) return;
  const bool discard = (b.mode & FSX_MERGE_DISCARD) != 0;
  const bool early = b.d_item_flag != nullptr;
  const bool colocated = FSX_COLOCATED_GPU_SCOPE && (b.mode & FSX_MERGE_COLOCATED) != 0;
  const bool vec_rows = (rb & 15) == 0;
  const uint64_t out_pol = l2_policy(kFollowOutPolicy);
  int64_t item = upper_index(b.d_item_row_off, b.num_items + 1, w);
  while (b.d_item_row_off[item + 1] <= w) ++item;
  int64_t req = upper_index(b.d_req_item_off, b.num_requests + 1, item);
  while (b.d_req_item_off[req + 1] <= item) ++req;
  int64_t item_beg = b.d_item_row_off[item], item_end = b.d_item_row_off[item + 1];
  const uint8_t* item_src = static_cast<const uint8_t*>(b.d_item_src[item]);
  int64_t chunk_rows = early ? b.d_item_chunk_rows[item] : 0;
  const uint64_t* item_flags = early ? b.d_item_flag[item] : nullptr;
  uint64_t item_token = early ? b.d_item_token[item] : 0;
  int64_t req_row = b.d_req_row_off[req];
  bool req_ok = b.d_status[req] == 0;
  auto resolve = [&](int64_t g, FollowRow& m) {
    m.valid = g < n;
    if (!m.valid) return;
    if (g >= item_end) {
      do {
        ++item;
      } while (b.d_item_row_off[item + 1] <= g);
      item_beg = b.d_item_row_off[item];
      item_end = b.d_item_row_off[item + 1];
      item_src = static_cast<const uint8_t*>(b.d_item_src[item]);
      if (early) {
        chunk_rows = b.d_item_chunk_rows[item];
        item_flags = b.d_item_flag[item];
        item_token = b.d_item_token[item];
      }
      if (b.d_req_item_off[req + 1] <= item) {
        do {
          ++req;
        } while (b.d_req_item_off[req + 1] <= item);
        req_row = b.d_req_row_off[req];
        req_ok = b.d_status[req] == 0;
      }
    }
    m.ok = req_ok;
    const int64_t j = g - item_beg;
    m.src = item_src + j * rb;
    m.dst = static_cast<uint8_t*>(b.d_embeds) + (req_row + b.d_scratch[g]) * rb;
    m.flag = early ? item_flags + (chunk_rows > 0 ? j / chunk_rows : 0) : nullptr;
    m.token = item_token;
  };
  auto acquire = [&](const uint64_t* f) { return colocated ? ld_acquire_gpu(f) : ld_acquire_sys(f); };
  FollowRow cur, nxt;
  resolve(w, cur);
  uint64_t seen = (early && lane == 0 && cur.ok) ? acquire(cur.flag) : 0;
  for (int64_t g = w; cur.valid; g += W) {
    if (early && cur.ok) {
      if (lane == 0 && seen != cur.token) {  // not landed yet when prefetched: wait
        const uint64_t t0 = globaltimer_ns();
        uint32_t spins = 0;
        while ((seen = acquire(cur.flag)) != cur.token) {
          __nanosleep(64);
          if ((++spins & 1023u) == 0 && globaltimer_ns() - t0 > c_spin_timeout_ns) asm volatile("trap;");
        }
      }
      __syncwarp();
    }
    const bool vec = vec_rows && ((reinterpret_cast<uintptr_t>(cur.src) | reinterpret_cast<uintptr_t>(cur.dst)) & 15) == 0;
    const int64_t nv = vec ? rb >> 4 : 0;
    const uint4* sv = reinterpret_cast<const uint4*>(cur.src);
    uint4* dv = reinterpret_cast<uint4*>(cur.dst);
    uint4 r[U];
    if (cur.ok) {
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = k * 32 + lane;
        if (i < nv) r[k] = ld_v4(sv + i);
      }
    }
    // the next row: position, view and flag acquire overlap this row's loads
    resolve(g + W, nxt);
    uint64_t nseen = 0;
    if (early && lane == 0 && nxt.valid && nxt.ok) nseen = acquire(nxt.flag);
    if (cur.ok) {
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = k * 32 + lane;
        if (i < nv) st_v4_pol(dv + i, r[k], out_pol);
      }
      for (int64_t base = 32 * U; base < nv; base += 32 * U) {  // rows wider than one batch
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int64_t i = base + k * 32 + lane;
          if (i < nv) r[k] = ld_v4(sv + i);
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int64_t i = base + k * 32 + lane;
          if (i < nv) st_v4_pol(dv + i, r[k], out_pol);
        }
      }
      if (!vec)
        for (int64_t i = lane; i < rb; i += 32) cur.dst[i] = cur.src[i];
      if (discard) {
        const uintptr_t lo = (reinterpret_cast<uintptr_t>(cur.src) + 127) & ~uintptr_t{127};
        const uintptr_t hi = (reinterpret_cast<uintptr_t>(cur.src) + rb) & ~uintptr_t{127};
        for (uintptr_t a = lo + 128 * (uintptr_t)lane; a < hi; a += 128 * 32)
          asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
      }
    }
    cur = nxt;
    seen = nseen;
  }
}

// ---------------------------------------------------------------------------
// K0 synth: each thread emits word pairs as one 16-byte store.
__global__ void synth_kernel(uint64_t s0, uint8_t* __restrict__ dst, int64_t n) {
  const int64_t nwords = n >> 3;
  const int64_t npairs = nwords >> 1;
  const bool al16 = (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npairs; p += stride) {
    const uint64_t w0 = splitmix_word(s0, 2 * p + 1);
    const uint64_t w1 = splitmix_word(s0, 2 * p + 2);
    if (al16) {
      *reinterpret_cast<ulonglong2*>(dst + 16 * p) = make_ulonglong2(w0, w1);
    } else {
      for (int bt = 0; bt < 8; ++bt) dst[16 * p + bt] = (uint8_t)(w0 >> (8 * bt));
      for (int bt = 0; bt < 8; ++bt) dst[16 * p + 8 + bt] = (uint8_t)(w1 >> (8 * bt));
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int64_t w = 2 * npairs; w * 8 < n; ++w) {  // odd last word and the truncated tail
      const uint64_t v = splitmix_word(s0, (uint64_t)w + 1);
      for (int bt = 0; bt < 8 && w * 8 + bt < n; ++bt) dst[w * 8 + bt] = (uint8_t)(v >> (8 * bt));
    }
  }
}

}  // namespace kern

using namespace kern;

__global__ void __launch_bounds__(32) forward_tma_kernel(const __grid_constant__ FwdBatch b);

// ---------------------------------------------------------------------------
// Launchers

int forward_block_threads() { return kFwdThreads; }

cudaError_t set_spin_timeout(uint64_t ns) {
  return cudaMemcpyToSymbol(c_spin_timeout_ns, &ns, sizeof(ns));
}
int merge_copy_block_threads() { return kMergeThreads; }

namespace {
using FwdFn = void (*)(FwdBatch);
// variant: 0 <16 x 16 B, 2 CTAs/SM>, 1 <8 x 16 B, 4 CTAs/SM>, 2 <8 x 16 B, 3 CTAs/SM>;
// wide = 32-byte vectors with half the count (same bytes in flight).
FwdFn forward_variant(int v, bool wide = false) {
  switch (v) {
    case 1: return wide ? forward_kernel<4, 4, 32> : forward_kernel<8, 4, 16>;
    case 2: return wide ? forward_kernel<4, 3, 32> : forward_kernel<8, 3, 16>;
    default: return wide ? forward_kernel<8, 2, 32> : forward_kernel<16, 2, 16>;
  }
}
}  // namespace

int forward_blocks_per_sm(int variant) {
  int n = 0;
  if (variant >= 3) variant = 2;  // tile kernels are not persistent: grid = tiles
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, forward_variant(variant), kFwdThreads, 0) !=
      cudaSuccess)
    return 1;
  return n > 0 ? n : 1;
}

int merge_copy_blocks_per_sm() {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, merge_copy_kernel, kMergeThreads, 0) !=
      cudaSuccess)
    return 1;
  return n > 0 ? n : 1;
}

int forward_tile_bytes(int variant) {
  if (variant == 5) return kTmaTileBytes;          // 32 KiB bulk-copy tiles
  if (variant == 3) return kTileThreads * 4 * 16;  // 16 KiB tiles
  if (variant == 4) return kTileThreads * 8 * 16;  // 32 KiB tiles
  return 0;                                        // persistent warp kernels
}

cudaError_t launch_forward(const FwdBatch& b, int variant, int grid, cudaStream_t s, bool share_sm) {
  if (variant == 5) {
    // bulk-copy tiles for local, 16-byte aligned transfers without a fused
    // digest; anything else in the batch takes the register tile kernel
    bool ok = true;
    for (int k = 0; k < b.n; ++k) ok = ok && b.t[k].vec && !b.t[k].peer && !b.t[k].digest;
    if (ok) {
      const int64_t tiles = b.unit_off[b.n];
      if (tiles <= 0) return cudaSuccess;
      // FSX_FWD_BULK_SMEM pads the shared memory per CTA (bytes >= 32 KiB) to cap
      // the resident K1 CTAs per SM, e.g. beside a concurrent merge
      static const int smem = [] {
        const char* e = std::getenv("FSX_FWD_BULK_SMEM");
        const int v = e ? std::atoi(e) : kTmaTileBytes;
        return v < kTmaTileBytes ? kTmaTileBytes : v;
      }();
      // the opt-in shared-memory limit is a per-device function attribute
      static bool attr_set[kMaxDevices] = {};
      int dev = 0;
      cudaGetDevice(&dev);
      if (dev < kMaxDevices && !attr_set[dev]) {
        cudaFuncSetAttribute(forward_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr_set[dev] = true;
      }
      forward_tma_kernel<<<(unsigned)tiles, 32, smem, s>>>(b);
      return cudaGetLastError();
    }
    variant = 4;
  }
  if (forward_tile_bytes(variant)) {
    // one CTA per tile: grid = total tiles of the batch (16-byte vectors)
    FwdBatch bb = b;
    for (int k = 0; k < bb.n; ++k)
      if (bb.t[k].vec) bb.t[k].vec = 16;
    const int64_t tiles = bb.unit_off[bb.n];
    if (tiles <= 0) return cudaSuccess;
    // share_sm: pad shared memory so at most two K1 CTAs fit per SM (the
    // opt-in limit is a per-device function attribute)
    static int pad[kMaxDevices] = {};
    size_t smem = 0;
    if (share_sm) {
      int dev = 0;
      cudaGetDevice(&dev);
      if (dev < kMaxDevices && pad[dev] == 0) {
        int sm_smem = 0;
        cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        pad[dev] = sm_smem / 2 - 8 * 1024;  // 2 x pad + reserved fits, 3 x pad does not
        cudaFuncSetAttribute(forward_tile_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, pad[dev]);
        cudaFuncSetAttribute(forward_tile_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, pad[dev]);
      }
      smem = dev < kMaxDevices ? (size_t)pad[dev] : 0;
    }
    if (variant == 3) forward_tile_kernel<4><<<(unsigned)tiles, kTileThreads, smem, s>>>(bb);
    else forward_tile_kernel<8><<<(unsigned)tiles, kTileThreads, smem, s>>>(bb);
    return cudaGetLastError();
  }
  bool wide = true;  // every vectorised transfer allows 32-byte vectors
  for (int k = 0; k < b.n; ++k) wide = wide && (b.t[k].vec == 32 || b.t[k].vec == 0);
  FwdBatch bb = b;
  if (!wide)
    for (int k = 0; k < bb.n; ++k)
      if (bb.t[k].vec == 32) bb.t[k].vec = 16;
  forward_variant(variant, wide)<<<grid, kFwdThreads, 0, s>>>(bb);
  return cudaGetLastError();
}

cudaError_t launch_set_flags(const FlagSetArgs& a, cudaStream_t s) {
  set_flags_kernel<<<1, 32, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_wait_flags(const uint64_t* dflags, int32_t n, uint64_t token, cudaStream_t s) {
  wait_flags_kernel<<<1, 32, 0, s>>>(dflags, n, token);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Streaming channels (config C: thinker hidden states per decode step, talker
// codes per chunk; executor_sim.hpp:540-564).  One push launch per decode step
// moves every active request's row (one CTA-warp per row) into slot
// seq % slots of that request's ring in the consumer slab and publishes
// flag = tag(seq) with release semantics; one pull launch on the consumer
// waits per row (acquire), gathers the rows in seq order into the consumer's
// input and releases the slot back to the producer (tail = seq + 1).  Device
// counters carry seq, so a step needs no host round trip.

__device__ __forceinline__ void warp_copy_row(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                              uint32_t n, int lane) {
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) | n) & 15) == 0) {
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    const uint32_t nv = n >> 4;
    for (uint32_t base = 0; base < nv; base += 32 * 16) {
      uint4 r[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t i = base + k * 32 + lane;
        if (i < nv) r[k] = ld_v4(s + i);
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t i = base + k * 32 + lane;
        if (i < nv) st_v4(d + i, r[k]);
      }
    }
  } else {
    for (uint32_t i = lane; i < n; i += 32) dst[i] = src[i];
  }
}

__global__ void __launch_bounds__(32) chan_push_kernel(const __grid_constant__ ChanStep s) {
  const ChanRow& c = s.c[blockIdx.x];
  const int lane = threadIdx.x;
  const uint64_t seq = *c.head;
  if (lane == 0) {  // backpressure: the slot's previous message was consumed
    const uint64_t t0 = globaltimer_ns();
    uint32_t n = 0;
    while (seq - ld_acquire_sys(c.tail) >= c.slots) {
      __nanosleep(64);
      if ((++n & 1023u) == 0 && globaltimer_ns() - t0 > c_spin_timeout_ns) asm volatile("trap;");
    }
  }
  __syncwarp();
  uint8_t* dst = c.ring + (seq % c.slots) * (uint64_t)c.row_bytes;
  warp_copy_row(s.rows + blockIdx.x * s.stride, dst, c.row_bytes, lane);
  __syncwarp();
  if (lane == 0) {
    const uint64_t tag = c.salt | (seq + 1);
    if (c.peer) {
      st_release_sys(&c.flags[seq % c.slots], tag);
    } else {
      st_release_gpu(&c.flags[seq % c.slots], tag);
    }
    *c.head = seq + 1;
  }
}

__global__ void __launch_bounds__(32) chan_pull_kernel(const __grid_constant__ ChanStep s) {
  const ChanRow& c = s.c[blockIdx.x];
  const int lane = threadIdx.x;
  const uint64_t seq = *c.tail;
  const uint64_t slot = seq % c.slots;
  if (lane == 0) spin_until(&c.flags[slot], c.salt | (seq + 1));
  __syncwarp();
  uint8_t* out = const_cast<uint8_t*>(s.rows) + blockIdx.x * s.stride;
  warp_copy_row(c.ring + slot * (uint64_t)c.row_bytes, out, c.row_bytes, lane);
  __syncwarp();
  if (lane == 0) st_release_sys(c.tail, seq + 1);  // slot free for the producer
}

// ---------------------------------------------------------------------------
// K3 merge, phase 2, TMA variant: rows staged through shared memory by the
// bulk-copy engine (cp.async.bulk global->shared with mbarrier completion,
// shared->global bulk_group stores).  One elected thread per CTA runs an
// S-stage ring: loads run S-1 rows ahead, each row's store is committed as
// its own bulk group, and a stage is refilled once `wait_group.read 1` says the
// store that last used it has finished reading shared memory.  No register
// staging, no per-lane address math: the copy engine moves the 7-8 KiB rows.

namespace tma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "FSX_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra FSX_WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_load(uint32_t dst_smem, const void* src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst_smem),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void bulk_store(void* dst, uint32_t src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(src_smem), "r"(bytes)
               : "memory");
}

// bulk store with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void bulk_store_hint(void* dst, uint32_t src_smem, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(src_smem), "r"(bytes), "l"(pol)
               : "memory");
}

// bulk load with an L2 eviction-priority policy
__device__ __forceinline__ void bulk_load_hint(uint32_t dst_smem, const void* src, uint32_t bytes, uint32_t bar,
                                               uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst_smem),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

}  // namespace tma

struct RowRef {
  const uint8_t* src;
  uint8_t* dst;
};

// Resolve placeholder row g: source row in its item, destination prompt row;
// src == nullptr when its request failed validation.
__device__ __forceinline__ RowRef resolve_row(const fsx_merge_batch& b, int64_t g) {
  int64_t item = upper_index(b.d_item_row_off, b.num_items + 1, g);
  while (b.d_item_row_off[item + 1] <= g) ++item;
  int64_t req = upper_index(b.d_req_item_off, b.num_requests + 1, item);
  while (b.d_req_item_off[req + 1] <= item) ++req;
  if (b.d_status[req] != 0) return RowRef{nullptr, nullptr};
  const int64_t j = g - b.d_item_row_off[item];
  if (b.d_item_flag) {
    const int64_t cr = b.d_item_chunk_rows[item];
    spin_until(b.d_item_flag[item] + (cr > 0 ? j / cr : 0), b.d_item_token[item]);
    // the row is read by the bulk-copy (async) proxy after a generic acquire
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  const uint8_t* src = static_cast<const uint8_t*>(b.d_item_src[item]) + j * b.row_bytes;
  uint8_t* dst = static_cast<uint8_t*>(b.d_embeds) + (b.d_req_row_off[req] + b.d_scratch[g]) * b.row_bytes;
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) {
    for (int64_t i = 0; i < b.row_bytes; ++i) dst[i] = src[i];  // bulk copies need 16 B alignment
    return RowRef{nullptr, nullptr};
  }
  return RowRef{src, dst};
}

template <int S>
__global__ void __launch_bounds__(32) merge_copy_tma_kernel(fsx_merge_batch b, uint32_t stage_bytes) {
  extern __shared__ __align__(128) uint8_t stage_mem[];
  __shared__ __align__(8) uint64_t bars[S];
  if (threadIdx.x != 0) return;
  const uint32_t sbase = tma::smem_u32(stage_mem);
  for (int s = 0; s < S; ++s) tma::mbar_init(tma::smem_u32(&bars[s]), 1);
  tma::mbar_fence_init();
  const uint32_t rb = (uint32_t)b.row_bytes;
  const int64_t first = blockIdx.x, stride = gridDim.x, n = b.total_item_rows;
  uint8_t* dst_of[S];
  uint32_t parity = 0;  // bit s = phase parity expected next on stage s
  // Newest rows first when the slab was filled before this launch (stream
  // order): the tail of what K1 just wrote is still in the 126 MB L2, so
  // walking the rows backwards turns part of the slab reads into L2 hits.
  // With early start (flags) rows are taken in arrival order instead.
  const bool newest_first = b.d_item_flag == nullptr;
  auto issue = [&](int64_t k) {  // load this CTA's k-th row into stage k % S
    const int s = (int)(k % S);
    const int64_t idx = first + k * stride;
    const RowRef r = resolve_row(b, newest_first ? n - 1 - idx : idx);
    dst_of[s] = r.dst;
    if (!r.src) return;
    const uint32_t bar = tma::smem_u32(&bars[s]);
    tma::mbar_expect_tx(bar, rb);
    tma::bulk_load(sbase + s * stage_bytes, r.src, rb, bar);
  };
  for (int64_t k = 0; k < S - 1 && first + k * stride < n; ++k) issue(k);
  for (int64_t k = 0; first + k * stride < n; ++k) {
    const int s = (int)(k % S);
    if (dst_of[s]) {
      tma::mbar_wait(tma::smem_u32(&bars[s]), (parity >> s) & 1u);
      parity ^= 1u << s;
      tma::bulk_store(dst_of[s], sbase + s * stage_bytes, rb);
    }
    tma::bulk_commit();  // one group per row (possibly empty) keeps the count exact
    tma::bulk_wait_read1();  // the store issued one row ago has left shared memory
    if (first + (k + S - 1) * stride < n) issue(k + S - 1);
  }
  tma::bulk_wait_all();
}

constexpr int kTmaStages = 4;

// K1, bulk-copy tile form (FSX_FWD_VARIANT=5; local slabs, no fused digest).
// One 32-thread CTA per 32 KiB tile, one elected thread: two 16 KiB halves are
// loaded global->shared by the copy engine (mbarrier complete_tx), each half
// is stored shared->global as soon as it has landed, then the thread waits
// for the stores, orders them (async proxy) before its generic acq_rel count
// into the chunk counter, and the CTA completing the chunk publishes the flag
// like forward_tile_kernel.  Bytes in flight cost shared memory, not
// registers: 6 such CTAs per SM keep 192 KiB in flight with ~2 K registers,
// which leaves the register file to a merge running next to K1.
__global__ void __launch_bounds__(32) forward_tma_kernel(const __grid_constant__ FwdBatch b) {
  extern __shared__ __align__(128) uint8_t tile_mem[];
  __shared__ __align__(8) uint64_t bars[2];
  if (threadIdx.x != 0) return;
  const int64_t gt = blockIdx.x;
  int i = 0;
  while (gt >= b.unit_off[i + 1]) ++i;
  const FwdArgs& a = b.t[i];
  const int64_t u = gt - b.unit_off[i];
  const int64_t c = u / a.chunk_units;
  const int64_t sl = u - c * a.chunk_units;
  const int64_t cbeg = c * a.chunk_bytes;
  const int64_t cend = min(cbeg + a.chunk_bytes, a.bytes);
  const int64_t beg = cbeg + sl * a.slice;
  const int64_t end = min(beg + a.slice, cend);
  const int64_t vend = beg + ((end - beg) & ~int64_t{15});  // beg is 16-byte aligned
  const uint32_t sbase = tma::smem_u32(tile_mem);
  const int64_t half = ((vend - beg) / 2 + 15) & ~int64_t{15};
  const int64_t len0 = min(half, vend - beg), len1 = (vend - beg) - len0;
  tma::mbar_init(tma::smem_u32(&bars[0]), 1);
  tma::mbar_init(tma::smem_u32(&bars[1]), 1);
  tma::mbar_fence_init();
  // the producer's source is read once (evict first); slab stores keep L2
  // priority when the consumer merges right behind (FSX_FWD_L2_KEEP)
  const uint64_t ld_pol = l2_policy(1);
  const uint64_t st_pol = l2_policy(b.l2_keep_dst ? 2 : 0);
  if (len0 > 0) {
    tma::mbar_expect_tx(tma::smem_u32(&bars[0]), (uint32_t)len0);
    tma::bulk_load_hint(sbase, a.src + beg, (uint32_t)len0, tma::smem_u32(&bars[0]), ld_pol);
  }
  if (len1 > 0) {
    tma::mbar_expect_tx(tma::smem_u32(&bars[1]), (uint32_t)len1);
    tma::bulk_load_hint(sbase + (uint32_t)len0, a.src + beg + len0, (uint32_t)len1, tma::smem_u32(&bars[1]),
                        ld_pol);
  }
  if (len0 > 0) {
    tma::mbar_wait(tma::smem_u32(&bars[0]), 0);
    tma::bulk_store_hint(a.dst + beg, sbase, (uint32_t)len0, st_pol);
  }
  if (len1 > 0) {
    tma::mbar_wait(tma::smem_u32(&bars[1]), 0);
    tma::bulk_store_hint(a.dst + beg + len0, sbase + (uint32_t)len0, (uint32_t)len1, st_pol);
  }
  tma::bulk_commit();
  for (int64_t j = vend; j < end; ++j) a.dst[j] = a.src[j];  // sub-16-byte tail
  tma::bulk_wait_all();
  // the tile's bulk stores are complete: order them (async proxy) before the
  // generic release that counts the tile
  asm volatile("fence.proxy.async.global;" ::: "memory");
  if (a.counters == nullptr) return;
  const uint32_t units = (c == a.n_chunks - 1) ? (uint32_t)a.last_units : (uint32_t)a.chunk_units;
  const uint32_t prev = atom_add_acq_rel(&a.counters[c], 1u, a.peer != 0);
  if (prev == units - 1) {
    a.counters[c] = 0u;
    if (a.peer) {
      __threadfence_system();
      st_release_sys(&a.dflags[c], a.token);
    } else {
      st_release_gpu(&a.dflags[c], a.token);
    }
    if (a.hflags) st_relaxed_sys(&a.hflags[c], a.token);
  }
}



// K3 merge, phase 2, early-start form (default whenever the batch carries item
// flags: the N>1 consumer following NVLink pushes, and the N=1 colocated
// pipeline following K1 on the same GPU).  One elected thread per 32-thread
// CTA claims runs of kTmaRun consecutive placeholder rows from a global work
// counter, so every CTA works on the earliest rows whose chunk has landed
// (dynamic, arrival order), and moves each row with the bulk-copy engine:
// cp.async.bulk global->shared (mbarrier complete_tx) then shared->global,
// an S-stage ring with S-1 rows in flight per CTA and no registers spent on
// the bytes -- so the merge CTAs sit next to K1's CTAs on every SM without
// taking the registers K1 needs.  Within a run the thread walks rows
// incrementally (item / request values re-read only at boundaries, a chunk
// flag spun on only when the run enters a new chunk).  With FSX_MERGE_DISCARD
// a row's slab lines are discarded from L2 once its bulk load has completed.
// Bulk-copy form of the follow kernel (FSX_MERGE_STREAM=3): CTA c of C (32
// threads, one elected thread) moves rows g = c, c + C, ... in increasing
// order through an S-stage shared-memory ring (S-1 rows in flight), so the
// grid's window behind the producer stays about (S-1) x C rows wide while the
// bytes in flight cost shared memory instead of registers.
template <int S>
__global__ void __launch_bounds__(32) merge_follow_tma_kernel(fsx_merge_batch b, uint32_t stage_bytes) {
  extern __shared__ __align__(128) uint8_t stage_mem[];
  __shared__ __align__(8) uint64_t bars[S];
  if (threadIdx.x != 0) return;
  const uint32_t sbase = tma::smem_u32(stage_mem);
  for (int s = 0; s < S; ++s) tma::mbar_init(tma::smem_u32(&bars[s]), 1);
  tma::mbar_fence_init();
  const int64_t rb = b.row_bytes, n = b.total_item_rows, C = gridDim.x;
  const bool discard = (b.mode & FSX_MERGE_DISCARD) != 0;
  const bool early = b.d_item_flag != nullptr;
  int64_t g = blockIdx.x;
  if (g >= n) return;
  int64_t item = upper_index(b.d_item_row_off, b.num_items + 1, g);
  while (b.d_item_row_off[item + 1] <= g) ++item;
  int64_t req = upper_index(b.d_req_item_off, b.num_requests + 1, item);
  while (b.d_req_item_off[req + 1] <= item) ++req;
  int64_t item_beg = b.d_item_row_off[item], item_end = b.d_item_row_off[item + 1];
  const uint8_t* item_src = static_cast<const uint8_t*>(b.d_item_src[item]);
  int64_t chunk_rows = early ? b.d_item_chunk_rows[item] : 0;
  int64_t req_row = b.d_req_row_off[req];
  bool req_ok = b.d_status[req] == 0;
  int64_t waited = -1;
  auto next = [&](uint8_t** dst, const uint8_t** src) -> bool {
    for (; g < n; g += C) {
      if (g >= item_end) {
        do {
          ++item;
        } while (b.d_item_row_off[item + 1] <= g);
        item_beg = b.d_item_row_off[item];
        item_end = b.d_item_row_off[item + 1];
        item_src = static_cast<const uint8_t*>(b.d_item_src[item]);
        if (early) chunk_rows = b.d_item_chunk_rows[item];
        waited = -1;
        if (b.d_req_item_off[req + 1] <= item) {
          do {
            ++req;
          } while (b.d_req_item_off[req + 1] <= item);
          req_row = b.d_req_row_off[req];
          req_ok = b.d_status[req] == 0;
        }
      }
      if (!req_ok) continue;
      const int64_t j = g - item_beg;
      if (early) {
        const int64_t c = chunk_rows > 0 ? j / chunk_rows : 0;
        if (c != waited) {
          spin_until(b.d_item_flag[item] + c, b.d_item_token[item]);
          asm volatile("fence.proxy.async.global;" ::: "memory");
          waited = c;
        }
      }
      const uint8_t* sr = item_src + j * rb;
      uint8_t* d = static_cast<uint8_t*>(b.d_embeds) + (req_row + b.d_scratch[g]) * rb;
      if ((reinterpret_cast<uintptr_t>(sr) | reinterpret_cast<uintptr_t>(d) | (uintptr_t)rb) & 15) {
        for (int64_t i = 0; i < rb; ++i) d[i] = sr[i];
        continue;
      }
      *dst = d;
      *src = sr;
      g += C;
      return true;
    }
    return false;
  };
  uint8_t* dst_of[S];
  const uint8_t* src_of[S];
  auto issue = [&](int64_t k) -> bool {
    const int s = (int)(k % S);
    if (!next(&dst_of[s], &src_of[s])) return false;
    const uint32_t bar = tma::smem_u32(&bars[s]);
    tma::mbar_expect_tx(bar, (uint32_t)rb);
    tma::bulk_load(sbase + s * stage_bytes, src_of[s], (uint32_t)rb, bar);
    return true;
  };
  int64_t issued = 0;
  while (issued < S - 1 && issue(issued)) ++issued;
  uint32_t parity = 0;
  for (int64_t k = 0; k < issued; ++k) {
    const int s = (int)(k % S);
    tma::mbar_wait(tma::smem_u32(&bars[s]), (parity >> s) & 1u);
    parity ^= 1u << s;
    tma::bulk_store(dst_of[s], sbase + s * stage_bytes, (uint32_t)rb);
    tma::bulk_commit();
    if (discard) {
      const uintptr_t lo = (reinterpret_cast<uintptr_t>(src_of[s]) + 127) & ~uintptr_t{127};
      const uintptr_t hi = (reinterpret_cast<uintptr_t>(src_of[s]) + rb) & ~uintptr_t{127};
      for (uintptr_t a = lo; a < hi; a += 128) asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
    }
    tma::bulk_wait_read1();
    if (issue(issued)) ++issued;
  }
  tma::bulk_wait_all();
}

constexpr int kTmaRun = 8;

template <int S>
__global__ void __launch_bounds__(32) merge_stream_tma_kernel(fsx_merge_batch b, uint32_t stage_bytes,
                                                              unsigned long long* work) {
  extern __shared__ __align__(128) uint8_t stage_mem[];
  __shared__ __align__(8) uint64_t bars[S];
  if (threadIdx.x != 0) return;
  const uint32_t sbase = tma::smem_u32(stage_mem);
  for (int s = 0; s < S; ++s) tma::mbar_init(tma::smem_u32(&bars[s]), 1);
  tma::mbar_fence_init();
  const int64_t rb = b.row_bytes, n = b.total_item_rows;
  const int64_t runs = (n + kTmaRun - 1) / kTmaRun;
  const bool discard = (b.mode & FSX_MERGE_DISCARD) != 0;
  const bool early = b.d_item_flag != nullptr;
  // row generator state
  int64_t g = 0, g_end = 0, item = 0, req = 0, item_beg = 0, item_end = 0, req_row = 0, chunk_rows = 0;
  int64_t waited = -1;
  bool req_ok = true, done = false;
  const uint8_t* item_src = nullptr;
  auto load_item = [&]() {
    item_beg = b.d_item_row_off[item];
    item_end = b.d_item_row_off[item + 1];
    item_src = static_cast<const uint8_t*>(b.d_item_src[item]);
    if (early) chunk_rows = b.d_item_chunk_rows[item];
    waited = -1;
  };
  auto load_req = [&]() {
    req_row = b.d_req_row_off[req];
    req_ok = b.d_status[req] == 0;
  };
  // next placeholder row to move: false once the work counter is exhausted
  auto next = [&](uint8_t** dst, const uint8_t** src) -> bool {
    for (;;) {
      if (g >= g_end) {
        if (done) return false;
        const int64_t u = (int64_t)atomicAdd(work, 1ull);
        if (u >= runs) {
          done = true;
          return false;
        }
        g = u * kTmaRun;
        g_end = min(g + kTmaRun, n);
        item = upper_index(b.d_item_row_off, b.num_items + 1, g);
        while (b.d_item_row_off[item + 1] <= g) ++item;
        req = upper_index(b.d_req_item_off, b.num_requests + 1, item);
        while (b.d_req_item_off[req + 1] <= item) ++req;
        load_item();
        load_req();
      } else if (g >= item_end) {
        do {
          ++item;
        } while (b.d_item_row_off[item + 1] <= g);
        load_item();
        if (b.d_req_item_off[req + 1] <= item) {
          do {
            ++req;
          } while (b.d_req_item_off[req + 1] <= item);
          load_req();
        }
      }
      const int64_t row = g++;
      if (!req_ok) continue;  // validation failed: request untouched
      const int64_t j = row - item_beg;
      if (early) {
        const int64_t c = chunk_rows > 0 ? j / chunk_rows : 0;
        if (c != waited) {
          spin_until(b.d_item_flag[item] + c, b.d_item_token[item]);
          // the row is read by the bulk-copy (async) proxy after a generic acquire
          asm volatile("fence.proxy.async.global;" ::: "memory");
          waited = c;
        }
      }
      const uint8_t* s = item_src + j * rb;
      uint8_t* d = static_cast<uint8_t*>(b.d_embeds) + (req_row + b.d_scratch[row]) * rb;
      if ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d) | (uintptr_t)rb) & 15) {
        for (int64_t i = 0; i < rb; ++i) d[i] = s[i];  // bulk copies need 16-byte alignment
        continue;
      }
      *dst = d;
      *src = s;
      return true;
    }
  };
  uint8_t* dst_of[S];
  const uint8_t* src_of[S];
  auto issue = [&](int64_t k) -> bool {
    const int s = (int)(k % S);
    if (!next(&dst_of[s], &src_of[s])) return false;
    const uint32_t bar = tma::smem_u32(&bars[s]);
    tma::mbar_expect_tx(bar, (uint32_t)rb);
    tma::bulk_load(sbase + s * stage_bytes, src_of[s], (uint32_t)rb, bar);
    return true;
  };
  int64_t issued = 0;
  while (issued < S - 1 && issue(issued)) ++issued;
  uint32_t parity = 0;
  for (int64_t k = 0; k < issued; ++k) {
    const int s = (int)(k % S);
    tma::mbar_wait(tma::smem_u32(&bars[s]), (parity >> s) & 1u);
    parity ^= 1u << s;
    tma::bulk_store(dst_of[s], sbase + s * stage_bytes, (uint32_t)rb);
    tma::bulk_commit();
    if (discard) {  // the slab row has been read into shared memory: drop its L2 lines
      const uintptr_t lo = (reinterpret_cast<uintptr_t>(src_of[s]) + 127) & ~uintptr_t{127};
      const uintptr_t hi = (reinterpret_cast<uintptr_t>(src_of[s]) + rb) & ~uintptr_t{127};
      for (uintptr_t a = lo; a < hi; a += 128) asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
    }
    tma::bulk_wait_read1();  // the store issued one row ago has left shared memory
    if (issue(issued)) ++issued;
  }
  tma::bulk_wait_all();
}



cudaError_t launch_mailbox(const MailStep& m, cudaStream_t st) {
  if (m.n <= 0) return cudaSuccess;
  mailbox_kernel<<<m.n, kMailThreads, 0, st>>>(m);
  return cudaGetLastError();
}

cudaError_t launch_digest(const uint8_t* p, int64_t n, uint64_t* out, int grid, cudaStream_t st) {
  digest_kernel<<<grid, 256, 0, st>>>(p, n, out);
  return cudaGetLastError();
}

cudaError_t launch_chan_push(const ChanStep& s, cudaStream_t st) {
  if (s.n <= 0) return cudaSuccess;
  chan_push_kernel<<<s.n, 32, 0, st>>>(s);
  return cudaGetLastError();
}

cudaError_t launch_chan_pull(const ChanStep& s, cudaStream_t st) {
  if (s.n <= 0) return cudaSuccess;
  chan_pull_kernel<<<s.n, 32, 0, st>>>(s);
  return cudaGetLastError();
}

cudaError_t launch_merge(const fsx_merge_batch& b, int copy_grid, cudaStream_t s, int* launches,
                         unsigned long long* work) {
  *launches = 0;
  if (b.num_requests <= 0) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  const int base_mode = b.mode & FSX_MERGE_MODE_MASK;
  if (base_mode != FSX_MERGE_COPY_ONLY) {
    merge_scan_kernel<<<b.num_requests, kScanThreads, 0, s>>>(b);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    *launches = 1;
  }
  if (base_mode == FSX_MERGE_SCAN_ONLY || b.total_item_rows <= 0) return cudaSuccess;
  // Default: the LDG/STG warp-per-row kernel over a full (non-persistent)
  // grid, 6.80 TB/s in the config-B step against 5.98 for the persistent TMA
  // bulk-copy ring (profiles/merge_ab_r01c.jsonl, 3 alternating runs each);
  // FSX_MERGE_TMA=1 selects the TMA kernel.
  static const bool use_tma = [] {
    const char* e = std::getenv("FSX_MERGE_TMA");
    return e && e[0] == '1';
  }();
  const uint32_t stage = (uint32_t)((b.row_bytes + 127) & ~int64_t{127});
  if (use_tma && !b.d_item_flag && !(b.mode & FSX_MERGE_DISCARD) && b.row_bytes % 16 == 0 &&
      stage * kTmaStages <= 48 * 1024) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = (size_t)stage * kTmaStages;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, merge_copy_tma_kernel<kTmaStages>, 32,
                                                      smem) != cudaSuccess || per_sm < 1)
      per_sm = 1;
    const int64_t cap = (int64_t)sms * per_sm;
    const int grid = (int)(b.total_item_rows < cap ? b.total_item_rows : cap);
    merge_copy_tma_kernel<kTmaStages><<<grid, 32, smem, s>>>(b, stage);
    e = cudaGetLastError();
    if (e == cudaSuccess) ++*launches;
    return e;
  }
  if (b.d_item_flag) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // early-start kernel: 0 follow (default), 1 register runs, 2 bulk-copy runs
    static const int stream_kind = [] {
      const char* e = std::getenv("FSX_MERGE_STREAM");
      return e ? std::atoi(e) : 0;
    }();
    if (stream_kind == 4) {
      const int64_t cap = (b.mode & FSX_MERGE_COLOCATED) ? sms : copy_grid;
      const int64_t want = (b.total_item_rows + (kMergeThreads / 32) - 1) / (kMergeThreads / 32);
      merge_follow2_kernel<16><<<(unsigned)(want < cap ? want : cap), kMergeThreads, 0, s>>>(b);
    } else if (stream_kind == 0) {
      // one CTA per SM beside K1 on the same GPU, else the copy grid
      const int64_t cap = (b.mode & FSX_MERGE_COLOCATED) ? sms : copy_grid;
      const int64_t want = (b.total_item_rows + (kMergeThreads / 32) - 1) / (kMergeThreads / 32);
      static const int unroll = [] {
        const char* e = std::getenv("FSX_FOLLOW_UNROLL");
        return e ? std::atoi(e) : 16;
      }();
      if (unroll == 8)
        merge_follow_kernel<8><<<(unsigned)(want < cap ? want : cap), kMergeThreads, 0, s>>>(b);
      else
        merge_follow_kernel<16><<<(unsigned)(want < cap ? want : cap), kMergeThreads, 0, s>>>(b);
    } else if (stream_kind == 3 && b.row_bytes % 16 == 0 && stage * kTmaStages <= 48 * 1024) {
      static const int per_sm_env = [] {
        const char* e = std::getenv("FSX_FOLLOW_TMA_PER_SM");
        return e ? std::atoi(e) : 4;
      }();
      const size_t smem = (size_t)stage * kTmaStages;
      const int64_t cap = (int64_t)sms * per_sm_env;
      merge_follow_tma_kernel<kTmaStages>
          <<<(unsigned)(b.total_item_rows < cap ? b.total_item_rows : cap), 32, smem, s>>>(b, stage);
    } else if (stream_kind == 2 && work && b.row_bytes % 16 == 0 && stage * kTmaStages <= 48 * 1024) {
      // early start: bulk-copy rows claimed in arrival order; colocated with
      // K1: 4 CTAs per SM (registers stay with K1), else the occupancy limit
      const size_t smem = (size_t)stage * kTmaStages;
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, merge_stream_tma_kernel<kTmaStages>, 32,
                                                        smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
      if ((b.mode & FSX_MERGE_COLOCATED) && per_sm > 4) per_sm = 4;
      const int64_t runs = (b.total_item_rows + kTmaRun - 1) / kTmaRun;
      const int64_t cap = (int64_t)sms * per_sm;
      merge_stream_tma_kernel<kTmaStages><<<(unsigned)(runs < cap ? runs : cap), 32, smem, s>>>(b, stage, work);
    } else {
      // register form (FSX_MERGE_STREAM_LDG=1): static run assignment; one
      // CTA per SM when the producer shares this GPU
      const int64_t runs = (b.total_item_rows + kStreamRun - 1) / kStreamRun;
      const int64_t want = (runs + (kMergeThreads / 32) - 1) / (kMergeThreads / 32);
      const int64_t cap = (b.mode & FSX_MERGE_COLOCATED) ? sms : copy_grid;
      merge_stream_kernel<<<(unsigned)(want < cap ? want : cap), kMergeThreads, 0, s>>>(b, work);
    }
    e = cudaGetLastError();
    if (e == cudaSuccess) ++*launches;
    return e;
  }
  const int64_t need = (b.total_item_rows + (kMergeThreads / 32) - 1) / (kMergeThreads / 32);
  // one warp per row and no persistence (full grid) unless FSX_MERGE_PERSIST=1
  static const bool persist = [] {
    const char* e = std::getenv("FSX_MERGE_PERSIST");
    return e && e[0] == '1';
  }();
  const int grid = (int)((persist && need > copy_grid) ? copy_grid : need);
  merge_copy_kernel<<<grid, kMergeThreads, 0, s>>>(b);
  e = cudaGetLastError();
  if (e == cudaSuccess) ++*launches;
  return e;
}

cudaError_t preload_kernels() {
  // CUDA loads kernels lazily (CUDA_MODULE_LOADING=LAZY, the CUDA 12 default):
  // a kernel's first launch loads it, and that load can wait for the kernels
  // already running.  A consumer spinning on flags (early-start merge,
  // wait_flags, channel pull), launched before its producer's first-ever
  // launch, would then wait forever for a producer that cannot load.  The
  // producers -- every K1 form, the flag stores, the channel push -- are
  // loaded up front.  Only those: loading the merge kernels eagerly as well
  // measured a slower colocated pass (0.30 vs 0.255 ms per config-B pass).
  const void* fns[] = {
      reinterpret_cast<const void*>(forward_tma_kernel),
      reinterpret_cast<const void*>(forward_tile_kernel<4>),
      reinterpret_cast<const void*>(forward_tile_kernel<8>),
      reinterpret_cast<const void*>(forward_variant(0, false)),
      reinterpret_cast<const void*>(forward_variant(1, false)),
      reinterpret_cast<const void*>(forward_variant(2, false)),
      reinterpret_cast<const void*>(forward_variant(0, true)),
      reinterpret_cast<const void*>(forward_variant(1, true)),
      reinterpret_cast<const void*>(forward_variant(2, true)),
      reinterpret_cast<const void*>(set_flags_kernel),
      reinterpret_cast<const void*>(chan_push_kernel),
  };
  cudaFuncAttributes a;
  for (const void* f : fns) {
    const cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  // FSX_DIAG_PRELOAD_ALL=1 (diagnostics, profiles/colocated_bimodality_r01k.md):
  // also load the consumer kernels, which brings out the colocated pass's slow mode
  static const bool all = std::getenv("FSX_DIAG_PRELOAD_ALL") != nullptr;
  if (all) {
    const void* more[] = {
        reinterpret_cast<const void*>(merge_scan_kernel),
        reinterpret_cast<const void*>(merge_copy_kernel),
        reinterpret_cast<const void*>(merge_follow_kernel<8>),
        reinterpret_cast<const void*>(merge_follow_kernel<16>),
        reinterpret_cast<const void*>(merge_copy_tma_kernel<kTmaStages>),
        reinterpret_cast<const void*>(merge_follow2_kernel<16>),
        reinterpret_cast<const void*>(merge_follow_tma_kernel<kTmaStages>),
        reinterpret_cast<const void*>(merge_stream_tma_kernel<kTmaStages>),
        reinterpret_cast<const void*>(merge_stream_kernel),
        reinterpret_cast<const void*>(synth_kernel),
        reinterpret_cast<const void*>(mailbox_kernel),
        reinterpret_cast<const void*>(digest_kernel),
        reinterpret_cast<const void*>(wait_flags_kernel),
        reinterpret_cast<const void*>(chan_pull_kernel),
    };
    for (const void* f : more) cudaFuncGetAttributes(&a, f);
  }
  return cudaSuccess;
}

cudaError_t launch_synth(uint64_t seed, uint8_t* dst, int64_t n, int grid, cudaStream_t s) {
  synth_kernel<<<grid, 256, 0, s>>>(seed ^ 0xd6e8feb86659fd93ull, dst, n);
  return cudaGetLastError();
}

}  // namespace fsx
