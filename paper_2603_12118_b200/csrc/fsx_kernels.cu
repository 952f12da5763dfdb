// fsx_kernels.cu -- sm_100a kernels of the sidecar data plane.
//
//   K0 synth_kernel         synth_payload_into (common.hpp:247-259) on the device
//   K1 forward_tile_kernel  payload placement of SidecarFabric::send/try_place_local
//      forward_tma_kernel   (sidecar.hpp:302-347, 465-483): a chunked push of the
//                           producer's bytes into the consumer slab (HBM or NVLink
//                           peer memory) with per-chunk completion flags; register
//                           tiles or bulk-copy (cp.async.bulk) tiles
//   K3 merge_scan_kernel    the consumer-side multimodal merge (derived contract,
//      merge_copy_kernel    SURVEY.md 8a-8; record_replay.hpp:404-416 slot order):
//      merge_follow_kernel  placeholder scan, then the row scatter -- stream
//      merge_colocated_kernel  ordered, or following the producer's chunk flags
//                           (producer on another GPU / beside it on this GPU)
//   K1+K3 merge_tee_kernel  the forward and the merge as one kernel: each item row
//                           is read once and stored into its slab segment (with
//                           the chunk flags) and into its placeholder row
//   flags / digest / small-message lane / channel kernels (see each)
//
// Everything here is integer byte movement: rows are opaque 16-byte vectors,
// never converted through a floating-point type, so bf16 NaN/Inf patterns in the
// synthetic payloads survive bit for bit.  No tensor cores: nothing is a
// contraction.  All kernels are HBM- or NVLink-bound; see DESIGN.md.
#include <cuda_runtime.h>
#include <stdint.h>

#include "fsx_kernels.cuh"

namespace fsx {
namespace kern {

constexpr int kTileThreads = 256;     // K1 register tiles: 256 threads x 8 x 16 B = 32 KiB
constexpr int kTileVecs = 8;
constexpr int kTmaTileBytes = 32768;  // K1 bulk-copy tile
constexpr int kMaxDevices = 64;       // per-device launch attributes
constexpr int kMergeThreads = 256;    // K3: one warp per placeholder row, 8 rows per CTA
constexpr int kMergeWarps = kMergeThreads / 32;
constexpr int kMergeUnroll = 16;      // 32 lanes x 16 x 16 B = 8 KiB of a row per batch
constexpr int kScanThreads = 1024;
constexpr int kScanRounds = 16;       // 1024 threads x 16 = 16384 token ids per round

// ---------------------------------------------------------------------------
// PTX helpers

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Coherent streaming load: used where the data may have been written by
// another kernel or a peer GPU during this kernel's lifetime (early start).
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

__device__ __forceinline__ void fence_sc_sys() { asm volatile("fence.sc.sys;" ::: "memory"); }

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Device spin on a completion flag.  A flag that never arrives (a producer
// that died, or a kernel the spinning CTAs keep from being scheduled) would
// hang the GPU, so after the watchdog time the kernel traps: the launch fails
// with an error the host sees instead of a hang.  Set per device by the
// runtime from FSX_SPIN_TIMEOUT_S (default 30 s).
__constant__ uint64_t c_spin_timeout_ns = 30ull * 1000000000ull;

template <bool kSys>
__device__ __forceinline__ void spin_until_scoped(const uint64_t* flag, uint64_t token) {
  auto load = [&] { return kSys ? ld_acquire_sys(flag) : ld_acquire_gpu(flag); };
  if (load() == token) return;
  const uint64_t t0 = globaltimer_ns();
  uint32_t n = 0;
  while (load() != token) {
    __nanosleep(64);
    if ((++n & 1023u) == 0 && globaltimer_ns() - t0 > c_spin_timeout_ns) asm volatile("trap;");
  }
}
// system scope: the producer is another GPU, another process or the host
__device__ __forceinline__ void spin_until(const uint64_t* flag, uint64_t token) {
  spin_until_scoped<true>(flag, token);
}
// gpu scope: producer and consumer on the same GPU (colocated early start)
__device__ __forceinline__ void spin_until_gpu(const uint64_t* flag, uint64_t token) {
  spin_until_scoped<false>(flag, token);
}

// splitmix64 finaliser (common.hpp:203-208): output k (1-based) of a stream
// with state s0 is mix(s0 + k * gamma), which makes every word independent.
__device__ __forceinline__ uint64_t splitmix_word(uint64_t s0, uint64_t k) {
  uint64_t z = s0 + k * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

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

__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t* p, uint32_t v, bool sys) {
  uint32_t old;
  if (sys)
    asm volatile("atom.add.acq_rel.sys.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  else
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// ---------------------------------------------------------------------------
// Chunk completion protocol (K1 and the tee kernel)
//
// A chunk is done when every piece of it (K1 tile, tee row) is stored.  The
// thread that finished a piece -- after a CTA barrier (register stores) or a
// bulk-group wait + proxy fence (bulk stores) has ordered the piece's stores
// before it -- adds the piece count to the chunk's counter with an acq_rel
// atomic; the arrival that completes the chunk resets the counter (the slot
// is clean for the next transfer that draws it) and publishes the token:
//   local slab     count at gpu scope, flag st.release.gpu (the counted
//                  pieces' stores happen-before it through the atomics);
//   peer slab,     count at system scope (every piece's stores are made
//   sys counting   visible at system scope by its own release), flag after
//                  fence.sc.sys with st.release.sys;
//   peer slab,     count at gpu scope (cheaper per piece: no system-scope
//   gpu counting   release per tile), and the completing thread makes every
//                  counted piece visible to the consumer GPU with one
//                  fence.sc.sys (cumulative over what its acquire observed)
//                  before st.release.sys of the flag (FSX_FWD_PEER_GPU_COUNT).
// The host mirror (hflags) is a posted store after the device flag.
__device__ __forceinline__ void complete_pieces(uint32_t* counter, uint32_t add, uint32_t need,
                                                bool peer, bool gpu_count, uint64_t* dflag,
                                                uint64_t* hflag, uint64_t token) {
  const uint32_t prev = atom_add_acq_rel(counter, add, peer && !gpu_count);
  if (prev + add != need) return;
  *counter = 0u;
  if (peer) {
    fence_sc_sys();
    st_release_sys(dflag, token);
  } else {
    st_release_gpu(dflag, token);
  }
  if (hflag) st_relaxed_sys(hflag, token);
}

__device__ __forceinline__ void count_tile(const FwdArgs& a, int64_t c, bool gpu_count) {
  const uint32_t need = (c == a.n_chunks - 1) ? (uint32_t)a.last_units : (uint32_t)a.chunk_units;
  complete_pieces(&a.counters[c], 1u, need, a.peer != 0, gpu_count, &a.dflags[c],
                  a.hflags ? &a.hflags[c] : nullptr, a.token);
}

// Tile gt of a forward batch: its transfer and byte range.
struct TileRef {
  int i;          // transfer
  int64_t u;      // unit within the transfer
  int64_t c;      // chunk
  int64_t beg, end;
};

template <class Batch>
__device__ __forceinline__ TileRef tile_of(const Batch& b, int64_t gt) {
  TileRef t;
  t.i = 0;
  while (gt >= b.unit_off[t.i + 1]) ++t.i;
  const FwdArgs& a = b.t[t.i];
  t.u = gt - b.unit_off[t.i];
  t.c = t.u / a.chunk_units;
  const int64_t s = t.u - t.c * a.chunk_units;
  const int64_t cbeg = t.c * a.chunk_bytes;
  const int64_t cend = min(cbeg + a.chunk_bytes, a.bytes);
  t.beg = cbeg + s * a.slice;
  t.end = min(t.beg + a.slice, cend);
  return t;
}

// ---------------------------------------------------------------------------
// K1, register tile form.  One CTA per 32 KiB tile, no persistence: the
// hardware CTA scheduler hands tiles to SMs as earlier ones retire, which on
// B200 sustains ~6.7 TB/s for a plain copy where a persistent grid-stride loop
// tops out near 5.9-6.3 (scripts/probe_sm_copy.cu).  Tiles are chunk-major in
// blockIdx order, so chunks complete roughly in order.  Each thread issues its
// 8 x 16 B loads (the producer's source is read once: L2 evict_first), then
// its stores; the CTA barriers and thread 0 counts the tile (protocol above).
// Optional fused dg64 of the source bytes (one atomic per tile).
template <int CAP>
__global__ void __launch_bounds__(kTileThreads) forward_tile_kernel(const __grid_constant__ FwdBatchT<CAP> b) {
  __shared__ uint64_t red[kTileThreads / 32];
  const TileRef tr = tile_of(b, blockIdx.x);
  const FwdArgs& a = b.t[tr.i];
  const int64_t beg = tr.beg, end = tr.end;
  const uint64_t ld_pol = l2_policy(1);
  const uint64_t st_pol = l2_policy(b.l2_keep_dst ? 2 : 0);
  const bool dig = a.digest != nullptr;
  uint64_t acc = 0;
  if (a.vec) {
    // beg is 16-byte aligned (slices and chunks are multiples of 16)
    const int64_t vend = end & ~int64_t{15};
    const int64_t nv = (vend - beg) >> 4;
    uint4 r[kTileVecs];
#pragma unroll
    for (int k = 0; k < kTileVecs; ++k) {
      const int64_t v = k * kTileThreads + threadIdx.x;
      if (v < nv) r[k] = ld_nc_v4_pol(a.src + beg + v * 16, ld_pol);
    }
#pragma unroll
    for (int k = 0; k < kTileVecs; ++k) {
      const int64_t v = k * kTileThreads + threadIdx.x;
      if (v < nv) st_v4_pol(a.dst + beg + v * 16, r[k], st_pol);
    }
    if (dig) {
#pragma unroll
      for (int k = 0; k < kTileVecs; ++k) {
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
  if (threadIdx.x != 0) return;
  if (dig) {
    uint64_t t = 0;
    for (int w = 0; w < kTileThreads / 32; ++w) t += red[w];
    if (tr.u == 0) t += (uint64_t)a.bytes * 0x9e3779b97f4a7c15ull;
    atomicAdd(reinterpret_cast<unsigned long long*>(a.digest), (unsigned long long)t);
  }
  count_tile(a, tr.c, b.peer_gpu_count != 0);
}

// K1, small-batch form: when the whole batch is <= 2 MiB a transfer is
// latency-bound, so tiles are 4 KiB -- one 16-byte vector per thread of a
// 256-thread CTA, one load round trip -- and the tile lookup is 32-bit (no
// 64-bit division on the path to the first load).  Same completion protocol
// and fused digest as the tile kernel; the runtime picks it (FwdBatch.small).
constexpr int kSmallTile = kTileThreads * 16;
template <int CAP>
__global__ void __launch_bounds__(kTileThreads) forward_small_kernel(const __grid_constant__ FwdBatchT<CAP> b) {
  __shared__ uint64_t red[kTileThreads / 32];
  const uint32_t gt = blockIdx.x;
  int i = 0;
  while (gt >= (uint32_t)b.unit_off[i + 1]) ++i;
  const FwdArgs& a = b.t[i];
  const uint32_t u = gt - (uint32_t)b.unit_off[i];
  const uint32_t cu = (uint32_t)a.chunk_units;
  const uint32_t c = u / cu;
  const uint32_t cbeg = c * (uint32_t)a.chunk_bytes;
  const uint32_t cend = min(cbeg + (uint32_t)a.chunk_bytes, (uint32_t)a.bytes);
  const uint32_t beg = cbeg + (u - c * cu) * (uint32_t)a.slice;  // slice <= kSmallTile
  const uint32_t end = min(beg + (uint32_t)a.slice, cend);
  uint64_t acc = 0;
  if (a.vec) {
    const uint32_t vend = end & ~15u;  // beg is 16-byte aligned
    const uint32_t at = beg + 16 * threadIdx.x;
    if (at < vend) {
      const uint4 r = __ldg(reinterpret_cast<const uint4*>(a.src + at));
      *reinterpret_cast<uint4*>(a.dst + at) = r;
      if (a.digest) acc = dg_vec(r, (uint64_t)(at >> 3));
    }
    if (threadIdx.x == 0 && vend < end) {
      for (uint32_t j = vend; j < end; ++j) a.dst[j] = a.src[j];
      if (a.digest) acc += dg_bytes(a.src, vend, end);
    }
  } else {
    for (uint32_t j = beg + threadIdx.x; j < end; j += kTileThreads) a.dst[j] = a.src[j];
  }
  if (a.digest) {
    acc = warp_sum_u64(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (a.digest) {
    uint64_t t = 0;
    for (int w = 0; w < kTileThreads / 32; ++w) t += red[w];
    if (u == 0) t += (uint64_t)a.bytes * 0x9e3779b97f4a7c15ull;
    atomicAdd(reinterpret_cast<unsigned long long*>(a.digest), (unsigned long long)t);
  }
  count_tile(a, c, b.peer_gpu_count != 0);
}

// ---------------------------------------------------------------------------
// Bulk-copy (TMA engine) helpers

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
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

}  // namespace tma

// K1, bulk-copy tile form (FSX_FWD_BULK).  One 32-thread CTA per 32 KiB tile,
// one elected thread: the tile's two 16 KiB halves are loaded global->shared by
// the copy engine (mbarrier complete_tx), each half is stored shared->global
// (cp.async.bulk, to this GPU's slab or to a peer's over NVLink) as soon as it
// has landed; then the thread waits for the stores to complete, orders them
// (async proxy) before its generic acq_rel count, and the tile is counted like
// the register form.  Bytes in flight cost shared memory, not registers.
template <int CAP>
__global__ void __launch_bounds__(32) forward_tma_kernel(const __grid_constant__ FwdBatchT<CAP> b) {
  extern __shared__ __align__(128) uint8_t tile_mem[];
  __shared__ __align__(8) uint64_t bars[2];
  if (threadIdx.x != 0) return;
  const TileRef tr = tile_of(b, blockIdx.x);
  const FwdArgs& a = b.t[tr.i];
  const int64_t beg = tr.beg, end = tr.end;
  const int64_t vend = beg + ((end - beg) & ~int64_t{15});  // beg is 16-byte aligned
  const uint32_t sbase = tma::smem_u32(tile_mem);
  const int64_t half = ((vend - beg) / 2 + 15) & ~int64_t{15};
  const int64_t len0 = min(half, vend - beg), len1 = (vend - beg) - len0;
  tma::mbar_init(tma::smem_u32(&bars[0]), 1);
  tma::mbar_init(tma::smem_u32(&bars[1]), 1);
  tma::mbar_fence_init();
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
  count_tile(a, tr.c, b.peer_gpu_count != 0);
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

// ---------------------------------------------------------------------------
// Small-message lane (fsx_put_small; LaneCtl / LaneDesc in fsx_kernels.cuh).
//
// One 1024-thread CTA per destination device serves the lane.  Warp 0 is the
// poller: it reads the next 8 descriptors (fields + publication mark, one
// PCIe round trip, ~1.2 us on the B200 hosts, scripts/probe_pcie_pull.cu),
// takes the ones whose mark matches their fields as published, copies them
// into a shared-memory cache and publishes the new tail to the workers in
// shared memory (the host's LaneCtl::tail only serves the exit handshake).  Warps 1..31 are workers: worker
// w moves messages m with m % 31 == w as soon as the shared tail passes m,
// independently of the others (no CTA barrier per batch, so messages
// published while others are in flight start at once).  A worker's lanes read
// 4 x 16 B of the staged bytes per round (volatile loads: mapped host memory
// is not L1-coherent and slots are reused), store them into the slab segment,
// digest them (`sent`), read the segment back (volatile, from L2) and digest
// that (`landed`); after __syncwarp lane 0 writes both digests and
// st.release.sys's done = seq + 1.
//
// Exit handshake (no cross-device atomics): once every worker has finished
// everything published and nothing new arrived for kLaneIdleNs, the poller
// stores `consumed` and exit_epoch = its epoch, fence.sc.sys, and re-reads
// the tail; the host publishes with store tail, mfence, load exit_epoch.  Of
// two racing sides at least one sees the other's store: either the poller
// sees the new tail and keeps serving (resetting exit_epoch), or the host
// sees the announcement and launches epoch + 1 behind it on the lane's
// stream, which resumes from `consumed`.  Workers only ever take messages
// below the tail the poller published, so an exiting instance and its
// successor never move the same message.  A spare instance is harmless (it
// starts after this one exits, finds nothing, idles out).
constexpr int kLaneThreads = 1024;
constexpr int kLaneWorkers = kLaneThreads / 32 - 1;
constexpr int kLaneUnroll = 4;
constexpr int kLaneCache = 256;  // shared descriptor cache (power of two)

__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_volatile_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint4 ld_volatile_v4(const void* p) {
  uint4 r;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}

__device__ __forceinline__ uint8_t ld_volatile_u8(const uint8_t* p) {
  uint16_t v;
  asm volatile("ld.volatile.global.u8 %0, [%1];" : "=h"(v) : "l"(p) : "memory");
  return (uint8_t)v;
}

// One worker warp moves one message (see above).
__device__ __forceinline__ void lane_move(LaneDesc* d, uint8_t* dst, const uint8_t* src, int n, uint64_t seq) {
  const int lane = threadIdx.x & 31;
  const bool vec = (((uintptr_t)dst | (uintptr_t)src) & 15) == 0;
  const int nv = vec ? n >> 4 : 0;
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  uint64_t sent = 0, landed = 0;
  for (int base = lane; base < nv; base += 32 * kLaneUnroll) {
    uint4 r[kLaneUnroll];
#pragma unroll
    for (int k = 0; k < kLaneUnroll; ++k)
      if (base + 32 * k < nv) r[k] = ld_volatile_v4(s4 + base + 32 * k);
#pragma unroll
    for (int k = 0; k < kLaneUnroll; ++k)
      if (base + 32 * k < nv) {
        st_v4(d4 + base + 32 * k, r[k]);
        sent += dg_vec(r[k], 2 * (uint64_t)(base + 32 * k));
      }
  }
  // sub-vector tail (and unaligned messages), lane 0, byte-wise
  const int from = nv * 16;
  if (lane == 0 && from < n) {
    for (int w8 = from >> 3; w8 * 8 < n; ++w8) {
      uint64_t v = 0;
      for (int b = 0; b < 8 && w8 * 8 + b < n; ++b) {
        const uint8_t x = ld_volatile_u8(src + w8 * 8 + b);
        dst[w8 * 8 + b] = x;
        v |= (uint64_t)x << (8 * b);
      }
      sent += dg_word(v, (uint64_t)w8);
    }
  }
  __syncwarp();
  for (int base = lane; base < nv; base += 32 * kLaneUnroll) {
    uint4 r[kLaneUnroll];
#pragma unroll
    for (int k = 0; k < kLaneUnroll; ++k)
      if (base + 32 * k < nv) r[k] = ld_volatile_v4(d4 + base + 32 * k);
#pragma unroll
    for (int k = 0; k < kLaneUnroll; ++k)
      if (base + 32 * k < nv) landed += dg_vec(r[k], 2 * (uint64_t)(base + 32 * k));
  }
  if (lane == 0 && from < n) {
    for (int w8 = from >> 3; w8 * 8 < n; ++w8) {
      uint64_t v = 0;
      for (int b = 0; b < 8 && w8 * 8 + b < n; ++b) v |= (uint64_t)ld_volatile_u8(dst + w8 * 8 + b) << (8 * b);
      landed += dg_word(v, (uint64_t)w8);
    }
  }
  sent = warp_sum_u64(sent);
  landed = warp_sum_u64(landed);
  __syncwarp();
  if (lane == 0) {
    const uint64_t len = (uint64_t)n * 0x9e3779b97f4a7c15ull;
    st_volatile_u64(&d->sent, sent + len);
    st_volatile_u64(&d->landed, landed + len);
    st_release_sys(&d->done, seq + 1);  // the warp's slab stores and the digests first
  }
}

__global__ void __launch_bounds__(kLaneThreads, 1) lane_kernel(LaneCtl* ctl, LaneDesc* ring, uint64_t epoch) {
  __shared__ uint64_t s_dst[kLaneCache], s_src[kLaneCache];
  __shared__ uint32_t s_n[kLaneCache];
  __shared__ uint64_t s_q[kLaneWorkers];  // per worker: its next message (all before it are done)
  __shared__ uint64_t s_tail;             // published to the workers
  __shared__ int s_exit;
  volatile uint64_t* vq = s_q;
  volatile uint64_t* vtail = &s_tail;
  volatile int* vexit = &s_exit;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t consumed = ld_volatile_u64(&ctl->consumed);
  if (threadIdx.x == 0) {
    s_tail = consumed;
    s_exit = 0;
  }
  if (warp > 0 && lane == 0) {
    const uint64_t w = (uint64_t)(warp - 1);
    s_q[w] = consumed + (w + kLaneWorkers - consumed % kLaneWorkers) % kLaneWorkers;
  }
  __syncthreads();
  if (warp == 0) {  // poller
    uint64_t pub = consumed;
    uint64_t idle_from = globaltimer_ns();
    for (;;) {
      // oldest message a worker may still read from the cache
      uint64_t oldest = lane < kLaneWorkers ? vq[lane] : ~0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) oldest = min(oldest, __shfl_xor_sync(0xffffffffu, oldest, o));
      // the next 8 descriptors in one round trip: lane l reads word l % 4 of
      // descriptor pub + l / 4 (the mark with acquire); a descriptor counts as
      // published when its mark matches the fields read beside it
      const uint64_t m = pub + (lane >> 2);
      const int wd = lane & 3;
      const uint64_t* dw = reinterpret_cast<const uint64_t*>(&ring[m % kLaneSlots]) + wd;
      const uint64_t v = wd == 3 ? ld_acquire_sys(dw) : ld_volatile_u64(dw);
      const int g0 = lane & ~3;
      const uint64_t f_dst = __shfl_sync(0xffffffffu, v, g0);
      const uint64_t f_src = __shfl_sync(0xffffffffu, v, g0 + 1);
      const uint64_t f_n = __shfl_sync(0xffffffffu, v, g0 + 2);
      const uint64_t f_pub = __shfl_sync(0xffffffffu, v, g0 + 3);
      const bool ok = f_pub == lane_pub(f_dst, f_src, f_n, m) && m < oldest + kLaneCache;
      const uint32_t okmask = __ballot_sync(0xffffffffu, ok && wd == 0);  // bit 4k: descriptor k
      // published descriptors in order from pub: the run of set bits 0, 4, 8, ...
      int count = 0;
      while (count < 8 && (okmask >> (4 * count)) & 1u) ++count;
      if (count > 0) {
        if (wd == 0 && (lane >> 2) < count) {
          const int c = (int)(m % kLaneCache);
          s_dst[c] = f_dst;
          s_src[c] = f_src;
          s_n[c] = (uint32_t)f_n;
        }
        __syncwarp();
        __threadfence_block();  // the cache entries before the tail the workers read
        const uint64_t t = pub + (uint64_t)count;
        if (lane == 0) *vtail = t;
        pub = t;
        idle_from = globaltimer_ns();
        continue;
      }
      // idle: every worker past everything published, nothing new for a while
      const bool drained = __all_sync(0xffffffffu, lane >= kLaneWorkers || vq[lane] >= pub);
      int leave = 0;
      if (drained && (globaltimer_ns() - idle_from > kLaneIdleNs || ld_volatile_u64(&ctl->stop) != 0)) {
        if (lane == 0) {
          st_volatile_u64(&ctl->consumed, pub);
          st_volatile_u64(&ctl->exit_epoch, epoch);
          fence_sc_sys();
          if (ld_acquire_sys(&ctl->tail) > pub) {
            st_volatile_u64(&ctl->exit_epoch, 0);  // keep serving
          } else {
            *vexit = 1;
            leave = 1;
          }
        }
        leave = __shfl_sync(0xffffffffu, leave, 0);
        if (leave) return;
      } else {
        __nanosleep(100);
      }
    }
  }
  // worker
  const int w = warp - 1;
  uint64_t q = s_q[w];
  for (;;) {
    if (*vtail <= q) {
      if (*vexit) return;
      __nanosleep(32);
      continue;
    }
    __threadfence_block();
    const int c = (int)(q % kLaneCache);
    lane_move(&ring[q % kLaneSlots], reinterpret_cast<uint8_t*>(s_dst[c]),
              reinterpret_cast<const uint8_t*>(s_src[c]), (int)s_n[c], q);
    q += kLaneWorkers;
    __syncwarp();
    if (lane == 0) vq[w] = q;
  }
}

__global__ void set_flags_kernel(FlagSetArgs a) {
  for (int i = threadIdx.x; i < a.n; i += blockDim.x) {
    if (a.gpu_scope) {
      st_release_gpu(&a.dflags[i], a.token);
      if (a.hflags) st_relaxed_sys(&a.hflags[i], a.token);
    } else {
      st_release_sys(&a.dflags[i], a.token);
      if (a.hflags) st_release_sys(&a.hflags[i], a.token);
    }
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
// its prompt row (index into d_embeds) written to
// scratch[item_row_off[first item] + k]; a request that fails validation gets
// -1 in all of its entries.  The copy kernels then need no request lookup.
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
        if (kk < want) b.d_scratch[kbase + kk] = (int32_t)(wbase + 32 * j);
      }
      k += __popc(m[j]);
    }
    __syncthreads();
    if (threadIdx.x == 0) running += tile_total;
    __syncthreads();
  }
  // (every thread has read `running` after the last barrier)
  if (running != want) {
    // validation failed: the request's rows are marked -1, so the copy
    // kernels leave its prompt untouched without looking the request up
    for (int64_t k = threadIdx.x; k < want; k += kScanThreads) b.d_scratch[kbase + k] = -1;
  }
  if (threadIdx.x == 0) b.d_status[r] = (running == want) ? 0 : FSX_E_VALIDATION;
}

// Item of placeholder row g, searched by the whole warp: the largest item i
// in [0, M) with item_row_off[i] <= g (zero-row items share an offset with
// the next item and are skipped by taking the largest).  Each round the 32
// lanes probe 32 evenly spaced offsets of the remaining range [lo, hi) and a
// ballot picks the sub-range, so M <= 32 items take one round of loads and
// M <= 1024 two -- where a binary search (and the request search after it)
// cost ~12 dependent loads per row, most of a warp's life on small rows.
// Invariant: off[lo] <= g < off[hi] (off[M] = total rows > g).
__device__ __forceinline__ int64_t warp_item_of(const int64_t* off, int64_t m, int64_t g, int lane) {
  int64_t lo = 0, hi = m;
  while (hi - lo > 1) {
    const int64_t span = hi - lo;
    const int64_t idx = lo + (span * lane) / 32;  // lane 0 probes lo
    const uint32_t le = __ballot_sync(0xffffffffu, off[idx] <= g);
    const int top = 31 - __clz(le);  // offsets are non-decreasing: le is a prefix of lanes
    const int64_t nlo = lo + (span * top) / 32;
    hi = top == 31 ? hi : lo + (span * (top + 1)) / 32;
    lo = nlo;
  }
  return lo;
}

// Store of one 16-byte vector with an optional L2 policy (pol < 0: plain).
__device__ __forceinline__ void st_v4_maybe_pol(void* p, const uint4& v, int pol, uint64_t policy) {
  if (pol < 0) st_v4(p, v);
  else st_v4_pol(p, v, policy);
}

// One row moved by one warp: all loads of a batch of the row in flight before
// its stores; `dst2` (optional) receives the same bytes (the tee kernel's slab
// segment).  pol / pol2: L2 policy of each destination's stores (-1 plain,
// else l2_policy's index).  Byte path when a row is not 16-byte aligned.
template <int U = kMergeUnroll>
__device__ __forceinline__ void warp_move_row(const uint8_t* src, uint8_t* dst, uint8_t* dst2, int64_t rb,
                                              int lane, bool coherent, int pol, int pol2) {
  const bool vec = ((rb & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) |
                     reinterpret_cast<uintptr_t>(dst2)) & 15) == 0;
  if (!vec) {
    for (int64_t i = lane; i < rb; i += 32) {
      const uint8_t v = src[i];
      if (dst) dst[i] = v;
      if (dst2) dst2[i] = v;
    }
    return;
  }
  const uint64_t policy = pol >= 0 ? l2_policy(pol) : 0;
  const uint64_t policy2 = pol2 >= 0 ? l2_policy(pol2) : 0;
  const int64_t nv = rb >> 4;
  const uint4* s = reinterpret_cast<const uint4*>(src);
  for (int64_t base = 0; base < nv; base += 32 * U) {
    uint4 r[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t i = base + k * 32 + lane;
      if (i < nv) r[k] = coherent ? ld_v4(s + i) : ld_nc_v4(s + i);
    }
    if (dst) {
      uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = base + k * 32 + lane;
        if (i < nv) st_v4_maybe_pol(d + i, r[k], pol, policy);
      }
    }
    if (dst2) {
      uint4* d = reinterpret_cast<uint4*>(dst2);
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t i = base + k * 32 + lane;
        if (i < nv) st_v4_maybe_pol(d + i, r[k], pol2, policy2);
      }
    }
  }
}

__device__ __forceinline__ void discard_row(const uint8_t* src, int64_t rb, int lane) {
  // drop a merged slab row's lines from L2 without writing them back (whole
  // 128-byte lines only): the segment is dead until it is released
  const uintptr_t lo = (reinterpret_cast<uintptr_t>(src) + 127) & ~uintptr_t{127};
  const uintptr_t hi = (reinterpret_cast<uintptr_t>(src) + rb) & ~uintptr_t{127};
  for (uintptr_t a = lo + 128 * (uintptr_t)lane; a < hi; a += 128 * 32)
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
}

// K3 merge, phase 2: one warp per placeholder row over a full (non-persistent)
// grid, 8 rows per CTA.  Lane 0 resolves the row's item and request (binary
// searches over the row offsets), then the warp moves the row with all of its
// 16-byte loads in flight.  kGated (early start, producer on another GPU or in
// another process): lane 0 first acquires the flag of the chunk the row sits
// in.  The hardware hands out CTAs in blockIdx (row) order and the producer
// completes chunks in the same order, so the resident CTAs are the ones right
// behind the producer; with every flag already set the gated form runs at the
// stream-ordered form's rate (the persistent grid-stride form it replaces
// reached 0.88 of the copy peak alone, bench r02b `kernels.follow`).
template <bool kGated, int U = kMergeUnroll>
__device__ __forceinline__ void merge_row(const fsx_merge_batch& b) {
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * kMergeWarps + (threadIdx.x >> 5);
  if (g >= b.total_item_rows) return;
  const int32_t row = b.d_scratch[g];  // prompt row, -1: request failed validation
  const int64_t item = warp_item_of(b.d_item_row_off, b.num_items, g, lane);
  if (row < 0) return;  // validation failed: request untouched
  const int64_t rb = b.row_bytes;
  const int64_t j = g - b.d_item_row_off[item];
  if (kGated) {
    if (lane == 0) {
      const int64_t cr = b.d_item_chunk_rows[item];
      spin_until(b.d_item_flag[item] + (cr > 0 ? j / cr : 0), b.d_item_token[item]);
    }
    __syncwarp();
  }
  const uint8_t* src = static_cast<const uint8_t*>(b.d_item_src[item]) + j * rb;
  uint8_t* dst = static_cast<uint8_t*>(b.d_embeds) + (int64_t)row * rb;
  warp_move_row<U>(src, dst, nullptr, rb, lane, /*coherent=*/true, -1, -1);
  if (b.mode & FSX_MERGE_DISCARD) discard_row(src, rb, lane);
}

// stream-ordered: the slab segments are complete when the kernel starts
__global__ void __launch_bounds__(kMergeThreads) merge_copy_kernel(fsx_merge_batch b) {
  merge_row<false>(b);
}

// early start behind a producer on another GPU / in another process.  Each
// warp's flag acquire is one more dependent round trip before its loads, so
// the gated form keeps more rows in flight: 3 CTAs per SM at 8 x 16 B per lane
constexpr int kFollowMinBlocksGated = 3;
__global__ void __launch_bounds__(kMergeThreads, kFollowMinBlocksGated) merge_follow_kernel(fsx_merge_batch b) {
  merge_row<true, 8>(b);
}

// K1 + K3 as one kernel (fsx_forward_merge): the tee.  Same grid as
// merge_copy_kernel over the placeholder rows of items [i0, i0 + n); each warp
// reads its item row ONCE from the producer's buffer and stores it twice --
// into the item's slab segment (the forward) and into its placeholder row
// (the merge; skipped for a request that failed validation, the forward still
// happens).  Chunk completion: the CTA barriers, then thread 0 walks its 8
// rows, groups consecutive rows of the same (item, chunk) and counts each
// group into that chunk's counter in rows (protocol above); zero-row items
// have their single flag published by CTA 0.
// Three CTAs per SM with 8 x 16 B in flight per lane (77 registers): 0.2196 ms
// per config-B pass against 0.240 for two CTAs per SM at 16 x 16 B, 0.222-0.226
// at 4 CTAs per SM (profiles/tee_variants_r02.txt).
constexpr int kTeeMinBlocks = 3;
constexpr int kTeeUnroll = 8;
__global__ void __launch_bounds__(kMergeThreads, kTeeMinBlocks) merge_tee_kernel(fsx_merge_batch b,
                                                                  const __grid_constant__ TeeBatch tb) {
  __shared__ int32_t s_item[kMergeWarps];
  __shared__ int64_t s_chunk[kMergeWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t g = tb.g0 + (int64_t)blockIdx.x * kMergeWarps + warp;
  int32_t key_item = -1;
  int64_t key_chunk = 0;
  if (g < tb.g1) {
    const int32_t row = b.d_scratch[g];  // prompt row, -1: request failed validation
    const int64_t item = warp_item_of(b.d_item_row_off, b.num_items, g, lane);
    const TeeItem& t = tb.t[item - tb.i0];
    const int64_t rb = b.row_bytes;
    const int64_t j = g - b.d_item_row_off[item];
    const uint8_t* src = static_cast<const uint8_t*>(b.d_item_src[item]) + j * rb;
    uint8_t* dst = row >= 0 ? static_cast<uint8_t*>(b.d_embeds) + (int64_t)row * rb : nullptr;
    // the prompt row is plain-stored; the slab copy keeps L2 priority when a
    // consumer on this GPU reads it next (FSX_FWD_L2_KEEP)
    warp_move_row<kTeeUnroll>(src, dst, t.dst + j * rb, rb, lane, /*coherent=*/false, -1, tb.l2_keep_dst ? 2 : -1);
    key_item = (int32_t)(item - tb.i0);
    key_chunk = j / t.chunk_rows;
  }
  if (lane == 0) {
    s_item[warp] = key_item;
    s_chunk[warp] = key_chunk;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int w = 0; w < kMergeWarps;) {
    const int32_t it = s_item[w];
    if (it < 0) break;  // rows past g1 are at the end of the CTA
    const int64_t c = s_chunk[w];
    int run = 1;
    while (w + run < kMergeWarps && s_item[w + run] == it && s_chunk[w + run] == c) ++run;
    const TeeItem& t = tb.t[it];
    const uint32_t need = (uint32_t)min(t.chunk_rows, t.rows - c * t.chunk_rows);
    complete_pieces(&t.counters[c], (uint32_t)run, need, t.peer != 0, tb.peer_gpu_count != 0, &t.dflags[c],
                    t.hflags ? &t.hflags[c] : nullptr, t.token);
    w += run;
  }
  if (blockIdx.x == 0) {
    for (int k = 0; k < tb.n; ++k) {
      const TeeItem& t = tb.t[k];
      if (t.rows != 0) continue;
      if (t.peer) {
        fence_sc_sys();
        st_release_sys(t.dflags, t.token);
      } else {
        st_release_gpu(t.dflags, t.token);
      }
      if (t.hflags) st_relaxed_sys(t.hflags, t.token);
    }
  }
}

// K3 merge, phase 2, early start beside a producer on THIS GPU (the colocated
// pass, FSX_MERGE_COLOCATED): a persistent grid of one CTA per SM, so spinning
// merge warps never take every slot the producer's K1 needs.  Warp w of W
// moves the placeholder rows g = w, w + W, w + 2W, ... in increasing order, so
// the grid works on a window of about W rows right behind the producer.
// Item / request values are re-read only when the warp's row crosses into the
// next item; lane 0 acquires the row's chunk flag (gpu scope, once per chunk)
// before the warp loads it.  FSX_MERGE_DISCARD drops merged slab lines from L2.
constexpr int kFollowMinBlocks = 3;
constexpr int kFollowUnroll = 8;
__global__ void __launch_bounds__(kMergeThreads, kFollowMinBlocks) merge_colocated_kernel(fsx_merge_batch b) {
  const int lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * kMergeWarps;
  const int64_t w = (int64_t)blockIdx.x * kMergeWarps + (threadIdx.x >> 5);
  const int64_t rb = b.row_bytes;
  const int64_t n = b.total_item_rows;
  if (w >= n) return;
  const bool discard = (b.mode & FSX_MERGE_DISCARD) != 0;
  int64_t item = warp_item_of(b.d_item_row_off, b.num_items, w, lane);
  int64_t item_beg = b.d_item_row_off[item], item_end = b.d_item_row_off[item + 1];
  const uint8_t* item_src = static_cast<const uint8_t*>(b.d_item_src[item]);
  int64_t chunk_rows = b.d_item_chunk_rows[item];
  int64_t waited = -1;
  for (int64_t g = w; g < n; g += W) {
    if (g >= item_end) {
      do {
        ++item;
      } while (b.d_item_row_off[item + 1] <= g);
      item_beg = b.d_item_row_off[item];
      item_end = b.d_item_row_off[item + 1];
      item_src = static_cast<const uint8_t*>(b.d_item_src[item]);
      chunk_rows = b.d_item_chunk_rows[item];
      waited = -1;
    }
    const int32_t row = b.d_scratch[g];
    if (row < 0) continue;  // validation failed: request untouched
    const int64_t j = g - item_beg;
    const int64_t c = chunk_rows > 0 ? j / chunk_rows : 0;
    if (c != waited) {
      if (lane == 0) spin_until_gpu(b.d_item_flag[item] + c, b.d_item_token[item]);
      __syncwarp();
      waited = c;
    }
    const uint8_t* src = item_src + j * rb;
    // the prompt rows are written once and not re-read here: evict them from
    // L2 first, so they do not push out slab rows the producer has just written
    warp_move_row<kFollowUnroll>(src, static_cast<uint8_t*>(b.d_embeds) + (int64_t)row * rb, nullptr, rb, lane,
                                 /*coherent=*/true, 1, -1);
    if (discard) discard_row(src, rb, lane);
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
    while (seq - (c.peer ? ld_acquire_sys(c.tail) : ld_acquire_gpu(c.tail)) >= c.slots) {
      __nanosleep(64);
      if ((++n & 1023u) == 0 && globaltimer_ns() - t0 > c_spin_timeout_ns) asm volatile("trap;");
    }
  }
  __syncwarp();
  uint8_t* dst = c.ring + (seq % c.slots) * (uint64_t)c.row_bytes;
  warp_copy_row(c.io, dst, c.row_bytes, lane);
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
  warp_copy_row(c.ring + slot * (uint64_t)c.row_bytes, c.io, c.row_bytes, lane);
  __syncwarp();
  // slot free for the producer: its reads are ordered before the tail store
  // (gpu scope when the producer shares this device -- a system-scope release
  // here cost ~3 us per pull launch -- system scope for a peer producer)
  if (lane == 0) {
    if (c.peer) {
      st_release_sys(c.tail, seq + 1);
    } else {
      st_release_gpu(c.tail, seq + 1);
    }
  }
}

}  // namespace kern

using namespace kern;

// ---------------------------------------------------------------------------
// Launchers

cudaError_t set_spin_timeout(uint64_t ns) {
  return cudaMemcpyToSymbol(c_spin_timeout_ns, &ns, sizeof(ns));
}

int forward_tile_bytes() { return kTileThreads * kTileVecs * 16; }

// One launch with the parameter block cut to CAP transfers.
template <int CAP>
cudaError_t launch_forward_cap(const FwdBatch& full, bool bulk, cudaStream_t s) {
  FwdBatchT<CAP> b;
  b.n = full.n;
  b.l2_keep_dst = full.l2_keep_dst;
  b.peer_gpu_count = full.peer_gpu_count;
  b.small = full.small;
  for (int k = 0; k <= full.n; ++k) b.unit_off[k] = full.unit_off[k];
  for (int k = 0; k < full.n; ++k) b.t[k] = full.t[k];
  const int64_t tiles = b.unit_off[b.n];
  if (tiles <= 0) return cudaSuccess;
  if (bulk) {
    // bulk-copy tiles need 16-byte aligned transfers and no fused digest;
    // a batch with any other transfer takes the register tile kernel
    bool ok = true;
    for (int k = 0; k < b.n; ++k) ok = ok && b.t[k].vec && !b.t[k].digest;
    if (ok) {
      // the opt-in shared-memory limit is a per-device function attribute
      static bool attr_set[kMaxDevices] = {};
      int dev = 0;
      cudaGetDevice(&dev);
      if (dev < kMaxDevices && !attr_set[dev]) {
        cudaFuncSetAttribute(forward_tma_kernel<CAP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kTmaTileBytes);
        attr_set[dev] = true;
      }
      forward_tma_kernel<CAP><<<(unsigned)tiles, 32, kTmaTileBytes, s>>>(b);
      return cudaGetLastError();
    }
  }
  if (b.small)
    forward_small_kernel<CAP><<<(unsigned)tiles, kTileThreads, 0, s>>>(b);
  else
    forward_tile_kernel<CAP><<<(unsigned)tiles, kTileThreads, 0, s>>>(b);
  return cudaGetLastError();
}

cudaError_t launch_forward(const FwdBatch& b, bool bulk, cudaStream_t s) {
  if (b.n <= 1) return launch_forward_cap<1>(b, bulk, s);
  if (b.n <= 8) return launch_forward_cap<8>(b, bulk, s);
  return launch_forward_cap<kFwdMaxBatch>(b, bulk, s);
}

cudaError_t launch_set_flags(const FlagSetArgs& a, cudaStream_t s) {
  set_flags_kernel<<<1, 32, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_wait_flags(const uint64_t* dflags, int32_t n, uint64_t token, cudaStream_t s) {
  wait_flags_kernel<<<1, 32, 0, s>>>(dflags, n, token);
  return cudaGetLastError();
}

cudaError_t launch_lane(LaneCtl* ctl, LaneDesc* ring, uint64_t epoch, cudaStream_t st) {
  lane_kernel<<<1, kLaneThreads, 0, st>>>(ctl, ring, epoch);
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

cudaError_t launch_merge(const fsx_merge_batch& b, cudaStream_t s, int* launches) {
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
  const int64_t need = (b.total_item_rows + kMergeWarps - 1) / kMergeWarps;
  if (b.d_item_flag && (b.mode & FSX_MERGE_COLOCATED)) {
    // early start beside a producer on this GPU: one resident CTA per SM
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    merge_colocated_kernel<<<(unsigned)(need < sms ? need : sms), kMergeThreads, 0, s>>>(b);
  } else if (b.d_item_flag) {
    merge_follow_kernel<<<(unsigned)need, kMergeThreads, 0, s>>>(b);
  } else {
    merge_copy_kernel<<<(unsigned)need, kMergeThreads, 0, s>>>(b);
  }
  e = cudaGetLastError();
  if (e == cudaSuccess) ++*launches;
  return e;
}

cudaError_t launch_merge_tee(const fsx_merge_batch& b, const TeeBatch& tb, cudaStream_t s) {
  const int64_t rows = tb.g1 - tb.g0;
  const int64_t grid = rows > 0 ? (rows + kMergeWarps - 1) / kMergeWarps : (tb.n > 0 ? 1 : 0);
  if (grid <= 0) return cudaSuccess;
  merge_tee_kernel<<<(unsigned)grid, kMergeThreads, 0, s>>>(b, tb);
  return cudaGetLastError();
}

cudaError_t preload_kernels() {
  // CUDA loads kernels lazily (CUDA_MODULE_LOADING=LAZY, the CUDA 12 default):
  // a kernel's first launch loads it, and that load can wait for the kernels
  // already running.  A consumer spinning on flags (early-start merge,
  // wait_flags, channel pull), launched before its producer's first-ever
  // launch, would then wait forever for a producer that cannot load.  The
  // producers -- both K1 forms, the tee, the flag stores, the channel push --
  // are loaded up front.  (Loading the consumer kernels eagerly as well made
  // the colocated early-start pass come up in its slow mode,
  // profiles/colocated_bimodality_r01k.md.)
  const void* fns[] = {
      reinterpret_cast<const void*>(forward_tma_kernel<1>),
      reinterpret_cast<const void*>(forward_tma_kernel<8>),
      reinterpret_cast<const void*>(forward_tma_kernel<kFwdMaxBatch>),
      reinterpret_cast<const void*>(forward_tile_kernel<1>),
      reinterpret_cast<const void*>(forward_tile_kernel<8>),
      reinterpret_cast<const void*>(forward_tile_kernel<kFwdMaxBatch>),
      reinterpret_cast<const void*>(forward_small_kernel<1>),
      reinterpret_cast<const void*>(forward_small_kernel<8>),
      reinterpret_cast<const void*>(forward_small_kernel<kFwdMaxBatch>),
      reinterpret_cast<const void*>(merge_tee_kernel),
      reinterpret_cast<const void*>(set_flags_kernel),
      reinterpret_cast<const void*>(chan_push_kernel),
      reinterpret_cast<const void*>(lane_kernel),
  };
  cudaFuncAttributes a;
  for (const void* f : fns) {
    const cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_synth(uint64_t seed, uint8_t* dst, int64_t n, int grid, cudaStream_t s) {
  synth_kernel<<<grid, 256, 0, s>>>(seed ^ 0xd6e8feb86659fd93ull, dst, n);
  return cudaGetLastError();
}

}  // namespace fsx
