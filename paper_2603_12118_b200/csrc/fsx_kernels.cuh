// fsx_kernels.cuh -- kernel argument blocks and host launchers (internal to
// libfsx).  The kernels live in fsx_kernels.cu; the C ABI in fsx_runtime.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "fsx.h"

namespace fsx {

// K1: chunked push copy with per-chunk completion flags.
struct FwdArgs {
  const uint8_t* src;
  uint8_t* dst;        // slab view (local or peer-mapped)
  int64_t bytes;
  int64_t chunk_bytes; // > 0
  int64_t slice;       // bytes per work unit (multiple of 16)
  int64_t chunk_units; // units per full chunk
  int64_t last_units;  // units of the last chunk
  int64_t total_units;
  int32_t n_chunks;
  int32_t vec;         // 16-byte path usable
  int32_t peer;        // dst is peer (NVLink) memory: chunk flags published at system scope
  uint32_t* counters;  // [n_chunks] on the source device, zero on entry, self-resetting
  uint64_t* dflags;    // [n_chunks] consumer-device flags (may be peer memory)
  uint64_t* hflags;    // [n_chunks] mapped pinned host flags, or nullptr
  uint64_t token;
  uint64_t* digest;    // optional: += dg64 of the bytes (vec path; see fsx_kernels.cu)
};

// Up to kFwdMaxBatch transfers of one source device in one K1 launch (kernel
// parameter space: ~8.5 KB of the 32 KB sm_100 allows, so a 64-image batch is
// one launch instead of four back-to-back launches with four tails): units
// are laid out transfer-major, chunk-major.
// The launch copies only a block sized to the batch (FwdBatchT<1 | 8 | 64>):
// kernel parameters are copied per launch, and the full 64-transfer block
// (~8.5 KB) alone cost ~1.5 us per K1 launch, the floor of small transfers.
constexpr int kFwdMaxBatch = FSX_FWD_MAX_BATCH;
template <int CAP>
struct FwdBatchT {
  int32_t n;
  int32_t l2_keep_dst;     // slab stores with L2 evict_last (consumer merges next)
  int32_t peer_gpu_count;  // peer chunks: count tiles at gpu scope, publish once at sys scope
  int32_t small;           // 4 KiB tiles (batch <= 2 MiB): the latency form of K1
  int64_t unit_off[CAP + 1];
  FwdArgs t[CAP];
};
using FwdBatch = FwdBatchT<kFwdMaxBatch>;

// The tee (fsx_forward_merge): per item of one launch, where its slab copy goes
// and how its chunks complete.  Pieces are rows: chunk c of an item holds rows
// [c * chunk_rows, min((c + 1) * chunk_rows, rows)).
struct TeeItem {
  uint8_t* dst;        // slab segment (local or peer-mapped)
  uint32_t* counters;  // [n_chunks] on the launching device, zero on entry, self-resetting
  uint64_t* dflags;    // [n_chunks]
  uint64_t* hflags;    // [n_chunks] or nullptr
  uint64_t token;
  int64_t chunk_rows;  // >= 1
  int64_t rows;
  int32_t n_chunks;
  int32_t peer;
};
constexpr int kTeeMaxItems = 64;
struct TeeBatch {
  int32_t i0, n;           // items [i0, i0 + n) of the merge batch
  int64_t g0, g1;          // their placeholder rows [g0, g1)
  int32_t peer_gpu_count;  // as FwdBatch
  int32_t l2_keep_dst;     // slab copy stored with L2 evict_last
  TeeItem t[kTeeMaxItems];
};

struct FlagSetArgs {
  uint64_t* dflags;
  uint64_t* hflags;
  int32_t n;
  uint64_t token;
  // 1: the bytes behind the flags were written on THIS device (a copy into a
  // local slab): gpu-scope release of the device flag, relaxed host mirror,
  // as K1 publishes a local chunk.  0: system-scope release (peer or host
  // writers).
  int32_t gpu_scope = 0;
};

// Streaming channels (config C): per-token rows pushed into a consumer ring.
struct ChanRow {
  uint8_t* ring;        // consumer slab region: slots * row_bytes
  uint64_t* flags;      // consumer flags: slots (value = tag(seq))
  uint64_t* head;       // producer state (next seq to write), producer device
  uint64_t* tail;       // consumer state (next seq to read), consumer device
  uint64_t salt;        // tag(seq) = salt | (seq + 1)
  uint32_t slots;
  uint32_t row_bytes;
  int32_t peer;         // ring is peer memory
  int32_t _pad;
  uint8_t* io;          // this row's producer source (push) / consumer output (pull)
};
constexpr int kChanMaxRows = 48;
struct ChanStep {
  int32_t n;
  int32_t _pad;
  ChanRow c[kChanMaxRows];
};

// Small host messages (fsx_put_small): the small-message lane.  Each message
// is staged in a slot of a mapped pinned mailbox and described by a LaneDesc
// in a per-device ring of mapped pinned host memory; the host publishes it by
// advancing LaneCtl::tail.  A one-CTA service kernel on the destination
// device polls the tail, moves each message into its slab segment, digests the
// bytes it read and the bytes it reads back from the slab, and marks the
// descriptor done -- no launch and no event per message or per batch.  The
// kernel exits after kLaneIdleNs without work (so a device-wide synchronize
// never waits on it for long); the host relaunches it when it publishes into
// a lane whose kernel has announced its exit (LaneCtl::exit_epoch, a
// store/fence/load handshake on both sides, see lane_kernel).
struct LaneDesc {                 // 64 B, mapped pinned host memory
  uint8_t* dst;                   // slab destination (device)
  const uint8_t* src;             // staged bytes (mapped pinned host memory)
  int64_t n;                      // bytes (<= FSX_SMALL_MAX)
  uint64_t pub;                   // lane_pub(dst, src, n, seq), written last by the host
  uint64_t sent;                  // dg64 of the bytes read from src (kernel)
  uint64_t landed;                // dg64 of the bytes read back from dst (kernel)
  uint64_t done;                  // seq + 1 once sent/landed are written (kernel)
  uint64_t _pad;
};

// Publication mark of descriptor `seq`: a mix of its three fields and its
// sequence number.  The lane's poller reads a descriptor's first 32 bytes in
// one round trip and takes it as published only if the mark matches what it
// read -- a stale slot (an older sequence number) or a read torn by the
// host's concurrent writes fails the check and is polled again.
__host__ __device__ inline uint64_t lane_pub(uint64_t dst, uint64_t src, uint64_t n, uint64_t seq) {
  uint64_t z = (seq + 1) * 0x9e3779b97f4a7c15ull ^ dst;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull ^ src;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull ^ n;
  z = z ^ (z >> 31);
  return z | 1;  // never 0 (a cleared slot)
}
struct LaneCtl {                  // mapped pinned host memory, one per device
  uint64_t tail;                  // descriptors published (host)
  uint64_t _p0[7];
  uint64_t consumed;              // descriptors processed, written at kernel exit
  uint64_t _p1[7];
  uint64_t exit_epoch;            // epoch of the kernel that announced its exit
  uint64_t stop;                  // host: exit as soon as idle (fsx_close)
  uint64_t _p2[6];
};
constexpr int kLaneSlots = 4096;                 // descriptor ring
constexpr uint64_t kLaneIdleNs = 200ull * 1000;  // service kernel exits after 200 us idle

// Launchers return cudaError_t of the launch.  `grid` is chosen by the caller.
cudaError_t launch_digest(const uint8_t* p, int64_t n, uint64_t* out, int grid, cudaStream_t st);
cudaError_t launch_lane(LaneCtl* ctl, LaneDesc* ring, uint64_t epoch, cudaStream_t st);
cudaError_t launch_chan_push(const ChanStep& s, cudaStream_t st);
cudaError_t launch_chan_pull(const ChanStep& s, cudaStream_t st);
// bulk: the bulk-copy tile kernel when every transfer allows it (16-byte
// aligned, no fused digest), else the register tile kernel.
cudaError_t launch_forward(const FwdBatch& b, bool bulk, cudaStream_t s);
cudaError_t launch_set_flags(const FlagSetArgs& a, cudaStream_t s);
cudaError_t launch_wait_flags(const uint64_t* dflags, int32_t n, uint64_t token, cudaStream_t s);
// Scan and/or row copy per b.mode.
cudaError_t launch_merge(const fsx_merge_batch& b, cudaStream_t s, int* launches);
// The tee kernel over items [tb.i0, tb.i0 + tb.n) (positions / statuses from a
// scan already ordered before it on `s`).
cudaError_t launch_merge_tee(const fsx_merge_batch& b, const TeeBatch& tb, cudaStream_t s);
// Load the producer kernels (K1 forms, the tee, flag stores, channel push)
// now instead of at their first launch; called per device by fsx_open.
cudaError_t preload_kernels();
cudaError_t launch_synth(uint64_t seed, uint8_t* dst, int64_t n, int grid, cudaStream_t s);

// Device spin watchdog (spin_until traps after this long), current device.
cudaError_t set_spin_timeout(uint64_t ns);

// K1 tile bytes (one CTA per tile) and the early-start merge's occupancy.
int forward_tile_bytes();

}  // namespace fsx
