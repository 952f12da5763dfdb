// fsx_runtime.cu -- the C ABI of libfsx (include/fsx.h): logical GPU map,
// per-consumer-GPU device receive slabs with the reference allocation policy,
// chunk-flag rings, and the launch paths of K0/K1/K3.
//
// Threading: every entry point is safe to call from any host thread (one mutex
// guards the bookkeeping; launches happen outside of it where possible).  The
// C++ fabric engine (include/fsx/fabric.hpp) calls in from the SimKernel
// thread and from its progress thread.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "fsx.h"
#include "fsx_kernels.cuh"
#include "nvtx3/nvToolsExt.h"

namespace {
// NVTX range over one C-ABI call (forward / merge / small-message flush /
// channel step), so nsys timelines and `ncu --nvtx` filters see the data
// plane's own phases.  Header-only NVTX v3: a no-op unless a tool attaches.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

namespace {

thread_local std::string t_err;

int fail(int code, const std::string& msg) {
  t_err = msg;
  return code;
}

#define FSX_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(FSX_E_INTERNAL, std::string(#call) + ": " + cudaGetErrorString(e_));   \
  } while (0)

constexpr int64_t kAlign = 64;             // sidecar.hpp:195
constexpr int64_t kFlagRing = 1 << 18;     // flags per consumer slab (2 MiB)
constexpr int64_t kCounterRing = 1 << 16;  // chunk counters per source device
// Address-ordered block list over [0, capacity).  First fit in offset order,
// 64-byte units, coalescing on free: the allocation policy of the reference
// NodeArena (sidecar.hpp:149-186), re-homed to a device slab.
class BlockList {
 public:
  void reset(int64_t capacity) {
    blocks_.clear();
    free_.clear();
    blocks_[0] = Block{capacity, true};
    free_[0] = capacity;
    used_segments_ = 0;
    used_bytes_ = 0;
    peak_ = 0;
  }

  // First fit in offset order, as NodeArena::allocate (sidecar.hpp:149-170);
  // the scan visits only free blocks (free_ mirrors the free entries of
  // blocks_), so its cost does not grow with the live segments.
  int64_t alloc(int64_t len) {
    const int64_t need = (std::max<int64_t>(len, 1) + kAlign - 1) & ~(kAlign - 1);
    for (auto fit = free_.begin(); fit != free_.end(); ++fit) {
      if (fit->second < need) continue;
      const int64_t off = fit->first;
      const int64_t rest = fit->second - need;
      auto it = blocks_.find(off);
      it->second = Block{need, false};
      free_.erase(fit);
      if (rest > 0) {
        blocks_.emplace_hint(std::next(it), off + need, Block{rest, true});
        free_.emplace(off + need, rest);
      }
      ++used_segments_;
      used_bytes_ += need;
      peak_ = std::max(peak_, used_bytes_);
      return off;
    }
    return -1;
  }

  // Free with coalescing of both neighbours (sidecar.hpp:172-186).
  bool release(int64_t off) {
    auto it = blocks_.find(off);
    if (it == blocks_.end() || it->second.free) return false;
    --used_segments_;
    used_bytes_ -= it->second.len;
    it->second.free = true;
    auto nx = std::next(it);
    if (nx != blocks_.end() && nx->second.free) {
      it->second.len += nx->second.len;
      free_.erase(nx->first);
      blocks_.erase(nx);
    }
    if (it != blocks_.begin()) {
      auto pv = std::prev(it);
      if (pv->second.free) {
        pv->second.len += it->second.len;
        blocks_.erase(it);
        free_[pv->first] = pv->second.len;
        return true;
      }
    }
    free_[it->first] = it->second.len;
    return true;
  }

  int64_t segments() const { return used_segments_; }
  int64_t bytes() const { return used_bytes_; }
  int64_t peak() const { return peak_; }

 private:
  struct Block {
    int64_t len;
    bool free;
  };
  std::map<int64_t, Block> blocks_;  // every block by offset
  std::map<int64_t, int64_t> free_;  // the free ones: offset -> len
  int64_t used_segments_ = 0, used_bytes_ = 0, peak_ = 0;
};

// Bump ring of contiguous index ranges (flags / counters / scratch).  Reuse
// of eager ranges is safe because flag values are unique tokens and counters
// reset themselves.  Ranges baked into a CUDA graph (taken, or named by a
// launch, while the stream is capturing) are pinned: replays keep using them
// for the life of the fabric, so the ring never hands them out again.
struct Ring {
  int64_t size = 0, next = 0;
  std::map<int64_t, int64_t> pinned;  // start -> end, disjoint
  // First free range of n at or after `next`, wrapping once; -1 when every
  // candidate overlaps a pinned range.
  int64_t take(int64_t n) {
    if (n > size) return -1;
    bool wrapped = false;
    for (;;) {
      if (next + n > size) {
        if (wrapped) return -1;
        wrapped = true;
        next = 0;
      }
      auto it = pinned.lower_bound(next + n);  // first pinned start >= end
      if (it != pinned.begin() && std::prev(it)->second > next) {
        next = std::prev(it)->second;  // overlaps a pinned range: skip past it
        continue;
      }
      const int64_t at = next;
      next += n;
      return at;
    }
  }
  void pin(int64_t at, int64_t n) {
    if (n <= 0) return;
    int64_t lo = at, hi = at + n;
    auto it = pinned.upper_bound(lo);
    if (it != pinned.begin() && std::prev(it)->second >= lo) --it;
    while (it != pinned.end() && it->first <= hi) {
      lo = std::min(lo, it->first);
      hi = std::max(hi, it->second);
      it = pinned.erase(it);
    }
    pinned[lo] = hi;
  }
};

// True while `st` is being captured into a CUDA graph.
bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive;
}

struct Slab {
  int gpu = -1;
  int device = -1;
  bool imported = false;
  uint8_t* base = nullptr;      // data region [0, capacity)
  int64_t capacity = 0;
  uint64_t* dflags = nullptr;   // kFlagRing device flags (right after the data region)
  uint64_t* hflags = nullptr;   // kFlagRing mapped pinned host flags (owner process only)
  BlockList blocks;
  Ring flags;
};

struct Device {
  int ordinal = -1;
  cudaStream_t stream = nullptr;
  uint32_t* counters = nullptr;
  Ring counter_ring;
  int sms = 0;
  uint64_t* state = nullptr;  // channel head/tail counters (kStatePool u64)
  int64_t state_next = 0;
  uint64_t* scratch = nullptr;  // short-lived u64 slots (digests), ring
  Ring scratch_ring;
  cudaStream_t notify = nullptr;     // flag stores of host->device forwards
  std::vector<cudaEvent_t> events;   // ring of copy-completion events
  uint64_t next_event = 0;
  // pinned staging ring for host->device copies from pageable memory
  // (fsx_forward_host): the host fills piece p+1 while the copy engine moves p
  std::mutex stage_mu;
  uint8_t* stage[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t stage_ev[3] = {nullptr, nullptr, nullptr};
  uint64_t stage_next = 0;
};

constexpr int64_t kStagePiece = int64_t{16} << 20;
constexpr int64_t kStageMin = int64_t{4} << 20;  // smaller pageable copies go direct

bool is_pinned_host(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// memcpy of a large piece on up to 4 threads (first-touched pageable source,
// pinned destination: one core moves ~15 GB/s on the B200 hosts)
// Persistent host copy workers for staging pageable spans (thread creation
// per piece cost more than the copy of a 2 MiB part).  min(15, cores - 1)
// threads; par_memcpy splits a piece across them and the calling thread.
class CopyPool {
 public:
  static CopyPool& get() {
    // never destroyed: the workers block on cv_ for the life of the process,
    // and destroying a condition variable with waiters at exit hangs in
    // pthread_cond_destroy (every C++ test binary hung after its last case)
    static CopyPool* pool = new CopyPool;
    return *pool;
  }
  int workers() const { return static_cast<int>(threads_.size()); }
  // Run fn(0..n-1) with part 0 on the caller; returns when all are done.
  void run(int n, const std::function<void(int)>& fn) {
    std::lock_guard<std::mutex> one(run_mu_);  // one job at a time (several devices may stage)
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &fn;
      parts_ = n;
      next_ = 1;
      pending_ = n - 1;
      ++epoch_;
    }
    cv_.notify_all();
    fn(0);
    for (;;) {  // help with parts not yet claimed
      int k;
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (next_ >= parts_) break;
        k = next_++;
      }
      fn(k);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_.notify_all();
    }
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  CopyPool() {
    const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
    const int n = static_cast<int>(std::min(15u, hw - 1));
    for (int i = 0; i < n; ++i) threads_.emplace_back([this] { loop(); });
    for (auto& t : threads_) t.detach();  // live for the process (static pool)
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return epoch_ != seen && job_ && next_ < parts_; });
      seen = epoch_;
      while (job_ && next_ < parts_) {
        const int k = next_++;
        const std::function<void(int)>* job = job_;
        lk.unlock();
        (*job)(k);
        lk.lock();
        if (--pending_ == 0) done_.notify_all();
      }
    }
  }
  std::mutex run_mu_, mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int parts_ = 0, next_ = 0, pending_ = 0;
  uint64_t epoch_ = 0;
  std::vector<std::thread> threads_;
};

// dg64 word terms (include/fsx.h, fsx_kernels.cu dg_word) of src[0, n), whose
// word 0 is word `word0` of the whole span, copying the bytes to dst on the
// way when dst is not null: one pass over the source for a staged host send
// (copy and digest were two passes, 6.4 ms per 112 MiB span).  n must be a
// multiple of 8 unless this piece ends the span (zero-padded last word).
uint64_t copy_digest(uint8_t* dst, const uint8_t* src, int64_t n, uint64_t word0) {
  constexpr uint64_t C1 = 0xbf58476d1ce4e5b9ull, C2 = 0x94d049bb133111ebull;
  uint64_t h0 = 0, h1 = 0, h2 = 0, h3 = 0;
  const int64_t words = n / 8;
  uint64_t c = (word0 + 1) * C1;
  int64_t k = 0;
  for (; k + 4 <= words; k += 4, c += 4 * C1) {
    uint64_t w[4];
    std::memcpy(w, src + k * 8, 32);
    if (dst) std::memcpy(dst + k * 8, w, 32);
    const uint64_t y0 = (w[0] ^ c) * C2, y1 = (w[1] ^ (c + C1)) * C2;
    const uint64_t y2 = (w[2] ^ (c + 2 * C1)) * C2, y3 = (w[3] ^ (c + 3 * C1)) * C2;
    h0 += y0 ^ (y0 >> 29);
    h1 += y1 ^ (y1 >> 29);
    h2 += y2 ^ (y2 >> 29);
    h3 += y3 ^ (y3 >> 29);
  }
  for (; k * 8 < n; ++k, c += C1) {
    uint64_t w = 0;
    const int64_t take = std::min<int64_t>(8, n - k * 8);
    std::memcpy(&w, src + k * 8, (size_t)take);
    if (dst) std::memcpy(dst + k * 8, &w, (size_t)take);
    const uint64_t y = (w ^ c) * C2;
    h0 += y ^ (y >> 29);
  }
  return h0 + h1 + h2 + h3;
}

// copy_digest split across the copy pool (parts at 64-byte boundaries).
uint64_t par_copy_digest(uint8_t* dst, const uint8_t* src, int64_t n, uint64_t word0) {
  CopyPool& pool = CopyPool::get();
  const int64_t parts = std::min<int64_t>(pool.workers() + 1, std::max<int64_t>(1, n / (int64_t{1} << 20)));
  if (parts < 2) return copy_digest(dst, src, n, word0);
  const int64_t per = ((n + parts - 1) / parts + 63) / 64 * 64;  // parts * per >= n
  std::vector<uint64_t> part(parts, 0);
  pool.run(static_cast<int>(parts), [&](int t) {
    const int64_t b = t * per, e = std::min(n, b + per);
    if (e > b) part[t] = copy_digest(dst ? dst + b : nullptr, src + b, e - b, word0 + b / 8);
  });
  uint64_t h = 0;
  for (uint64_t v : part) h += v;
  return h;
}

void par_memcpy(uint8_t* dst, const uint8_t* src, int64_t n) {
  CopyPool& pool = CopyPool::get();
  const int64_t parts = std::min<int64_t>(pool.workers() + 1, std::max<int64_t>(1, n / (int64_t{1} << 20)));
  if (parts < 2) {
    std::memcpy(dst, src, (size_t)n);
    return;
  }
  const int64_t per = ((n + parts - 1) / parts + 63) / 64 * 64;  // parts * per >= n
  pool.run(static_cast<int>(parts), [=](int t) {
    const int64_t b = t * per, e = std::min(n, b + per);
    if (e > b) std::memcpy(dst + b, src + b, (size_t)(e - b));
  });
}

constexpr size_t kEventRing = 1024;

constexpr int64_t kStatePool = 1 << 16;
constexpr int64_t kScratchRing = 1 << 14;

int digest_grid(const Device* d, int64_t n) {
  const int64_t want = (n / 16 + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)d->sms * 8));
}

// A streaming channel: one producer->consumer stream (a streaming DataRef,
// e.g. one request's thinker hidden states) delivered in seq order through a
// ring of `slots` rows in the consumer slab.
struct Channel {
  bool open = false;
  int src_gpu = -1, dst_gpu = -1, src_dev = -1, dst_dev = -1;
  int64_t ring_off = -1, flag_base = -1;
  uint32_t slots = 0, row_bytes = 0;
  uint64_t* head = nullptr;  // producer device
  uint64_t* tail = nullptr;  // consumer device
  uint64_t salt = 0;
};

}  // namespace

struct fsx_fabric {
  std::mutex mu;
  std::map<int, int> node_of;
  std::map<int, int> device_of;
  std::map<int, std::unique_ptr<Slab>> slabs;
  std::map<int, std::unique_ptr<Device>> devices;
  std::vector<Channel> channels;
  std::map<void*, int> ipc_maps;  // fsx_ipc_open mappings -> device
  // fsx_put_small: pinned mapped mailbox (first-fit slots for the staged
  // bytes), per destination device a small-message lane (descriptor ring +
  // control block in mapped pinned memory, served by lane_kernel), tickets
  struct Lane {
    fsx::LaneCtl* ctl = nullptr;
    fsx::LaneDesc* ring = nullptr;
    cudaStream_t stream = nullptr;
    uint64_t tail = 0;         // descriptors published
    uint64_t epoch = 0;        // epoch of the last launched service kernel (0: none yet)
    int64_t outstanding = 0;   // published, ticket not yet freed
    std::vector<int64_t> slot_ticket;  // ring slot -> ticket whose descriptor it holds (-1: none)
  };
  std::map<int, Lane> lanes;   // by device ordinal
  uint8_t* mail = nullptr;
  BlockList mail_blocks;
  struct Ticket {
    bool used = false;
    int64_t slot = -1;   // mailbox offset of the staged bytes; -1: device source (no staging)
    int device = -1;
    uint64_t seq = 0;    // lane descriptor sequence number
    int64_t n = 0;       // message bytes
    uint8_t* dst = nullptr;  // its slab segment (device)
    // a ticket held across a full turn of the ring (an orphaned or parked
    // message) has its served descriptor copied here before the slot is reused
    bool harvested = false;
    uint64_t sent = 0, landed = 0;
  };
  std::vector<Ticket> tickets;
  std::vector<int64_t> free_tickets;
  std::atomic<uint64_t> next_token{1};
  std::atomic<int64_t> forwards{0}, bytes_forwarded{0}, merges{0}, merged_rows{0}, launches{0},
      dma_forwards{0};
};

namespace {

int find_gpu(fsx_fabric* f, int gpu, int* device) {
  auto it = f->device_of.find(gpu);
  if (it == f->device_of.end())
    return fail(FSX_E_NOT_FOUND, "gpu " + std::to_string(gpu) + " not in topology map");
  if (device) *device = it->second;
  return FSX_OK;
}

Slab* slab_of(fsx_fabric* f, int gpu) {
  auto it = f->slabs.find(gpu);
  return it == f->slabs.end() ? nullptr : it->second.get();
}

// Lazily create per-device state (stream, counter ring, grid sizes).
int device_state(fsx_fabric* f, int ordinal, Device** out) {
  auto it = f->devices.find(ordinal);
  if (it != f->devices.end()) {
    *out = it->second.get();
    return FSX_OK;
  }
  auto d = std::make_unique<Device>();
  d->ordinal = ordinal;
  FSX_CUDA(cudaSetDevice(ordinal));
  FSX_CUDA(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
  FSX_CUDA(cudaMalloc(&d->counters, kCounterRing * sizeof(uint32_t)));
  FSX_CUDA(cudaMemset(d->counters, 0, kCounterRing * sizeof(uint32_t)));
  d->counter_ring.size = kCounterRing;
  FSX_CUDA(cudaDeviceGetAttribute(&d->sms, cudaDevAttrMultiProcessorCount, ordinal));
  {
    // device spin watchdog: flags that never arrive trap instead of hanging
    const char* e = std::getenv("FSX_SPIN_TIMEOUT_S");
    const double secs = e ? std::atof(e) : 30.0;
    FSX_CUDA(fsx::set_spin_timeout((uint64_t)(std::max(secs, 0.001) * 1e9)));
  }
  *out = d.get();
  f->devices.emplace(ordinal, std::move(d));
  return FSX_OK;
}

cudaStream_t pick_stream(Device* d, void* stream) {
  return stream ? static_cast<cudaStream_t>(stream) : d->stream;
}

}  // namespace

extern "C" {

const char* fsx_last_error(void) { return t_err.c_str(); }

const char* fsx_version(void) { return "fsx 0.1 (sm_100a)"; }

int fsx_device_count(int* n) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) c = 0;
  *n = c;
  return FSX_OK;
}

int fsx_abi_sizes(int32_t* merge_batch, int32_t* transfer, int32_t* stats) {
  *merge_batch = (int32_t)sizeof(fsx_merge_batch);
  *transfer = (int32_t)sizeof(fsx_transfer);
  *stats = (int32_t)sizeof(fsx_stats);
  return FSX_OK;
}

int fsx_open(int n_gpus, const int* gpu_ids, const int* node_ids, const int* devices,
             fsx_fabric** out) {
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return fail(FSX_E_CONFIG, "no CUDA device visible: libfsx has no CPU fallback");
  if (n_gpus <= 0) return fail(FSX_E_CONFIG, "empty topology map");
  auto f = std::make_unique<fsx_fabric>();
  for (int i = 0; i < n_gpus; ++i) {
    const int dev = (devices && devices[i] >= 0) ? devices[i] : gpu_ids[i] % count;
    if (dev >= count) return fail(FSX_E_CONFIG, "device ordinal out of range");
    f->node_of[gpu_ids[i]] = node_ids[i];
    f->device_of[gpu_ids[i]] = dev;
  }
  // Peer access between every pair of distinct bound devices (NVLink/NVSwitch).
  std::vector<int> devs;
  for (auto& [g, d] : f->device_of) devs.push_back(d);
  std::sort(devs.begin(), devs.end());
  devs.erase(std::unique(devs.begin(), devs.end()), devs.end());
  for (int a : devs) {
    for (int b : devs) {
      if (a == b) continue;
      int can = 0;
      FSX_CUDA(cudaDeviceCanAccessPeer(&can, a, b));
      if (!can) return fail(FSX_E_CONFIG, "no peer access between devices");
      FSX_CUDA(cudaSetDevice(a));
      cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return fail(FSX_E_CONFIG, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
      cudaGetLastError();
    }
  }
  for (int d : devs) {
    Device* st = nullptr;
    int rc = device_state(f.get(), d, &st);
    if (rc == FSX_OK) {
      // producer kernels loaded now, not at their first launch (fsx_kernels.cuh)
      cudaSetDevice(d);
      const cudaError_t e = fsx::preload_kernels();
      if (e != cudaSuccess) rc = fail(FSX_E_CONFIG, std::string("kernel preload: ") + cudaGetErrorString(e));
    }
    if (rc) {
      const std::string msg = t_err;
      fsx_close(f.release());  // release the streams/counters created so far
      return fail(rc, msg);
    }
  }
  *out = f.release();
  return FSX_OK;
}

int fsx_close(fsx_fabric* f) {
  if (!f) return FSX_OK;
  for (auto& [o, l] : f->lanes) {  // service kernels exit once idle
    reinterpret_cast<volatile uint64_t*>(&l.ctl->stop)[0] = 1;
    cudaSetDevice(o);
    if (l.stream) {
      cudaStreamSynchronize(l.stream);
      cudaStreamDestroy(l.stream);
    }
    cudaFreeHost(l.ctl);
  }
  for (auto& [o, d] : f->devices) {
    cudaSetDevice(o);
    cudaStreamSynchronize(d->stream);
    if (d->notify) cudaStreamSynchronize(d->notify);
  }
  for (auto& [g, s] : f->slabs) {
    cudaSetDevice(s->device);
    if (s->imported) {
      if (s->base) cudaIpcCloseMemHandle(s->base);
    } else {
      if (s->base) cudaFree(s->base);
      if (s->hflags) cudaFreeHost(s->hflags);
    }
  }
  if (f->mail) cudaFreeHost(f->mail);
  for (auto& [p, o] : f->ipc_maps) {
    cudaSetDevice(o);
    cudaIpcCloseMemHandle(p);
  }
  for (auto& [o, d] : f->devices) {
    cudaSetDevice(o);
    if (d->counters) cudaFree(d->counters);
    if (d->state) cudaFree(d->state);
    if (d->scratch) cudaFree(d->scratch);
    for (auto e : d->events) cudaEventDestroy(e);
    for (int k = 0; k < 3; ++k) {
      if (d->stage[k]) cudaFreeHost(d->stage[k]);
      if (d->stage_ev[k]) cudaEventDestroy(d->stage_ev[k]);
    }
    if (d->notify) cudaStreamDestroy(d->notify);
    if (d->stream) cudaStreamDestroy(d->stream);
  }
  delete f;
  return FSX_OK;
}

int fsx_node_of(fsx_fabric* f, int gpu, int* node) {
  auto it = f->node_of.find(gpu);
  if (it == f->node_of.end())
    return fail(FSX_E_NOT_FOUND, "gpu " + std::to_string(gpu) + " not in topology map");
  *node = it->second;
  return FSX_OK;
}

int fsx_route(fsx_fabric* f, int src_gpu, int dst_gpu, int* transport) {
  int a = 0, b = 0;
  int rc = fsx_node_of(f, src_gpu, &a);
  if (rc) return rc;
  rc = fsx_node_of(f, dst_gpu, &b);
  if (rc) return rc;
  *transport = a == b ? FSX_TRANSPORT_LOCAL_BUFFER : FSX_TRANSPORT_NETWORK_STREAM;
  return FSX_OK;
}

int fsx_device_of(fsx_fabric* f, int gpu, int* device) { return find_gpu(f, gpu, device); }

// ---------------------------------------------------------------------------
// Slabs

int fsx_slab_register(fsx_fabric* f, int gpu, int64_t bytes) {
  int dev = 0;
  int rc = find_gpu(f, gpu, &dev);
  if (rc) return rc;
  if (bytes <= 0) return fail(FSX_E_CONFIG, "slab size must be positive");
  std::lock_guard<std::mutex> lk(f->mu);
  if (f->slabs.count(gpu)) return fail(FSX_E_CONFIG, "slab already registered for gpu");
  auto s = std::make_unique<Slab>();
  s->gpu = gpu;
  s->device = dev;
  s->capacity = (bytes + kAlign - 1) & ~(kAlign - 1);
  FSX_CUDA(cudaSetDevice(dev));
  // One allocation: data region followed by the device flag ring, so a single
  // IPC handle exports both.
  cudaError_t e = cudaMalloc(&s->base, s->capacity + kFlagRing * sizeof(uint64_t));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(FSX_E_OOM, std::string("slab cudaMalloc: ") + cudaGetErrorString(e));
  }
  s->dflags = reinterpret_cast<uint64_t*>(s->base + s->capacity);
  FSX_CUDA(cudaMemset(s->dflags, 0, kFlagRing * sizeof(uint64_t)));
  FSX_CUDA(cudaHostAlloc(&s->hflags, kFlagRing * sizeof(uint64_t),
                         cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(s->hflags, 0, kFlagRing * sizeof(uint64_t));
  FSX_CUDA(cudaDeviceSynchronize());
  s->blocks.reset(s->capacity);
  s->flags.size = kFlagRing;
  f->slabs.emplace(gpu, std::move(s));
  return FSX_OK;
}

int fsx_slab_alloc(fsx_fabric* f, int gpu, int64_t len, int64_t* off) {
  std::lock_guard<std::mutex> lk(f->mu);
  Slab* s = slab_of(f, gpu);
  if (!s) return fail(FSX_E_NOT_FOUND, "no slab registered for gpu " + std::to_string(gpu));
  if (s->imported) return fail(FSX_E_CONFIG, "imported slabs are allocated by their owner");
  *off = s->blocks.alloc(len);
  return FSX_OK;
}

int fsx_slab_free(fsx_fabric* f, int gpu, int64_t off) {
  std::lock_guard<std::mutex> lk(f->mu);
  Slab* s = slab_of(f, gpu);
  if (!s) return fail(FSX_E_NOT_FOUND, "no slab registered for gpu " + std::to_string(gpu));
  if (!s->blocks.release(off)) return fail(FSX_E_INTERNAL, "double free in slab");
  return FSX_OK;
}

int fsx_slab_alloc_n(fsx_fabric* f, int gpu, int32_t n, const int64_t* lens, int64_t* offs) {
  std::lock_guard<std::mutex> lk(f->mu);
  Slab* s = slab_of(f, gpu);
  if (!s) return fail(FSX_E_NOT_FOUND, "no slab registered for gpu " + std::to_string(gpu));
  if (s->imported) return fail(FSX_E_CONFIG, "imported slabs are allocated by their owner");
  for (int32_t i = 0; i < n; ++i) {
    offs[i] = s->blocks.alloc(lens[i]);
    if (offs[i] < 0) {
      for (int32_t j = 0; j < i; ++j) s->blocks.release(offs[j]);
      for (int32_t j = 0; j < n; ++j) offs[j] = -1;
      return FSX_OK;
    }
  }
  return FSX_OK;
}

int fsx_slab_free_n(fsx_fabric* f, int gpu, int32_t n, const int64_t* offs) {
  std::lock_guard<std::mutex> lk(f->mu);
  Slab* s = slab_of(f, gpu);
  if (!s) return fail(FSX_E_NOT_FOUND, "no slab registered for gpu " + std::to_string(gpu));
  bool ok = true;
  for (int32_t i = 0; i < n; ++i) ok = s->blocks.release(offs[i]) && ok;
  return ok ? FSX_OK : fail(FSX_E_INTERNAL, "double free in slab");
}

int fsx_slab_ptr(fsx_fabric* f, int gpu, int64_t off, void** d_ptr) {
  std::lock_guard<std::mutex> lk(f->mu);
  Slab* s = slab_of(f, gpu);
  if (!s) return fail(FSX_E_NOT_FOUND, "no slab registered for gpu " + std::to_string(gpu));
  if (off < 0 || off > s->capacity) return fail(FSX_E_VALIDATION, "slab offset out of range");
  *d_ptr = s->base + off;
  return FSX_OK;
}

int fsx_slab_usage(fsx_fabric* f, int gpu, int64_t* segments, int64_t* bytes_in_use,
                   int64_t* peak_bytes, int64_t* capacity) {
  std::lock_guard<std::mutex> lk(f->mu);
  Slab* s = slab_of(f, gpu);
  if (!s) return fail(FSX_E_NOT_FOUND, "no slab registered for gpu " + std::to_string(gpu));
  if (segments) *segments = s->blocks.segments();
  if (bytes_in_use) *bytes_in_use = s->blocks.bytes();
  if (peak_bytes) *peak_bytes = s->blocks.peak();
  if (capacity) *capacity = s->capacity;
  return FSX_OK;
}

int fsx_slab_read(fsx_fabric* f, int gpu, int64_t off, void* h_dst, int64_t n, void* stream) {
  Slab* s = nullptr;
  Device* dev = nullptr;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    s = slab_of(f, gpu);
    if (!s) return fail(FSX_E_NOT_FOUND, "no slab registered for gpu " + std::to_string(gpu));
    if (off < 0 || n < 0 || off + n > s->capacity)
      return fail(FSX_E_VALIDATION, "slab read out of range");
    int rc = device_state(f, s->device, &dev);
    if (rc) return rc;
  }
  if (n == 0) return FSX_OK;
  FSX_CUDA(cudaSetDevice(s->device));
  cudaStream_t st = pick_stream(dev, stream);
  if (n < kStageMin || is_pinned_host(h_dst)) {
    FSX_CUDA(cudaMemcpyAsync(h_dst, s->base + off, n, cudaMemcpyDeviceToHost, st));
    FSX_CUDA(cudaStreamSynchronize(st));
    return FSX_OK;
  }
  // pageable destination (a ChunkCallback's fresh std::vector, sidecar.hpp:
  // 543-561): D2H into the pinned staging ring, three pieces in flight, each
  // landed piece copied out by the copy threads (which also take the
  // destination's first-touch page faults in parallel)
  std::lock_guard<std::mutex> stage_lk(dev->stage_mu);
  for (int k = 0; k < 3; ++k) {
    if (!dev->stage[k]) FSX_CUDA(cudaHostAlloc(&dev->stage[k], kStagePiece, cudaHostAllocDefault));
    if (!dev->stage_ev[k]) FSX_CUDA(cudaEventCreateWithFlags(&dev->stage_ev[k], cudaEventDisableTiming));
    FSX_CUDA(cudaEventSynchronize(dev->stage_ev[k]));  // a host->device staging copy still reading it
  }
  const int64_t pieces = (n + kStagePiece - 1) / kStagePiece;
  auto issue = [&](int64_t i) -> cudaError_t {
    const int64_t beg = i * kStagePiece, len = std::min(kStagePiece, n - beg);
    cudaError_t e = cudaMemcpyAsync(dev->stage[i % 3], s->base + off + beg, len, cudaMemcpyDeviceToHost, st);
    return e != cudaSuccess ? e : cudaEventRecord(dev->stage_ev[i % 3], st);
  };
  for (int64_t i = 0; i < std::min<int64_t>(3, pieces); ++i) FSX_CUDA(issue(i));
  for (int64_t i = 0; i < pieces; ++i) {
    const int64_t beg = i * kStagePiece, len = std::min(kStagePiece, n - beg);
    FSX_CUDA(cudaEventSynchronize(dev->stage_ev[i % 3]));
    par_memcpy(static_cast<uint8_t*>(h_dst) + beg, dev->stage[i % 3], len);
    if (i + 3 < pieces) FSX_CUDA(issue(i + 3));
  }
  return FSX_OK;
}

int fsx_slab_write(fsx_fabric* f, int gpu, int64_t off, const void* h_src, int64_t n, void* stream) {
  Slab* s = nullptr;
  Device* dev = nullptr;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    s = slab_of(f, gpu);
    if (!s) return fail(FSX_E_NOT_FOUND, "no slab registered for gpu " + std::to_string(gpu));
    if (off < 0 || n < 0 || off + n > s->capacity)
      return fail(FSX_E_VALIDATION, "slab write out of range");
    int rc = device_state(f, s->device, &dev);
    if (rc) return rc;
  }
  if (n == 0) return FSX_OK;
  FSX_CUDA(cudaSetDevice(s->device));
  cudaStream_t st = pick_stream(dev, stream);
  FSX_CUDA(cudaMemcpyAsync(s->base + off, h_src, n, cudaMemcpyDefault, st));
  FSX_CUDA(cudaStreamSynchronize(st));
  return FSX_OK;
}

int fsx_ipc_open(fsx_fabric* f, int gpu, const void* handle64, void** d_ptr) {
  int dev = 0;
  int rc = find_gpu(f, gpu, &dev);
  if (rc) return rc;
  *d_ptr = nullptr;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  FSX_CUDA(cudaSetDevice(dev));
  void* p = nullptr;
  FSX_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  std::lock_guard<std::mutex> lk(f->mu);
  f->ipc_maps[p] = dev;
  *d_ptr = p;
  return FSX_OK;
}

int fsx_ipc_close(fsx_fabric* f, void* d_ptr) {
  int dev = -1;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    auto it = f->ipc_maps.find(d_ptr);
    if (it == f->ipc_maps.end()) return fail(FSX_E_NOT_FOUND, "pointer was not opened by fsx_ipc_open");
    dev = it->second;
    f->ipc_maps.erase(it);
  }
  FSX_CUDA(cudaSetDevice(dev));
  FSX_CUDA(cudaIpcCloseMemHandle(d_ptr));
  return FSX_OK;
}

int fsx_slab_export(fsx_fabric* f, int gpu, void* handle64, int64_t* bytes) {
  std::lock_guard<std::mutex> lk(f->mu);
  Slab* s = slab_of(f, gpu);
  if (!s || s->imported) return fail(FSX_E_NOT_FOUND, "no owned slab for gpu");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
  cudaIpcMemHandle_t h;
  FSX_CUDA(cudaSetDevice(s->device));
  FSX_CUDA(cudaIpcGetMemHandle(&h, s->base));
  std::memcpy(handle64, &h, sizeof(h));
  *bytes = s->capacity;
  return FSX_OK;
}

int fsx_slab_import(fsx_fabric* f, int gpu, const void* handle64, int64_t bytes) {
  int dev = 0;
  int rc = find_gpu(f, gpu, &dev);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(f->mu);
  if (f->slabs.count(gpu)) return fail(FSX_E_CONFIG, "slab already registered for gpu");
  auto s = std::make_unique<Slab>();
  s->gpu = gpu;
  s->device = dev;  // device of THIS process the mapping is opened on
  s->imported = true;
  s->capacity = bytes;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  FSX_CUDA(cudaSetDevice(dev));
  void* p = nullptr;
  FSX_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  s->base = static_cast<uint8_t*>(p);
  s->dflags = reinterpret_cast<uint64_t*>(s->base + s->capacity);
  s->flags.size = kFlagRing;
  f->slabs.emplace(gpu, std::move(s));
  return FSX_OK;
}

// ---------------------------------------------------------------------------
// Flags

int fsx_flags_alloc(fsx_fabric* f, int dst_gpu, int32_t n, int64_t* flag_base) {
  std::lock_guard<std::mutex> lk(f->mu);
  Slab* s = slab_of(f, dst_gpu);
  if (!s) return fail(FSX_E_NOT_FOUND, "no slab registered for gpu " + std::to_string(dst_gpu));
  if (n <= 0 || n > kFlagRing / 4) return fail(FSX_E_VALIDATION, "bad flag count");
  *flag_base = s->flags.take(n);
  if (*flag_base < 0) return fail(FSX_E_OOM, "flag ring exhausted by graph-pinned ranges");
  return FSX_OK;
}

int fsx_flag_ptr(fsx_fabric* f, int dst_gpu, int64_t flag_idx, uint64_t** d_flag) {
  std::lock_guard<std::mutex> lk(f->mu);
  Slab* s = slab_of(f, dst_gpu);
  if (!s) return fail(FSX_E_NOT_FOUND, "no slab registered for gpu " + std::to_string(dst_gpu));
  if (flag_idx < 0 || flag_idx >= kFlagRing) return fail(FSX_E_VALIDATION, "flag index out of range");
  *d_flag = s->dflags + flag_idx;
  return FSX_OK;
}

int fsx_forward(fsx_fabric* f, int src_gpu, const void* d_src, int dst_gpu, int64_t dst_off,
                int64_t bytes, int64_t chunk_bytes, int64_t flag_base, uint64_t* token,
                void* stream) {
  return fsx_forward_ex(f, src_gpu, d_src, dst_gpu, dst_off, bytes, chunk_bytes, flag_base, token,
                        FSX_FWD_HOST_NOTIFY, stream);
}

int fsx_forward_ex(fsx_fabric* f, int src_gpu, const void* d_src, int dst_gpu, int64_t dst_off,
                   int64_t bytes, int64_t chunk_bytes, int64_t flag_base, uint64_t* token,
                   uint32_t options, void* stream) {
  fsx_transfer t{src_gpu, dst_gpu, d_src, dst_off, bytes, chunk_bytes, flag_base,
                 token ? *token : 0};
  const int rc = fsx_forward_batch(f, 1, &t, options, stream);
  if (rc == FSX_OK && token) *token = t.token;
  return rc;
}

// The copy-engine form of a forward batch (FSX_FWD_DMA, fsx.h): per chunk one
// cudaMemcpyAsync into the slab, then per transfer one set_flags_kernel (one
// thread per chunk flag, release stores, + the host mirror) behind the copies
// in stream order -- the same flags and tokens K1 publishes, so every consumer
// (fsx_wait, early-start merges, fsx_stream_wait_flags) is unchanged; a
// transfer's chunk flags turn together, after its last chunk.  The
// fsx_forward_host pattern, device to device.  A stream memory operation
// (cuStreamWriteValue64) for the flag measured 5.1 us per transfer against
// 1.7 us for the flag kernel (profiles/k1_floor_dma_r02s.jsonl).  Returns
// kNotDma when the batch is not eligible (a fused digest, FSX_FWD_KERNEL /
// FSX_FWD_BULK, more than FSX_FWD_DMA_MAX_CHUNKS chunks or
// FSX_FWD_DMA_MAX_BYTES bytes, L2_KEEP, or a peer destination, unless
// FSX_FWD_DMA); the caller then launches K1.  Validation is K1's.
constexpr int kNotDma = -1;
int forward_dma(fsx_fabric* f, int src_dev, int32_t n, fsx_transfer* t, uint32_t options,
                cudaStream_t st, bool graph) {
  if (options & (FSX_FWD_KERNEL | FSX_FWD_BULK)) return kNotDma;
  const bool forced = (options & FSX_FWD_DMA) != 0;
  // automatic only in the latency regime, and not when the caller asked for
  // K1's L2 residency hint (a same-GPU merge reads the slab right after)
  if (!forced && (options & FSX_FWD_L2_KEEP)) return kNotDma;
  int64_t batch_bytes = 0;
  for (int32_t i = 0; i < n; ++i) batch_bytes += t[i].bytes;
  if (!forced && batch_bytes > FSX_FWD_DMA_MAX_BYTES) return kNotDma;
  struct Op {
    uint8_t* dst;
    const uint8_t* src;
    int64_t bytes, chunk, n_chunks;
    uint64_t* dflags;
    uint64_t* hflags;
    bool peer;
  };
  std::vector<Op> ops(n);
  int64_t chunks = 0;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    for (int32_t i = 0; i < n; ++i) {
      const fsx_transfer& x = t[i];
      if (x.d_digest) return kNotDma;
      int64_t chunk = x.chunk_bytes;
      if (chunk <= 0 || chunk >= x.bytes) chunk = std::max<int64_t>(x.bytes, 1);
      const int64_t n_chunks = x.bytes == 0 ? 1 : (x.bytes + chunk - 1) / chunk;
      chunks += n_chunks;
      if (!forced && chunks > FSX_FWD_DMA_MAX_CHUNKS) return kNotDma;
      Slab* s = slab_of(f, x.dst_gpu);
      if (!s) return kNotDma;  // K1's path reports it
      if (!forced && (s->imported || s->device != src_dev)) return kNotDma;
      if (x.dst_off < 0 || x.dst_off + x.bytes > s->capacity)
        return fail(FSX_E_VALIDATION, "forward overruns the destination slab");
      if (x.flag_base < 0 || x.flag_base + n_chunks > kFlagRing)
        return fail(FSX_E_VALIDATION, "flag range out of the ring");
      ops[i] = Op{s->base + x.dst_off, static_cast<const uint8_t*>(x.d_src), x.bytes, chunk, n_chunks,
                  s->dflags + x.flag_base,
                  (s->hflags && (options & FSX_FWD_HOST_NOTIFY)) ? s->hflags + x.flag_base : nullptr,
                  s->imported || s->device != src_dev};
    }
    for (int32_t i = 0; i < n; ++i) {
      if (graph) slab_of(f, t[i].dst_gpu)->flags.pin(t[i].flag_base, ops[i].n_chunks);
      if (t[i].token == 0) t[i].token = f->next_token.fetch_add(1);
    }
  }
  for (int32_t i = 0; i < n; ++i) {
    const Op& o = ops[i];
    for (int64_t c = 0; c < o.n_chunks; ++c) {
      const int64_t beg = c * o.chunk, len = std::min(o.chunk, o.bytes - beg);
      if (len > 0) FSX_CUDA(cudaMemcpyAsync(o.dst + beg, o.src + beg, len, cudaMemcpyDefault, st));
    }
    fsx::FlagSetArgs fa{o.dflags, o.hflags, static_cast<int32_t>(o.n_chunks), t[i].token, o.peer ? 0 : 1};
    FSX_CUDA(fsx::launch_set_flags(fa, st));
    f->launches++;
    f->bytes_forwarded += o.bytes;
    f->forwards++;
    f->dma_forwards++;
  }
  return FSX_OK;
}

int fsx_forward_batch(fsx_fabric* f, int32_t n, fsx_transfer* t, uint32_t options, void* stream) {
  NvtxRange nvtx_range("fsx.forward");
  if (n <= 0) return n == 0 ? FSX_OK : fail(FSX_E_VALIDATION, "negative transfer count");
  int src_dev = 0;
  int rc = find_gpu(f, t[0].src_gpu, &src_dev);
  if (rc) return rc;
  for (int32_t i = 0; i < n; ++i) {
    int d = 0;
    rc = find_gpu(f, t[i].src_gpu, &d);
    if (rc) return rc;
    if (d != src_dev) return fail(FSX_E_VALIDATION, "a forward batch must share one source device");
    if (t[i].bytes < 0) return fail(FSX_E_VALIDATION, "negative byte count");
    if (t[i].chunk_bytes > 0 && t[i].chunk_bytes < t[i].bytes && t[i].chunk_bytes % 16)
      return fail(FSX_E_VALIDATION, "chunk_bytes must be a multiple of 16");
  }
  Device* dev = nullptr;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    rc = device_state(f, src_dev, &dev);
    if (rc) return rc;
  }
  // one CTA per tile; a chunk is counted complete tile by tile.  Tiles are
  // 32 KiB, or 4 KiB when the whole batch is at most 2 MiB: a small transfer
  // is latency-bound, and 8x more CTAs with one vector per thread finish it
  // sooner (64 KiB: 2.0 vs 2.5 us, 1 MiB: 2.4 vs 2.7 us; 4 MiB is faster with
  // 32 KiB tiles; profiles/launch_floor_r02c.jsonl)
  int64_t batch_bytes = 0;
  for (int32_t i = 0; i < n; ++i) batch_bytes += t[i].bytes;
  const int64_t unit = batch_bytes <= (int64_t{2} << 20) ? 4096 : fsx::forward_tile_bytes();
  FSX_CUDA(cudaSetDevice(src_dev));
  cudaStream_t st = pick_stream(dev, stream);
  const bool graph = capturing(st);
  rc = forward_dma(f, src_dev, n, t, options, st, graph);
  if (rc != kNotDma) return rc;
  for (int32_t first = 0; first < n; first += fsx::kFwdMaxBatch) {
    const int32_t cnt = std::min<int32_t>(n - first, fsx::kFwdMaxBatch);
    fsx::FwdBatch b{};
    b.n = cnt;
    b.l2_keep_dst = (options & FSX_FWD_L2_KEEP) ? 1 : 0;
    b.peer_gpu_count = (options & FSX_FWD_PEER_GPU_COUNT) ? 1 : 0;
    b.small = unit == 4096 ? 1 : 0;
    for (int32_t k = 0; k < cnt; ++k) {
      fsx_transfer& x = t[first + k];
      fsx::FwdArgs& a = b.t[k];
      int64_t chunk = x.chunk_bytes;
      if (chunk <= 0 || chunk >= x.bytes) chunk = std::max<int64_t>(x.bytes, 1);
      const int64_t n_chunks = x.bytes == 0 ? 1 : (x.bytes + chunk - 1) / chunk;
      {
        std::lock_guard<std::mutex> lk(f->mu);
        Slab* s = slab_of(f, x.dst_gpu);
        if (!s) return fail(FSX_E_NOT_FOUND, "no slab registered for gpu " + std::to_string(x.dst_gpu));
        if (x.dst_off < 0 || x.dst_off + x.bytes > s->capacity)
          return fail(FSX_E_VALIDATION, "forward overruns the destination slab");
        if (x.flag_base < 0 || x.flag_base + n_chunks > kFlagRing)
          return fail(FSX_E_VALIDATION, "flag range out of the ring");
        const int64_t c0 = dev->counter_ring.take(n_chunks);
        if (c0 < 0) return fail(FSX_E_OOM, "chunk counter ring exhausted by graph-pinned ranges");
        if (graph) {  // baked into the graph: never handed out again
          dev->counter_ring.pin(c0, n_chunks);
          s->flags.pin(x.flag_base, n_chunks);
        }
        a.counters = dev->counters + c0;
        a.dst = s->base + x.dst_off;
        a.dflags = s->dflags + x.flag_base;
        a.hflags = (s->hflags && (options & FSX_FWD_HOST_NOTIFY)) ? s->hflags + x.flag_base : nullptr;
        a.peer = (s->imported || s->device != src_dev) ? 1 : 0;
      }
      a.src = static_cast<const uint8_t*>(x.d_src);
      a.bytes = x.bytes;
      a.chunk_bytes = chunk;
      a.slice = std::min<int64_t>(unit, std::max<int64_t>(16, chunk));
      a.slice = (a.slice + 15) & ~int64_t{15};
      a.chunk_units = (chunk + a.slice - 1) / a.slice;
      const int64_t last_len = x.bytes - (n_chunks - 1) * chunk;
      a.last_units = std::max<int64_t>(1, (last_len + a.slice - 1) / a.slice);
      a.total_units = (n_chunks - 1) * a.chunk_units + a.last_units;
      a.n_chunks = (int32_t)n_chunks;
      a.vec = ((reinterpret_cast<uintptr_t>(a.src) | reinterpret_cast<uintptr_t>(a.dst)) & 15) == 0 ? 16 : 0;
      if (x.token == 0) x.token = f->next_token.fetch_add(1);
      a.token = x.token;
      // the fused digest needs the 16-byte path; otherwise digest the source
      // with a separate pass after the copy (below)
      a.digest = a.vec ? x.d_digest : nullptr;
      b.unit_off[k + 1] = b.unit_off[k] + a.total_units;
      f->bytes_forwarded += x.bytes;
      f->forwards++;
    }
    // K1 form: FSX_FWD_BULK / FSX_FWD_KERNEL as asked; otherwise the bulk-copy
    // tiles for a local batch above the small-batch size without the L2 hint
    // (256 MiB alone: 81.5 us bulk vs 90.3 us register tiles, 64 MiB 24.0 vs
    // 26.7, 4 MiB 4.8 vs 6.0 with an L2 flush, profiles/k1_sweep_flush_*_r02s);
    // peer batches keep the register tiles unless asked (the N > 1 probe
    // picks the peer form per run)
    bool any_peer = false;
    for (int32_t k = 0; k < cnt; ++k) any_peer = any_peer || b.t[k].peer;
    const bool bulk = (options & FSX_FWD_BULK) != 0 ||
                      (!(options & (FSX_FWD_KERNEL | FSX_FWD_L2_KEEP)) && !any_peer && !b.small);
    FSX_CUDA(fsx::launch_forward(b, bulk, st));
    f->launches++;
    for (int32_t k = 0; k < cnt; ++k) {
      const fsx_transfer& x = t[first + k];
      if (x.d_digest && !b.t[k].vec) {
        FSX_CUDA(fsx::launch_digest(static_cast<const uint8_t*>(x.d_src), x.bytes, x.d_digest,
                                    digest_grid(dev, x.bytes), st));
        f->launches++;
      }
    }
  }
  return FSX_OK;
}

int fsx_digest(fsx_fabric* f, int gpu, const void* d_ptr, int64_t n, uint64_t* d_accum,
               void* stream) {
  int ordinal = 0;
  int rc = find_gpu(f, gpu, &ordinal);
  if (rc) return rc;
  if (n < 0 || !d_accum) return fail(FSX_E_VALIDATION, "bad digest range");
  Device* dev = nullptr;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    rc = device_state(f, ordinal, &dev);
    if (rc) return rc;
  }
  FSX_CUDA(cudaSetDevice(ordinal));
  FSX_CUDA(fsx::launch_digest(static_cast<const uint8_t*>(d_ptr), n, d_accum, digest_grid(dev, n),
                              pick_stream(dev, stream)));
  f->launches++;
  return FSX_OK;
}

int fsx_u64_slot(fsx_fabric* f, int gpu, uint64_t** d_slot, void* stream) {
  int ordinal = 0;
  int rc = find_gpu(f, gpu, &ordinal);
  if (rc) return rc;
  Device* dev = nullptr;
  uint64_t* slot = nullptr;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    rc = device_state(f, ordinal, &dev);
    if (rc) return rc;
    if (!dev->scratch) {
      FSX_CUDA(cudaSetDevice(ordinal));
      FSX_CUDA(cudaMalloc(&dev->scratch, kScratchRing * sizeof(uint64_t)));
      dev->scratch_ring.size = kScratchRing;
    }
    const int64_t at = dev->scratch_ring.take(1);
    if (at < 0) return fail(FSX_E_OOM, "scratch ring exhausted by graph-pinned slots");
    if (capturing(pick_stream(dev, stream))) dev->scratch_ring.pin(at, 1);
    slot = dev->scratch + at;
  }
  FSX_CUDA(cudaSetDevice(ordinal));
  FSX_CUDA(cudaMemsetAsync(slot, 0, sizeof(uint64_t), pick_stream(dev, stream)));
  *d_slot = slot;
  return FSX_OK;
}

int fsx_read_u64(fsx_fabric* f, int gpu, const uint64_t* d, uint64_t* h, void* stream) {
  int ordinal = 0;
  int rc = find_gpu(f, gpu, &ordinal);
  if (rc) return rc;
  Device* dev = nullptr;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    rc = device_state(f, ordinal, &dev);
    if (rc) return rc;
  }
  FSX_CUDA(cudaSetDevice(ordinal));
  cudaStream_t st = pick_stream(dev, stream);
  FSX_CUDA(cudaMemcpyAsync(h, d, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  FSX_CUDA(cudaStreamSynchronize(st));
  return FSX_OK;
}

int fsx_forward_host(fsx_fabric* f, const void* h_src, int dst_gpu, int64_t dst_off,
                     int64_t bytes, int64_t chunk_bytes, int64_t flag_base, uint64_t* token,
                     void* stream) {
  return fsx_forward_host_digest(f, h_src, dst_gpu, dst_off, bytes, chunk_bytes, flag_base, token, stream,
                                 nullptr);
}

int fsx_forward_host_digest(fsx_fabric* f, const void* h_src, int dst_gpu, int64_t dst_off,
                            int64_t bytes, int64_t chunk_bytes, int64_t flag_base, uint64_t* token,
                            void* stream, uint64_t* digest) {
  NvtxRange nvtx_range("fsx.forward_host");
  if (bytes < 0) return fail(FSX_E_VALIDATION, "negative byte count");
  if (chunk_bytes <= 0 || chunk_bytes >= bytes) chunk_bytes = std::max<int64_t>(bytes, 1);
  else if (chunk_bytes % 16) return fail(FSX_E_VALIDATION, "chunk_bytes must be a multiple of 16");
  const int64_t n_chunks = bytes == 0 ? 1 : (bytes + chunk_bytes - 1) / chunk_bytes;
  Slab* s = nullptr;
  Device* dev = nullptr;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    s = slab_of(f, dst_gpu);
    if (!s) return fail(FSX_E_NOT_FOUND, "no slab registered for gpu " + std::to_string(dst_gpu));
    if (dst_off < 0 || dst_off + bytes > s->capacity)
      return fail(FSX_E_VALIDATION, "forward overruns the destination slab");
    if (flag_base < 0 || flag_base + n_chunks > kFlagRing)
      return fail(FSX_E_VALIDATION, "flag range out of the ring");
    int rc = device_state(f, s->device, &dev);
    if (rc) return rc;
  }
  const uint64_t tok = (token && *token) ? *token : f->next_token.fetch_add(1);
  cudaStream_t st = pick_stream(dev, stream);
  FSX_CUDA(cudaSetDevice(s->device));
  // The copies stay back to back on `st` (the copy engine never idles); each
  // chunk's flag store runs on the device's notify stream once an event
  // recorded after that chunk's copy has fired.
  if (!dev->notify) {
    FSX_CUDA(cudaStreamCreateWithFlags(&dev->notify, cudaStreamNonBlocking));
    dev->events.resize(kEventRing);
    for (auto& e : dev->events) FSX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // pageable source: staged through the pinned ring (the driver's own staging
  // of a pageable cudaMemcpyAsync moves ~9 GB/s here); returns once every
  // source byte is copied out, like a pageable cudaMemcpyAsync
  const bool staged = bytes >= kStageMin && !is_pinned_host(h_src);
  std::unique_lock<std::mutex> stage_lk(dev->stage_mu, std::defer_lock);
  if (staged) {
    stage_lk.lock();
    for (int k = 0; k < 3; ++k) {
      if (!dev->stage[k]) FSX_CUDA(cudaHostAlloc(&dev->stage[k], kStagePiece, cudaHostAllocDefault));
      if (!dev->stage_ev[k]) FSX_CUDA(cudaEventCreateWithFlags(&dev->stage_ev[k], cudaEventDisableTiming));
    }
  }
  uint64_t dg = 0;  // dg64 word terms of the source (digest != nullptr)
  for (int64_t c = 0; c < n_chunks; ++c) {
    const int64_t beg = c * chunk_bytes, len = std::min(chunk_bytes, bytes - beg);
    if (len > 0 && staged) {
      for (int64_t p = beg; p < beg + len; p += kStagePiece) {
        const int64_t pl = std::min(kStagePiece, beg + len - p);
        const int k = (int)(dev->stage_next++ % 3);
        FSX_CUDA(cudaEventSynchronize(dev->stage_ev[k]));  // its previous copy has run
        if (digest)
          dg += par_copy_digest(dev->stage[k], static_cast<const uint8_t*>(h_src) + p, pl, (uint64_t)p / 8);
        else
          par_memcpy(dev->stage[k], static_cast<const uint8_t*>(h_src) + p, pl);
        FSX_CUDA(cudaMemcpyAsync(s->base + dst_off + p, dev->stage[k], pl, cudaMemcpyHostToDevice, st));
        FSX_CUDA(cudaEventRecord(dev->stage_ev[k], st));
      }
    } else if (len > 0) {
      FSX_CUDA(cudaMemcpyAsync(s->base + dst_off + beg, static_cast<const uint8_t*>(h_src) + beg,
                               len, cudaMemcpyHostToDevice, st));
    }
    cudaEvent_t ev = dev->events[dev->next_event++ % kEventRing];
    FSX_CUDA(cudaEventRecord(ev, st));
    FSX_CUDA(cudaStreamWaitEvent(dev->notify, ev, 0));
    fsx::FlagSetArgs fa{s->dflags + flag_base + c, s->hflags ? s->hflags + flag_base + c : nullptr,
                        1, tok};
    FSX_CUDA(fsx::launch_set_flags(fa, dev->notify));
    f->launches++;
  }
  // unstaged (pinned / small) source: digested while the DMA reads it
  if (digest && !staged) dg = par_copy_digest(nullptr, static_cast<const uint8_t*>(h_src), bytes, 0);
  if (digest) *digest = (uint64_t)bytes * 0x9e3779b97f4a7c15ull + dg;
  f->forwards++;
  f->bytes_forwarded += bytes;
  if (token) *token = tok;
  return FSX_OK;
}

constexpr int64_t kMailBytes = int64_t{16} << 20;

namespace {

// The lane of `device`, created on first use (caller holds f->mu).
int lane_of(fsx_fabric* f, int device, fsx_fabric::Lane** out) {
  auto it = f->lanes.find(device);
  if (it != f->lanes.end()) {
    *out = &it->second;
    return FSX_OK;
  }
  fsx_fabric::Lane l;
  FSX_CUDA(cudaSetDevice(device));
  void* mem = nullptr;
  const size_t bytes = sizeof(fsx::LaneCtl) + sizeof(fsx::LaneDesc) * fsx::kLaneSlots;
  FSX_CUDA(cudaHostAlloc(&mem, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(mem, 0, bytes);
  l.ctl = static_cast<fsx::LaneCtl*>(mem);
  l.ring = reinterpret_cast<fsx::LaneDesc*>(static_cast<uint8_t*>(mem) + sizeof(fsx::LaneCtl));
  FSX_CUDA(cudaStreamCreateWithFlags(&l.stream, cudaStreamNonBlocking));
  l.slot_ticket.assign(fsx::kLaneSlots, -1);
  *out = &f->lanes.emplace(device, std::move(l)).first->second;
  return FSX_OK;
}

inline uint64_t vload(const uint64_t* p) { return *reinterpret_cast<const volatile uint64_t*>(p); }
inline void vstore(uint64_t* p, uint64_t v) { *reinterpret_cast<volatile uint64_t*>(p) = v; }

// Release a waited ticket's mailbox slot and ring-slot claim (holds f->mu).
void ticket_release(fsx_fabric* f, int64_t ticket) {
  fsx_fabric::Ticket& t = f->tickets[ticket];
  if (t.slot >= 0) f->mail_blocks.release(t.slot);
  fsx_fabric::Lane& l = f->lanes.at(t.device);
  --l.outstanding;
  int64_t& claim = l.slot_ticket[t.seq % fsx::kLaneSlots];
  if (claim == ticket) claim = -1;
  t = fsx_fabric::Ticket{};
  f->free_tickets.push_back(ticket);
}

// A served message: its mailbox slot (-1: device source), bytes, slab
// segment and both device digests.
struct Served {
  int64_t slot = -1, n = 0;
  uint8_t* dst = nullptr;
  uint64_t sent = 0, landed = 0;
};

// Wait until the ticket's message has been served (caller does not hold
// f->mu).  Spins on the descriptor's done mark (host memory the kernel
// writes over PCIe); FSX_E_TIMEOUT after FSX_SPIN_TIMEOUT_S (default 30 s).
// The digests come from the descriptor, or from the ticket if a publisher
// harvested them before reusing the slot (checked again after the read, so a
// slot reused between the done mark and the read is never trusted).
int lane_wait(fsx_fabric* f, int64_t ticket, Served* out, bool release = false) {
  const fsx::LaneDesc* d = nullptr;
  uint64_t seq = 0;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    if (ticket < 0 || ticket >= (int64_t)f->tickets.size() || !f->tickets[ticket].used)
      return fail(FSX_E_NOT_FOUND, "unknown small-message ticket");
    const fsx_fabric::Ticket& t = f->tickets[ticket];
    *out = Served{t.slot, t.n, t.dst, t.sent, t.landed};
    if (t.harvested) {
      if (release) ticket_release(f, ticket);
      return FSX_OK;
    }
    d = &f->lanes.at(t.device).ring[t.seq % fsx::kLaneSlots];
    seq = t.seq;
  }
  if (vload(&d->done) != seq + 1) {
    const char* e = std::getenv("FSX_SPIN_TIMEOUT_S");
    const double secs = e ? std::atof(e) : 30.0;
    const auto t0 = std::chrono::steady_clock::now();
    uint32_t n = 0;
    while (vload(&d->done) != seq + 1) {
      if ((++n & 4095u) == 0) {
        {
          std::lock_guard<std::mutex> lk(f->mu);
          const fsx_fabric::Ticket& t = f->tickets[ticket];
          if (t.harvested) {
            out->sent = t.sent;
            out->landed = t.landed;
            if (release) ticket_release(f, ticket);
            return FSX_OK;
          }
        }
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > secs)
          return fail(FSX_E_TIMEOUT, "small-message lane: message not served within the watchdog time");
        std::this_thread::yield();
      }
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  out->sent = vload(&d->sent);
  out->landed = vload(&d->landed);
  std::lock_guard<std::mutex> lk(f->mu);
  const fsx_fabric::Ticket& t = f->tickets[ticket];
  if (t.harvested) {  // the slot was reused after the done mark was read
    out->sent = t.sent;
    out->landed = t.landed;
  }
  if (release) ticket_release(f, ticket);
  return FSX_OK;
}

}  // namespace

namespace {

// Publish one message on the destination device's lane: host bytes are
// staged in a mailbox slot; a device source (this GPU's memory or a peer's,
// peer access is enabled at fsx_open) is read by the lane kernel in place.
int put_small_locked(fsx_fabric* f, int dst_gpu, int64_t dst_off, const void* src, int64_t n, bool device,
                     int64_t* ticket) {  // caller holds f->mu
  *ticket = -1;
  if (n <= 0 || n > FSX_SMALL_MAX) return FSX_OK;
  Slab* s = slab_of(f, dst_gpu);
  if (!s) return fail(FSX_E_NOT_FOUND, "no slab registered for gpu " + std::to_string(dst_gpu));
  if (dst_off < 0 || dst_off + n > s->capacity)
    return fail(FSX_E_VALIDATION, "small put overruns the destination slab");
  if (!device && !f->mail) {
    FSX_CUDA(cudaHostAlloc(&f->mail, kMailBytes, cudaHostAllocMapped | cudaHostAllocPortable));
    f->mail_blocks.reset(kMailBytes);
  }
  fsx_fabric::Lane* l = nullptr;
  int rc = lane_of(f, s->device, &l);
  if (rc) return rc;
  int64_t slot = -1;
  if (!device) {
    slot = f->mail_blocks.alloc((n + 63) / 64 * 64);
    if (slot < 0) return FSX_OK;  // mailbox full: caller takes the synchronous path
  }
  int64_t id;
  if (f->free_tickets.empty()) {
    f->tickets.emplace_back();
    id = (int64_t)f->tickets.size() - 1;
  } else {
    id = f->free_tickets.back();
    f->free_tickets.pop_back();
  }
  const uint64_t seq = l->tail;
  fsx::LaneDesc* d = &l->ring[seq % fsx::kLaneSlots];
  int64_t& claim = l->slot_ticket[seq % fsx::kLaneSlots];
  if (claim >= 0) {
    // the ticket published one turn of the ring ago is still held (parked /
    // orphaned message): its message was served long since (the lane is
    // FIFO); keep its digests with the ticket before the slot is rewritten
    fsx_fabric::Ticket& old = f->tickets[claim];
    if (old.used && !old.harvested && old.seq % fsx::kLaneSlots == seq % fsx::kLaneSlots) {
      const auto t0 = std::chrono::steady_clock::now();
      while (vload(&d->done) != old.seq + 1) {
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > 30.0)
          return fail(FSX_E_TIMEOUT, "small-message lane: a ring slot was never served");
        std::this_thread::yield();
      }
      std::atomic_thread_fence(std::memory_order_acquire);
      old.sent = vload(&d->sent);
      old.landed = vload(&d->landed);
      old.harvested = true;
    }
  }
  fsx_fabric::Ticket& tk = f->tickets[id];
  tk = fsx_fabric::Ticket{true, slot, s->device, seq, n, s->base + dst_off};
  claim = id;
  // the descriptor lines were last written by the device (a PCIe write drops
  // them from the host caches): fetch this one and the next for writing while
  // the bytes are copied
  __builtin_prefetch(d, 1);
  __builtin_prefetch(&l->ring[(seq + 1) % fsx::kLaneSlots], 1);
  if (!device) std::memcpy(f->mail + slot, src, (size_t)n);
  d->dst = s->base + dst_off;
  d->src = device ? static_cast<const uint8_t*>(src) : f->mail + slot;
  d->n = n;
  vstore(&d->done, 0);
  // the publication mark last: the lane's poller reads fields and mark in one
  // round trip and trusts the fields only when the mark matches them
  std::atomic_thread_fence(std::memory_order_release);
  vstore(&d->pub, fsx::lane_pub(reinterpret_cast<uint64_t>(d->dst), reinterpret_cast<uint64_t>(d->src),
                                (uint64_t)n, seq));
  // descriptor and bytes before the tail (x86 keeps stores in order; this
  // orders the compiler), then the exit handshake of lane_kernel: store tail,
  // full fence, load exit_epoch
  std::atomic_thread_fence(std::memory_order_release);
  vstore(&l->ctl->tail, seq + 1);
  l->tail = seq + 1;
  ++l->outstanding;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  if (l->epoch == 0 || vload(&l->ctl->exit_epoch) == l->epoch) {
    FSX_CUDA(cudaSetDevice(s->device));
    FSX_CUDA(fsx::launch_lane(l->ctl, l->ring, l->epoch + 1, l->stream));
    ++l->epoch;
    f->launches++;
  }
  f->forwards++;
  f->bytes_forwarded += n;
  *ticket = id;
  return FSX_OK;
}

int put_small_impl(fsx_fabric* f, int dst_gpu, int64_t dst_off, const void* src, int64_t n, bool device,
                   int64_t* ticket) {
  std::lock_guard<std::mutex> lk(f->mu);
  return put_small_locked(f, dst_gpu, dst_off, src, n, device, ticket);
}

}  // namespace

int fsx_put_small(fsx_fabric* f, int dst_gpu, int64_t dst_off, const void* h_src, int64_t n,
                  int64_t* ticket) {
  return put_small_impl(f, dst_gpu, dst_off, h_src, n, false, ticket);
}

int fsx_put_small_alloc(fsx_fabric* f, int dst_gpu, const void* src, int64_t n, int src_is_device,
                        int64_t* dst_off, int64_t* ticket) {
  *dst_off = -1;
  *ticket = -1;
  std::lock_guard<std::mutex> lk(f->mu);
  Slab* s = slab_of(f, dst_gpu);
  if (!s) return fail(FSX_E_NOT_FOUND, "no slab registered for gpu " + std::to_string(dst_gpu));
  if (s->imported) return fail(FSX_E_CONFIG, "imported slabs are allocated by their owner");
  *dst_off = s->blocks.alloc(std::max<int64_t>(n, 1));
  if (*dst_off < 0) return FSX_OK;  // slab full: the caller parks the send (backlog)
  return put_small_locked(f, dst_gpu, *dst_off, src, n, src_is_device != 0, ticket);
}

int fsx_put_small_device(fsx_fabric* f, int dst_gpu, int64_t dst_off, const void* d_src, int64_t n,
                         int64_t* ticket) {
  return put_small_impl(f, dst_gpu, dst_off, d_src, n, true, ticket);
}

int fsx_flush_small(fsx_fabric* f) {
  (void)f;  // messages are served as they are published (small-message lane)
  return FSX_OK;
}

int fsx_ticket_wait(fsx_fabric* f, int64_t ticket, const void** h_bytes, uint64_t* digest) {
  Served sv;
  int rc = lane_wait(f, ticket, &sv);
  if (rc) return rc;
  if (h_bytes) *h_bytes = sv.slot >= 0 ? f->mail + sv.slot : nullptr;  // device source: no host copy
  if (digest) *digest = sv.landed;
  return FSX_OK;
}

int fsx_ticket_digests(fsx_fabric* f, int64_t ticket, uint64_t* sent, uint64_t* landed) {
  Served sv;
  int rc = lane_wait(f, ticket, &sv);
  if (rc) return rc;
  if (sent) *sent = sv.sent;
  if (landed) *landed = sv.landed;
  return FSX_OK;
}

int fsx_ticket_take(fsx_fabric* f, int64_t ticket, void* h_dst, int64_t n, uint64_t* sent,
                    uint64_t* landed) {
  Served sv;
  int rc = lane_wait(f, ticket, &sv);
  if (rc) return rc;
  if (n < 0 || n > sv.n) return fail(FSX_E_VALIDATION, "ticket take longer than the message");
  if (h_dst && n > 0) {
    if (sv.slot >= 0)
      std::memcpy(h_dst, f->mail + sv.slot, (size_t)n);
    else  // device source: the landed segment
      FSX_CUDA(cudaMemcpy(h_dst, sv.dst, (size_t)n, cudaMemcpyDeviceToHost));
  }
  if (sent) *sent = sv.sent;
  if (landed) *landed = sv.landed;
  std::lock_guard<std::mutex> lk(f->mu);
  ticket_release(f, ticket);
  return FSX_OK;
}

int fsx_ticket_free(fsx_fabric* f, int64_t ticket) {
  // the slot and the slab segment may only be reused once the message is served
  Served sv;
  return lane_wait(f, ticket, &sv, /*release=*/true);
}

int fsx_chunk_ready(fsx_fabric* f, int dst_gpu, int64_t flag_idx, uint64_t token, int* ready) {
  Slab* s = nullptr;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    s = slab_of(f, dst_gpu);
  }
  if (!s) return fail(FSX_E_NOT_FOUND, "no slab registered for gpu " + std::to_string(dst_gpu));
  if (!s->hflags) return fail(FSX_E_CONFIG, "host flags are only mapped in the slab owner");
  if (flag_idx < 0 || flag_idx >= kFlagRing) return fail(FSX_E_VALIDATION, "flag index out of range");
  const uint64_t v = __atomic_load_n(&s->hflags[flag_idx], __ATOMIC_ACQUIRE);
  *ready = v == token;
  return FSX_OK;
}

int fsx_wait(fsx_fabric* f, int dst_gpu, int64_t flag_base, int32_t n, uint64_t token,
             int64_t timeout_us) {
  Slab* s = nullptr;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    s = slab_of(f, dst_gpu);
  }
  if (!s) return fail(FSX_E_NOT_FOUND, "no slab registered for gpu " + std::to_string(dst_gpu));
  if (!s->hflags) return fail(FSX_E_CONFIG, "host flags are only mapped in the slab owner");
  if (flag_base < 0 || n < 0 || flag_base + n > kFlagRing)
    return fail(FSX_E_VALIDATION, "flag range out of the ring");
  const auto t0 = std::chrono::steady_clock::now();
  for (int32_t i = 0; i < n; ++i) {
    int spins = 0;
    while (__atomic_load_n(&s->hflags[flag_base + i], __ATOMIC_ACQUIRE) != token) {
      if (++spins > 1024) {
        std::this_thread::yield();
        if (timeout_us >= 0 &&
            std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(timeout_us))
          return fail(FSX_E_TIMEOUT, "chunk flags not set before the timeout");
      }
    }
  }
  return FSX_OK;
}

int fsx_stream_wait_flags(fsx_fabric* f, int dst_gpu, int64_t flag_base, int32_t n,
                          uint64_t token, void* stream) {
  Slab* s = nullptr;
  Device* dev = nullptr;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    s = slab_of(f, dst_gpu);
    if (!s) return fail(FSX_E_NOT_FOUND, "no slab registered for gpu " + std::to_string(dst_gpu));
    int rc = device_state(f, s->device, &dev);
    if (rc) return rc;
  }
  if (flag_base < 0 || n < 0 || flag_base + n > kFlagRing)
    return fail(FSX_E_VALIDATION, "flag range out of the ring");
  FSX_CUDA(cudaSetDevice(s->device));
  FSX_CUDA(fsx::launch_wait_flags(s->dflags + flag_base, n, token, pick_stream(dev, stream)));
  f->launches++;
  return FSX_OK;
}

int fsx_signal_flags(fsx_fabric* f, int dst_gpu, int64_t flag_base, int32_t n, uint64_t token,
                     int src_gpu, void* stream) {
  int src_dev = 0;
  int rc = find_gpu(f, src_gpu, &src_dev);
  if (rc) return rc;
  fsx::FlagSetArgs fa{};
  Device* dev = nullptr;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    Slab* s = slab_of(f, dst_gpu);
    if (!s) return fail(FSX_E_NOT_FOUND, "no slab registered for gpu " + std::to_string(dst_gpu));
    if (flag_base < 0 || n <= 0 || flag_base + n > kFlagRing)
      return fail(FSX_E_VALIDATION, "flag range out of the ring");
    rc = device_state(f, src_dev, &dev);
    if (rc) return rc;
    fa = fsx::FlagSetArgs{s->dflags + flag_base, s->hflags ? s->hflags + flag_base : nullptr, n,
                          token};
  }
  FSX_CUDA(cudaSetDevice(src_dev));
  FSX_CUDA(fsx::launch_set_flags(fa, pick_stream(dev, stream)));
  f->launches++;
  return FSX_OK;
}

// ---------------------------------------------------------------------------
// Merge / synth / stats

int fsx_merge(fsx_fabric* f, int gpu, const fsx_merge_batch* b, void* stream) {
  NvtxRange nvtx_range("fsx.merge");
  int ordinal = 0;
  int rc = find_gpu(f, gpu, &ordinal);
  if (rc) return rc;
  if (!b || b->num_requests < 0 || b->num_items < 0 || b->row_bytes <= 0)
    return fail(FSX_E_VALIDATION, "bad merge batch");
  if (b->num_requests > 0 &&
      (!b->d_embeds || !b->d_token_ids || !b->d_req_row_off || !b->d_req_item_off ||
       !b->d_item_row_off || !b->d_status || (b->total_item_rows > 0 && (!b->d_item_src || !b->d_scratch))))
    return fail(FSX_E_VALIDATION, "merge batch is missing a device array");
  if (b->d_item_flag && (!b->d_item_token || !b->d_item_chunk_rows))
    return fail(FSX_E_VALIDATION, "early-start merge needs tokens and chunk rows");
  if (b->total_rows > INT32_MAX)  // d_scratch holds int32 prompt row indices
    return fail(FSX_E_VALIDATION, "merge batch has more than 2^31 - 1 prompt rows");
  const int base_mode = b->mode & FSX_MERGE_MODE_MASK;
  if (base_mode > FSX_MERGE_COPY_ONLY ||
      (b->mode & ~(FSX_MERGE_MODE_MASK | FSX_MERGE_DISCARD | FSX_MERGE_COLOCATED)))
    return fail(FSX_E_VALIDATION, "unknown merge mode");
  if ((b->mode & FSX_MERGE_COLOCATED) && !b->d_item_flag)
    return fail(FSX_E_VALIDATION, "FSX_MERGE_COLOCATED is an early-start option (item flags)");
  Device* dev = nullptr;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    rc = device_state(f, ordinal, &dev);
    if (rc) return rc;
  }
  FSX_CUDA(cudaSetDevice(ordinal));
  int launched = 0;
  cudaError_t e = fsx::launch_merge(*b, pick_stream(dev, stream), &launched);
  f->launches += launched;
  if (e != cudaSuccess) return fail(FSX_E_INTERNAL, std::string("merge launch: ") + cudaGetErrorString(e));
  if (base_mode != FSX_MERGE_SCAN_ONLY) {
    f->merges++;
    f->merged_rows += b->total_item_rows;
  }
  return FSX_OK;
}

int fsx_forward_place(fsx_fabric* f, int src_gpu, int dst_gpu, const fsx_merge_batch* b,
                      int64_t done_flag, uint64_t token, void* stream) {
  NvtxRange nvtx_range("fsx.forward_place");
  int src_dev = 0, dst_dev = 0;
  int rc = find_gpu(f, src_gpu, &src_dev);
  if (rc) return rc;
  rc = find_gpu(f, dst_gpu, &dst_dev);
  if (rc) return rc;
  if (!b) return fail(FSX_E_VALIDATION, "bad merge batch");
  const int base_mode = b->mode & FSX_MERGE_MODE_MASK;
  if (base_mode == FSX_MERGE_SCAN_ONLY || (b->mode & ~FSX_MERGE_MODE_MASK) || b->d_item_flag)
    return fail(FSX_E_VALIDATION,
                "forward_place takes FSX_MERGE_FULL or FSX_MERGE_COPY_ONLY, no early-start or discard bits");
  // the kernel runs on the producer's device; every consumer array must be
  // addressable from it (same device, or peer access enabled by fsx_open)
  rc = fsx_merge(f, src_gpu, b, stream);
  if (rc) return rc;
  f->forwards++;
  f->bytes_forwarded += b->total_item_rows * b->row_bytes;
  if (done_flag >= 0) return fsx_signal_flags(f, dst_gpu, done_flag, 1, token, src_gpu, stream);
  return FSX_OK;
}

int fsx_forward_merge(fsx_fabric* f, int32_t n, fsx_transfer* t, const fsx_merge_batch* b,
                      uint32_t options, void* stream) {
  NvtxRange nvtx_range("fsx.forward_merge");
  if (!b || n < 0 || n != b->num_items) return fail(FSX_E_VALIDATION, "forward_merge: one transfer per item");
  const int base_mode = b->mode & FSX_MERGE_MODE_MASK;
  if (base_mode == FSX_MERGE_SCAN_ONLY || (b->mode & ~FSX_MERGE_MODE_MASK) || b->d_item_flag)
    return fail(FSX_E_VALIDATION,
                "forward_merge takes FSX_MERGE_FULL or FSX_MERGE_COPY_ONLY, no early-start or discard bits");
  if (b->row_bytes <= 0) return fail(FSX_E_VALIDATION, "bad row_bytes");
  if (b->total_rows > INT32_MAX)  // d_scratch holds int32 prompt row indices
    return fail(FSX_E_VALIDATION, "merge batch has more than 2^31 - 1 prompt rows");
  if (n == 0) return fsx_merge(f, 0, b, stream);  // nothing to forward: statuses only
  int src_dev = 0;
  int rc = find_gpu(f, t[0].src_gpu, &src_dev);
  if (rc) return rc;
  int64_t rows_total = 0;
  for (int32_t i = 0; i < n; ++i) {
    int d = 0;
    rc = find_gpu(f, t[i].src_gpu, &d);
    if (rc) return rc;
    if (d != src_dev) return fail(FSX_E_VALIDATION, "a forward batch must share one source device");
    if (t[i].bytes < 0 || t[i].bytes % b->row_bytes)
      return fail(FSX_E_VALIDATION, "forward_merge: item bytes must be whole rows");
    if (t[i].chunk_bytes > 0 && t[i].chunk_bytes < t[i].bytes && t[i].chunk_bytes % b->row_bytes)
      return fail(FSX_E_VALIDATION, "forward_merge: chunk_bytes must be whole rows");
    if (t[i].d_digest) return fail(FSX_E_VALIDATION, "forward_merge has no fused digest");
    rows_total += t[i].bytes / b->row_bytes;
  }
  if (rows_total != b->total_item_rows)
    return fail(FSX_E_VALIDATION, "forward_merge: transfers do not cover the batch's item rows");
  Device* dev = nullptr;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    rc = device_state(f, src_dev, &dev);
    if (rc) return rc;
  }
  FSX_CUDA(cudaSetDevice(src_dev));
  cudaStream_t st = pick_stream(dev, stream);
  if (base_mode == FSX_MERGE_FULL) {  // positions and statuses first, in stream order
    fsx_merge_batch scan = *b;
    scan.mode = FSX_MERGE_SCAN_ONLY;
    int launched = 0;
    const cudaError_t e = fsx::launch_merge(scan, st, &launched);
    if (e != cudaSuccess) return fail(FSX_E_INTERNAL, std::string("merge scan launch: ") + cudaGetErrorString(e));
    f->launches += launched;
  }
  const bool graph = capturing(st);
  int64_t g = 0;
  for (int32_t first = 0; first < n; first += fsx::kTeeMaxItems) {
    const int32_t cnt = std::min<int32_t>(n - first, fsx::kTeeMaxItems);
    fsx::TeeBatch tb{};
    tb.i0 = first;
    tb.n = cnt;
    tb.g0 = g;
    tb.peer_gpu_count = (options & FSX_FWD_PEER_GPU_COUNT) ? 1 : 0;
    tb.l2_keep_dst = (options & FSX_FWD_L2_KEEP) ? 1 : 0;
    for (int32_t k = 0; k < cnt; ++k) {
      fsx_transfer& x = t[first + k];
      fsx::TeeItem& a = tb.t[k];
      a.rows = x.bytes / b->row_bytes;
      a.chunk_rows = (x.chunk_bytes <= 0 || x.chunk_bytes >= x.bytes) ? std::max<int64_t>(a.rows, 1)
                                                                       : x.chunk_bytes / b->row_bytes;
      const int64_t n_chunks = a.rows == 0 ? 1 : (a.rows + a.chunk_rows - 1) / a.chunk_rows;
      a.n_chunks = (int32_t)n_chunks;
      std::lock_guard<std::mutex> lk(f->mu);
      Slab* s = slab_of(f, x.dst_gpu);
      if (!s) return fail(FSX_E_NOT_FOUND, "no slab registered for gpu " + std::to_string(x.dst_gpu));
      if (x.dst_off < 0 || x.dst_off + x.bytes > s->capacity)
        return fail(FSX_E_VALIDATION, "forward overruns the destination slab");
      if (x.flag_base < 0 || x.flag_base + n_chunks > kFlagRing)
        return fail(FSX_E_VALIDATION, "flag range out of the ring");
      const int64_t c0 = dev->counter_ring.take(n_chunks);
      if (c0 < 0) return fail(FSX_E_OOM, "chunk counter ring exhausted by graph-pinned ranges");
      if (graph) {
        dev->counter_ring.pin(c0, n_chunks);
        s->flags.pin(x.flag_base, n_chunks);
      }
      a.counters = dev->counters + c0;
      a.dst = s->base + x.dst_off;
      a.dflags = s->dflags + x.flag_base;
      a.hflags = (s->hflags && (options & FSX_FWD_HOST_NOTIFY)) ? s->hflags + x.flag_base : nullptr;
      a.peer = (s->imported || s->device != src_dev) ? 1 : 0;
      if (x.token == 0) x.token = f->next_token.fetch_add(1);
      a.token = x.token;
      g += a.rows;
      f->bytes_forwarded += x.bytes;
      f->forwards++;
    }
    tb.g1 = g;
    FSX_CUDA(fsx::launch_merge_tee(*b, tb, st));
    f->launches++;
  }
  f->merges++;
  f->merged_rows += b->total_item_rows;
  return FSX_OK;
}

int fsx_synth_payload(fsx_fabric* f, int gpu, uint64_t seed, void* d_dst, int64_t n,
                      void* stream) {
  int ordinal = 0;
  int rc = find_gpu(f, gpu, &ordinal);
  if (rc) return rc;
  if (n < 0) return fail(FSX_E_VALIDATION, "negative byte count");
  if (n == 0) return FSX_OK;
  Device* dev = nullptr;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    rc = device_state(f, ordinal, &dev);
    if (rc) return rc;
  }
  FSX_CUDA(cudaSetDevice(ordinal));
  const int64_t pairs = (n / 16) + 1;
  const int grid = (int)std::min<int64_t>((pairs + 255) / 256, (int64_t)dev->sms * 8);
  FSX_CUDA(fsx::launch_synth(seed, static_cast<uint8_t*>(d_dst), n, std::max(grid, 1),
                             pick_stream(dev, stream)));
  f->launches++;
  return FSX_OK;
}

int fsx_copy_engine(fsx_fabric* f, int src_gpu, void* d_dst, const void* d_src, int64_t n,
                    void* stream) {
  int ordinal = 0;
  int rc = find_gpu(f, src_gpu, &ordinal);
  if (rc) return rc;
  if (n < 0) return fail(FSX_E_VALIDATION, "negative byte count");
  Device* dev = nullptr;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    rc = device_state(f, ordinal, &dev);
    if (rc) return rc;
  }
  FSX_CUDA(cudaSetDevice(ordinal));
  if (n) FSX_CUDA(cudaMemcpyAsync(d_dst, d_src, n, cudaMemcpyDefault, pick_stream(dev, stream)));
  return FSX_OK;
}

int fsx_pointer_device(const void* p, int* device) {
  *device = -1;
  if (!p) return FSX_OK;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return FSX_OK;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) *device = a.device;
  return FSX_OK;
}

int fsx_pointer_kind(const void* p, int* kind) {
  *kind = FSX_PTR_PAGEABLE;
  if (!p) return FSX_OK;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return FSX_OK;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) *kind = FSX_PTR_DEVICE;
  else if (a.type == cudaMemoryTypeHost) *kind = FSX_PTR_PINNED;
  return FSX_OK;
}

int fsx_copy_to_host(void* h_dst, const void* d_src, int64_t n) {
  if (n < 0) return fail(FSX_E_VALIDATION, "negative byte count");
  if (n == 0) return FSX_OK;
  FSX_CUDA(cudaMemcpy(h_dst, d_src, n, cudaMemcpyDefault));
  return FSX_OK;
}

// ---------------------------------------------------------------------------
// Streaming channels

namespace {

int state_slot(fsx_fabric* f, Device* d, uint64_t** out) {
  if (!d->state) {
    FSX_CUDA(cudaSetDevice(d->ordinal));
    FSX_CUDA(cudaMalloc(&d->state, kStatePool * sizeof(uint64_t)));
    FSX_CUDA(cudaMemset(d->state, 0, kStatePool * sizeof(uint64_t)));
  }
  if (d->state_next >= kStatePool) return fail(FSX_E_OOM, "channel state pool exhausted");
  *out = d->state + d->state_next++;
  FSX_CUDA(cudaSetDevice(d->ordinal));
  FSX_CUDA(cudaMemset(*out, 0, sizeof(uint64_t)));
  (void)f;
  return FSX_OK;
}

// One launch's rows: channel + the row's producer source (push) or consumer
// output (pull).
struct ChanIo {
  int32_t ch;
  uint8_t* io;
};

int build_step(fsx_fabric* f, int32_t n, const ChanIo* rows, bool push, fsx::ChanStep* st,
               int* device) {
  st->n = n;
  for (int32_t i = 0; i < n; ++i) {
    const int32_t ch = rows[i].ch;
    if (ch < 0 || ch >= (int32_t)f->channels.size() || !f->channels[ch].open)
      return fail(FSX_E_NOT_FOUND, "unknown or closed channel " + std::to_string(ch));
    const Channel& c = f->channels[ch];
    const int dev = push ? c.src_dev : c.dst_dev;
    if (i == 0) *device = dev;
    else if (dev != *device) return fail(FSX_E_VALIDATION, "channels of one step must share a device");
    Slab* s = slab_of(f, c.dst_gpu);
    fsx::ChanRow& r = st->c[i];
    r.ring = s->base + c.ring_off;
    r.flags = s->dflags + c.flag_base;
    r.head = c.head;
    r.tail = c.tail;
    r.salt = c.salt;
    r.slots = c.slots;
    r.row_bytes = c.row_bytes;
    r.peer = (s->imported || c.src_dev != c.dst_dev) ? 1 : 0;
    r.io = rows[i].io;
  }
  return FSX_OK;
}

// Every group's rows in launches of up to kChanMaxRows rows (one launch for a
// whole decode step of up to 48 streams, whatever their row sizes).
int chan_step(fsx_fabric* f, int32_t n_groups, const fsx_chan_group* groups, bool push,
              void* stream) {
  if (n_groups < 0) return fail(FSX_E_VALIDATION, "negative group count");
  std::vector<ChanIo> rows;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    for (int32_t g = 0; g < n_groups; ++g) {
      const fsx_chan_group& gr = groups[g];
      if (gr.n < 0) return fail(FSX_E_VALIDATION, "negative channel count");
      if (gr.n > 0 && !gr.channels) return fail(FSX_E_VALIDATION, "null channel list");
      for (int32_t i = 0; i < gr.n; ++i) {
        const int32_t ch = gr.channels[i];
        if (ch >= 0 && ch < (int32_t)f->channels.size() && gr.stride < (int64_t)f->channels[ch].row_bytes)
          return fail(FSX_E_VALIDATION, "row stride below row size");
        rows.push_back({ch, static_cast<uint8_t*>(gr.d_rows) + i * gr.stride});
      }
    }
  }
  const int32_t n = (int32_t)rows.size();
  for (int32_t first = 0; first < n; first += fsx::kChanMaxRows) {
    const int32_t cnt = std::min<int32_t>(n - first, fsx::kChanMaxRows);
    fsx::ChanStep st{};
    int device = 0;
    Device* dev = nullptr;
    {
      std::lock_guard<std::mutex> lk(f->mu);
      int rc = build_step(f, cnt, rows.data() + first, push, &st, &device);
      if (rc) return rc;
      rc = device_state(f, device, &dev);
      if (rc) return rc;
    }
    FSX_CUDA(cudaSetDevice(device));
    cudaStream_t s = pick_stream(dev, stream);
    FSX_CUDA(push ? fsx::launch_chan_push(st, s) : fsx::launch_chan_pull(st, s));
    f->launches++;
    if (push) {
      f->forwards += cnt;
      for (int32_t i = 0; i < cnt; ++i) f->bytes_forwarded += st.c[i].row_bytes;
    }
  }
  return FSX_OK;
}

}  // namespace

int fsx_channel_open(fsx_fabric* f, int src_gpu, int dst_gpu, int64_t row_bytes, int32_t slots,
                     int32_t* channel) {
  int src_dev = 0, dst_dev = 0;
  int rc = find_gpu(f, src_gpu, &src_dev);
  if (rc) return rc;
  rc = find_gpu(f, dst_gpu, &dst_dev);
  if (rc) return rc;
  if (row_bytes <= 0 || row_bytes > (int64_t{1} << 30) || slots <= 0 || slots > 4096)
    return fail(FSX_E_VALIDATION, "bad channel geometry");
  std::lock_guard<std::mutex> lk(f->mu);
  Slab* s = slab_of(f, dst_gpu);
  if (!s || s->imported) return fail(FSX_E_NOT_FOUND, "no owned slab for the consumer gpu");
  Channel c;
  c.src_gpu = src_gpu;
  c.dst_gpu = dst_gpu;
  c.src_dev = src_dev;
  c.dst_dev = dst_dev;
  c.slots = (uint32_t)slots;
  c.row_bytes = (uint32_t)row_bytes;
  c.ring_off = s->blocks.alloc(row_bytes * slots);
  if (c.ring_off < 0) return fail(FSX_E_OOM, "consumer slab cannot hold the channel ring");
  c.flag_base = s->flags.take(slots);
  Device *ps = nullptr, *cs = nullptr;
  rc = device_state(f, src_dev, &ps);
  if (!rc) rc = device_state(f, dst_dev, &cs);
  if (!rc) rc = state_slot(f, ps, &c.head);
  if (!rc) rc = state_slot(f, cs, &c.tail);
  if (rc) {
    s->blocks.release(c.ring_off);
    return rc;
  }
  c.salt = (uint64_t)(f->channels.size() + 1) << 40;
  c.open = true;
  *channel = (int32_t)f->channels.size();
  f->channels.push_back(c);
  return FSX_OK;
}

int fsx_channel_close(fsx_fabric* f, int32_t channel) {
  std::lock_guard<std::mutex> lk(f->mu);
  if (channel < 0 || channel >= (int32_t)f->channels.size() || !f->channels[channel].open)
    return fail(FSX_E_NOT_FOUND, "unknown or closed channel");
  Channel& c = f->channels[channel];
  Slab* s = slab_of(f, c.dst_gpu);
  if (s) s->blocks.release(c.ring_off);
  c.open = false;
  return FSX_OK;
}

int fsx_channel_push(fsx_fabric* f, int32_t n, const int32_t* channels, const void* d_rows,
                     int64_t row_stride, void* stream) {
  NvtxRange nvtx_range("fsx.channel_push");
  const fsx_chan_group g{n, channels, const_cast<void*>(d_rows), row_stride};
  return chan_step(f, 1, &g, true, stream);
}

int fsx_channel_pull(fsx_fabric* f, int32_t n, const int32_t* channels, void* d_out,
                     int64_t out_stride, void* stream) {
  NvtxRange nvtx_range("fsx.channel_pull");
  const fsx_chan_group g{n, channels, d_out, out_stride};
  return chan_step(f, 1, &g, false, stream);
}

int fsx_channel_push_groups(fsx_fabric* f, int32_t n_groups, const fsx_chan_group* groups,
                            void* stream) {
  NvtxRange nvtx_range("fsx.channel_push");
  return chan_step(f, n_groups, groups, true, stream);
}

int fsx_channel_pull_groups(fsx_fabric* f, int32_t n_groups, const fsx_chan_group* groups,
                            void* stream) {
  NvtxRange nvtx_range("fsx.channel_pull");
  return chan_step(f, n_groups, groups, false, stream);
}

int fsx_channel_progress(fsx_fabric* f, int32_t channel, uint64_t* produced, uint64_t* consumed) {
  uint64_t *h = nullptr, *t = nullptr;
  {
    std::lock_guard<std::mutex> lk(f->mu);
    if (channel < 0 || channel >= (int32_t)f->channels.size())
      return fail(FSX_E_NOT_FOUND, "unknown channel");
    h = f->channels[channel].head;
    t = f->channels[channel].tail;
  }
  FSX_CUDA(cudaMemcpy(produced, h, sizeof(uint64_t), cudaMemcpyDefault));
  FSX_CUDA(cudaMemcpy(consumed, t, sizeof(uint64_t), cudaMemcpyDefault));
  return FSX_OK;
}

int fsx_get_stats(fsx_fabric* f, fsx_stats* out) {
  std::memset(out, 0, sizeof(*out));
  out->forwards = f->forwards.load();
  out->bytes_forwarded = f->bytes_forwarded.load();
  out->merges = f->merges.load();
  out->merged_rows = f->merged_rows.load();
  out->kernel_launches = f->launches.load();
  out->dma_forwards = f->dma_forwards.load();
  std::lock_guard<std::mutex> lk(f->mu);
  for (auto& [g, s] : f->slabs) {
    out->segments_in_use += s->blocks.segments();
    out->bytes_in_use += s->blocks.bytes();
  }
  return FSX_OK;
}

int fsx_synchronize(fsx_fabric* f) {
  for (auto& [o, d] : f->devices) {
    FSX_CUDA(cudaSetDevice(o));
    FSX_CUDA(cudaStreamSynchronize(d->stream));
    if (d->notify) FSX_CUDA(cudaStreamSynchronize(d->notify));
  }
  return FSX_OK;
}

}  // extern "C"
