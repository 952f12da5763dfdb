// fsx/fabric.hpp -- C++ SidecarFabric engine over the libfsx C ABI.
//
// Re-implements the behaviour of the reference sidecar fabric
// (/root/reference/proj/include/fissim/sidecar.hpp:240-616) on B200 receive
// slabs:
//   * routing and topology            sidecar.hpp:250-260
//   * producer send + placement       sidecar.hpp:302-347, 465-483
//   * ordered per-ref delivery        sidecar.hpp:498-563
//   * raw (notify-then-read) interest sidecar.hpp:276-290
//   * backpressure backlog + timeout  sidecar.hpp:329-334, 571-602
//   * orphan reclaim                  sidecar.hpp:511-524
//   * fail_ref / purge / cancel       sidecar.hpp:292-297, 373-401
//   * stats                           sidecar.hpp:403-415
// The bytes never go through host arenas: every destination GPU owns a device
// slab (fsx_slab_*), payloads land there through K1 (device source, NVLink or
// HBM) or a host->device copy (host span), chunk flags gate delivery, and
// ChunkCallback consumers get an owned host vector (fsx_slab_read) while raw
// consumers read the slab in place (slab_ptr) and ack_raw() it.
//
// The engine is a template over a Traits policy so the same code runs
//   * standalone (fsx::StandaloneTraits below: fsx::EventLoop, fsx::Error,
//     fsx::DataRef) for this repo's own C++ tests, and
//   * as a drop-in for the reference (include/fsx/dropin/fissim/sidecar.hpp:
//     fissim::SimKernel, fissim::Error, fissim::DataRef, fissim::ForwardEnvelope).
//
// Threading: like the reference (sidecar.hpp:299-301, 604-615) every method
// runs on the event-kernel thread; the engine holds no locks of its own.
#pragma once

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <queue>
#include <set>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#if defined(__linux__)
#include <sys/mman.h>
#endif

#include "fsx.h"

// Phase hooks for host-overhead probes (tests/cpp/probe_send_phases.cpp
// defines it before including this header); compiled out otherwise.
#ifndef FSX_PHASE
#define FSX_PHASE(i) ((void)0)
#endif

namespace fsx {

enum class Transport { LocalBuffer, NetworkStream };

inline const char* transport_name(Transport t) {
  return t == Transport::LocalBuffer ? "local_buffer" : "network_stream";
}

// Same knobs as the reference SidecarConfig (sidecar.hpp:38-57); the modeled
// latency keeps event timestamps identical to the reference in Virtual mode.
struct SidecarConfig {
  int64_t arena_bytes = int64_t{1} << 30;  // per destination GPU slab
  double local_base_ms = 0.5;
  double local_per_mb_ms = 0.8125;
  double net_base_ms = 1.0;
  double net_per_mb_ms = 0.8125;
  double send_timeout_ms = 10000;
  double orphan_timeout_ms = 30000;
  int64_t stream_chunk_bytes = 256 * 1024;
  // fsx additions
  int64_t device_chunk_bytes = int64_t{8} << 20;  // flag granularity of K1 pushes
  int64_t wait_timeout_us = 30'000'000;            // GPU completion watchdog
  // send() borrows its span for the call only (sidecar.hpp:302, 327).  A
  // pageable host span is fully copied out before the copy call returns, so
  // send() then returns without waiting for the bytes to land; the delivery
  // waits instead (if it comes first).  Device spans and pinned host spans
  // are read by the GPU asynchronously, so send() waits for them -- unless
  // the caller keeps them unchanged until the delivery (stream-ordered
  // producers), which this flag declares.
  bool async_borrowed_sources = false;

  double latency_ms(Transport t, int64_t bytes) const {
    const double mb = static_cast<double>(bytes) / (1024.0 * 1024.0);
    return t == Transport::LocalBuffer ? local_base_ms + local_per_mb_ms * mb
                                       : net_base_ms + net_per_mb_ms * mb;
  }
};

struct SidecarStats {
  int64_t transfers = 0;
  int64_t bytes_forwarded = 0;
  int64_t integrity_errors = 0;
  int64_t orphan_reclaims = 0;
  double added_latency_ms = 0;
  size_t segments_in_use = 0;
  int64_t bytes_in_use = 0;
};

// Wire checksum of the envelope (common.hpp:221-241), needed bit-for-bit for
// interop with reference peers on the network transport.
inline uint64_t checksum64(const uint8_t* p, size_t n) {
  constexpr uint64_t kMul = 0x2545f4914f6cdd1dull;
  uint64_t h = 0x9e3779b97f4a7c15ull ^ (static_cast<uint64_t>(n) * 0xff51afd7ed558ccdull);
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    uint64_t w;
    std::memcpy(&w, p + i, 8);
    h = (h ^ w) * kMul;
    h ^= h >> 29;
  }
  uint64_t tail = 0;
  for (unsigned sh = 0; i < n; ++i, sh += 8) tail |= static_cast<uint64_t>(p[i]) << sh;
  h = (h ^ tail) * kMul;
  return h ^ (h >> 32);
}

// dg64, the lane-parallel device digest (include/fsx.h): host form, used for
// host-span payloads whose bytes never pass through K1's registers.
// Sum of the dg64 word terms for words [k0, k1) of p[0..n) (the sum is mod
// 2^64, so word ranges add up independently).
inline uint64_t digest64_words(const uint8_t* p, size_t n, size_t k0, size_t k1) {
  constexpr uint64_t C1 = 0xbf58476d1ce4e5b9ull, C2 = 0x94d049bb133111ebull;
  // the per-word terms are independent: four accumulators keep the
  // multiplier busy, 2.8x faster than one chain
  uint64_t h0 = 0, h1 = 0, h2 = 0, h3 = 0;
  const size_t full = std::min(k1, n / 8);
  size_t k = k0;
  uint64_t c = static_cast<uint64_t>(k0 + 1) * C1;  // (k + 1) * C1
  for (; k + 4 <= full; k += 4, c += 4 * C1) {
    uint64_t w[4];
    std::memcpy(w, p + k * 8, 32);  // little-endian host
    const uint64_t y0 = (w[0] ^ c) * C2, y1 = (w[1] ^ (c + C1)) * C2;
    const uint64_t y2 = (w[2] ^ (c + 2 * C1)) * C2, y3 = (w[3] ^ (c + 3 * C1)) * C2;
    h0 += y0 ^ (y0 >> 29);
    h1 += y1 ^ (y1 >> 29);
    h2 += y2 ^ (y2 >> 29);
    h3 += y3 ^ (y3 >> 29);
  }
  for (; k < k1 && k * 8 < n; ++k, c += C1) {
    uint64_t w = 0;
    const size_t take = n - k * 8 < 8 ? n - k * 8 : 8;
    std::memcpy(&w, p + k * 8, take);  // zero-padded tail
    const uint64_t y = (w ^ c) * C2;
    h0 += y ^ (y >> 29);
  }
  return h0 + h1 + h2 + h3;
}

inline uint64_t digest64(const uint8_t* p, size_t n) {
  return static_cast<uint64_t>(n) * 0x9e3779b97f4a7c15ull + digest64_words(p, n, 0, (n + 7) / 8);
}

// digest64 of a large host span on several threads (embeddings of tens of
// MiB would otherwise cost ~10 ms per 112 MiB on one core).
inline uint64_t digest64_par(const uint8_t* p, size_t n) {
  constexpr size_t kMin = size_t{16} << 20;
  const size_t hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t parts = std::min<size_t>({hw, size_t{8}, n / kMin});
  if (parts < 2) return digest64(p, n);
  const size_t words = (n + 7) / 8, per = (words + parts - 1) / parts;
  std::vector<uint64_t> partial(parts, 0);
  std::vector<std::thread> th;
  for (size_t t = 1; t < parts; ++t)
    th.emplace_back([&, t] { partial[t] = digest64_words(p, n, t * per, std::min(words, (t + 1) * per)); });
  partial[0] = digest64_words(p, n, 0, std::min(words, per));
  for (auto& x : th) x.join();
  uint64_t h = static_cast<uint64_t>(n) * 0x9e3779b97f4a7c15ull;
  for (uint64_t v : partial) h += v;
  return h;
}

// An owned byte vector of n bytes for a delivery (ChunkCallback takes the
// vector by value, sidecar.hpp:543-544, 561).  Large ones are advised onto
// transparent huge pages before their first touch: a fresh 112 MiB vector
// otherwise costs ~28 k page faults (43 ms on the B200 hosts, 14 ms advised).
inline std::vector<uint8_t> owned_buffer(size_t n) {
  std::vector<uint8_t> v;
#if defined(__linux__) && defined(MADV_HUGEPAGE)
  constexpr size_t kHuge = size_t{2} << 20;
  if (n >= 4 * kHuge) {
    v.reserve(n);
    const uintptr_t p = reinterpret_cast<uintptr_t>(v.data());
    const uintptr_t a = (p + kHuge - 1) & ~uintptr_t(kHuge - 1);
    if (a < p + n) madvise(reinterpret_cast<void*>(a), (p + n - a) & ~uintptr_t(kHuge - 1), MADV_HUGEPAGE);
  }
#endif
  v.resize(n);
  return v;
}

// Status codes of the C ABI are 1 + fissim::ErrorCode ordinal.
namespace status {
constexpr int kValidation = FSX_E_VALIDATION;
constexpr int kNotFound = FSX_E_NOT_FOUND;
constexpr int kIntegrity = FSX_E_INTEGRITY;
constexpr int kProtocol = FSX_E_PROTOCOL;
constexpr int kTimeout = FSX_E_TIMEOUT;
constexpr int kConfig = FSX_E_CONFIG;
constexpr int kInternal = FSX_E_INTERNAL;
}  // namespace status

template <class Traits>
class Fabric {
 public:
  using Kernel = typename Traits::Kernel;
  using Envelope = typename Traits::Envelope;
  using Error = typename Traits::Error;
  using Ref = typename Traits::DataRef;
  using ChunkCallback = std::function<void(const Envelope&, std::vector<uint8_t>)>;
  using RefErrorCallback = std::function<void(const Error&)>;
  using RawChunkCallback = std::function<void(const Envelope&, int64_t)>;
  // Early start (fsx addition): the segment's offset plus the chunk flags its
  // bytes are landing under -- chunk c is in the slab once flag
  // flag_base + c of the destination GPU equals token (fsx_stream_wait_flags,
  // an early-start fsx_merge, fsx_wait, fsx_chunk_ready).
  struct ChunkFlags {
    int64_t flag_base = 0;
    int32_t n_chunks = 0;  // 0: already landed (small message / staged network arrival)
    uint64_t token = 0;
    int64_t chunk_bytes = 0;
  };
  using EarlyChunkCallback = std::function<void(const Envelope&, int64_t offset, const ChunkFlags&)>;
  using FailureHandler = std::function<void(const std::string&, const std::string&, const Error&)>;

  // devices: logical gpu -> CUDA ordinal (missing -> gpu % device_count).
  Fabric(Kernel& kernel, std::map<int, int> gpu_to_node, SidecarConfig config = {},
         std::map<int, int> devices = {})
      : kernel_(kernel), topo_(std::move(gpu_to_node)), config_(config) {
    std::vector<int> ids, nodes, devs;
    for (const auto& [g, n] : topo_) {
      ids.push_back(g);
      nodes.push_back(n);
      auto it = devices.find(g);
      devs.push_back(it == devices.end() ? -1 : it->second);
    }
    fsx_fabric* h = nullptr;
    check(fsx_open(static_cast<int>(ids.size()), ids.data(), nodes.data(), devs.data(), &h));
    h_ = h;
  }

  Fabric(const Fabric&) = delete;
  Fabric& operator=(const Fabric&) = delete;

  ~Fabric() {
    if (h_) fsx_close(h_);
  }

  // -- topology (sidecar.hpp:250-260) -----------------------------------------
  Transport route(int src_gpu, int dst_gpu) const {
    return node_of(src_gpu) == node_of(dst_gpu) ? Transport::LocalBuffer : Transport::NetworkStream;
  }

  int node_of(int gpu) const {
    auto it = topo_.find(gpu);
    if (it == topo_.end())
      Traits::raise(status::kNotFound, "gpu " + std::to_string(gpu) + " not in topology map");
    return it->second;
  }

  // -- consumer side (sidecar.hpp:263-297) -----------------------------------
  void register_interest(int gpu, const std::string& ref_id, ChunkCallback on_chunk,
                         RefErrorCallback on_error = {}) {
    node_of(gpu);
    RefState& st = refs_[key_of(ref_id, gpu)];
    st.dst_gpu = gpu;
    st.on_chunk = std::move(on_chunk);
    st.raw_cb = nullptr;
    st.on_error = std::move(on_error);
    st.has_interest = true;
    drain(st);
  }

  void register_interest_raw(int gpu, const std::string& ref_id, RawChunkCallback on_chunk,
                             RefErrorCallback on_error = {}) {
    node_of(gpu);
    RefState& st = refs_[key_of(ref_id, gpu)];
    st.dst_gpu = gpu;
    st.raw_cb = std::move(on_chunk);
    st.on_error = std::move(on_error);
    st.has_interest = true;
    drain(st);
  }

  // Early-start interest (no reference counterpart; SURVEY.md 7 "hard parts"):
  // like register_interest_raw, but the callback runs when the payload is
  // PLACED -- on the sender's event, before the bytes have landed and before
  // the modeled delivery latency -- with the chunk flags that gate each
  // chunk, so a device consumer (an early-start merge, a prefill gated by
  // fsx_stream_wait_flags) can start on chunk 0 while later chunks are still
  // in flight.  Chunks are handed over in placement order (env.seq tells the
  // consumer where each goes); the consumer owns the segment until ack_raw.
  void register_interest_early(int gpu, const std::string& ref_id, EarlyChunkCallback on_chunk,
                               RefErrorCallback on_error = {}) {
    node_of(gpu);
    RefState& st = refs_[key_of(ref_id, gpu)];
    st.dst_gpu = gpu;
    any_early_ = true;
    st.early_cb = std::move(on_chunk);
    st.on_chunk = nullptr;
    st.raw_cb = nullptr;
    st.on_error = std::move(on_error);
    st.has_interest = true;
    drain(st);
  }

  // Raw consumers release their segment.  `slab_gpu` is the destination GPU
  // whose slab holds it (the envelope location reads "gpu<G>:off<K>").
  // Only segments handed to a raw callback and not yet acked are accepted:
  // an ack naming any other (gpu, offset) -- e.g. a node id passed where the
  // reference's ack_raw(node, off) took one -- raises Internal instead of
  // freeing whatever live segment sits there.
  void ack_raw(int slab_gpu, int64_t offset) {
    FSX_PHASE(20);
    if (raw_held_.erase({slab_gpu, offset}) == 0)
      Traits::raise(status::kInternal, "ack_raw of gpu " + std::to_string(slab_gpu) + " offset " +
                                           std::to_string(offset) +
                                           ": no segment held by a raw consumer there");
    release_segment(slab_gpu, offset);
    FSX_PHASE(21);
    place_backlog(slab_gpu);
  }

  void cancel_interest(const std::string& ref_id, int gpu) {
    auto it = refs_.find(key_of(ref_id, gpu));
    if (it == refs_.end()) return;
    drop_parked(it->second);
    refs_.erase(it);
  }

  // Device view of a delivered segment (zero-copy read for raw consumers).
  void* slab_ptr(int gpu, int64_t offset) {
    void* p = nullptr;
    check(fsx_slab_ptr(h_, gpu, offset, &p));
    return p;
  }

  // -- producer side (sidecar.hpp:302-347, 367-370) --------------------------
  // `payload` may point to host memory (copied host->device into the consumer
  // slab) or to device memory of src_gpu's device (pushed by K1 over NVLink or
  // HBM).  The span is borrowed for the duration of the call only.
  void send(const std::string& request_id, const Ref& ref, int src_gpu, int dst_gpu,
            std::span<const uint8_t> payload, int64_t seq, bool final_chunk) {
    FSX_PHASE(14);
    const int64_t n = static_cast<int64_t>(payload.size());
    if (!Traits::streaming(ref) && n != Traits::total_bytes(ref))
      Traits::raise(status::kProtocol, "payload length " + std::to_string(n) +
                                           " does not match descriptor total_bytes " +
                                           std::to_string(Traits::total_bytes(ref)) + " for ref " +
                                           Traits::ref_id(ref));
    const Transport t = route(src_gpu, dst_gpu);
    Pending ps;
    ps.env.request_id = request_id;
    ps.env.ref_id = Traits::ref_id(ref);
    ps.env.seq = seq;
    ps.env.chunk_bytes = n;
    ps.env.total_bytes = Traits::total_bytes(ref);
    Traits::set_transport(ps.env, t == Transport::LocalBuffer);
    ps.env.final = final_chunk;
    ps.env.send_time = Traits::now(kernel_);
    ps.env.src_gpu = src_gpu;
    ps.env.dst_gpu = dst_gpu;
    ps.deadline = Traits::now(kernel_) + config_.send_timeout_ms;
    ps.src = payload.data();
    FSX_PHASE(0);
    ps.src_is_device = n > 0 && device_of_pointer(payload.data()) >= 0;
    FSX_PHASE(1);

    if (t == Transport::NetworkStream) {
      // Cross-node: envelope and bytes travel together (sidecar.hpp:337-346),
      // staged into the destination slab on arrival.
      ps.env.checksum = checksum64_any(ps);
      own_bytes(ps);
      const double lat = config_.latency_ms(t, n);
      added_latency_ms_ += lat;
      auto shared = std::make_shared<Pending>(std::move(ps));
      Traits::schedule(kernel_, Traits::now(kernel_) + lat, "sidecar.net_deliver",
                       [this, shared] { handle_network(shared->env, std::move(shared->bytes)); });
      return;
    }
    // local: the envelope carries dg64 (set while placing: fused into K1 for
    // device payloads, host digest for host spans), not the serial checksum64
    ps.env.checksum = 0;
    if (!place_local(ps)) {
      own_bytes(ps);  // borrowed span dies with the call: keep the bytes for the backlog
      const int slab = ps.env.dst_gpu;
      backlog_[slab].push_back(std::move(ps));
      arm_timeout(slab);
    }
  }

  void send_payload(const std::string& request_id, const Ref& ref, int src_gpu, int dst_gpu,
                    std::span<const uint8_t> payload) {
    send(request_id, ref, src_gpu, dst_gpu, payload, 0, true);
  }

  // Network arrival (sidecar.hpp:351-364, 487-496): verify, stage, deliver now.
  void handle_network(Envelope env, std::vector<uint8_t> bytes) {
    if (env.chunk_bytes != static_cast<int64_t>(bytes.size()))
      Traits::raise(status::kProtocol, "network envelope chunk_bytes mismatch for ref " + env.ref_id);
    Pending ps;
    ps.env = std::move(env);
    ps.bytes = std::move(bytes);
    ps.owned = true;
    ps.src = ps.bytes.data();
    ps.deadline = Traits::now(kernel_) + config_.send_timeout_ms;
    ps.network = true;
    if (!stage_network(ps)) {
      const int slab = ps.env.dst_gpu;
      backlog_[slab].push_back(std::move(ps));
      arm_timeout(slab);
    }
  }

  // -- failure and cleanup (sidecar.hpp:373-401) ------------------------------
  void fail_ref(const std::string& ref_id, const Error& err) {
    const std::string prefix = ref_id + "@";
    for (auto it = refs_.lower_bound(prefix); it != refs_.end(); ++it) {
      if (it->first.compare(0, prefix.size(), prefix) != 0) break;
      it->second.failed = std::make_shared<Error>(err);
      if (it->second.on_error) it->second.on_error(err);
    }
  }

  void purge_request(const std::string& request_id) {
    const std::string prefix = request_id + "/";
    for (auto it = refs_.begin(); it != refs_.end();) {
      const bool mine = it->second.request_id == request_id ||
                        (it->first.size() > prefix.size() && it->first.compare(0, prefix.size(), prefix) == 0);
      if (mine) {
        drop_parked(it->second);
        it = refs_.erase(it);
      } else {
        ++it;
      }
    }
    for (auto& [slab, q] : backlog_) {
      q.erase(std::remove_if(q.begin(), q.end(),
                             [&](const Pending& p) { return p.env.request_id == request_id; }),
              q.end());
    }
  }

  SidecarStats stats() const {
    SidecarStats s;
    s.transfers = transfers_;
    s.bytes_forwarded = bytes_forwarded_;
    s.integrity_errors = integrity_errors_;
    s.orphan_reclaims = orphan_reclaims_;
    s.added_latency_ms = added_latency_ms_;
    for (int g : slabs_) {
      int64_t segs = 0, used = 0;
      if (fsx_slab_usage(h_, g, &segs, &used, nullptr, nullptr) == FSX_OK) {
        s.segments_in_use += static_cast<size_t>(segs);
        s.bytes_in_use += used;
      }
    }
    return s;
  }

  // CUDA IPC export of gpu's receive slab (created on first use), for worker
  // processes that read delivered segments in place: the role of the shm
  // arena name in the reference's worker handshake (executor_worker.hpp:63-87).
  int64_t export_slab(int gpu, void* handle64) {
    node_of(gpu);
    ensure_slab(gpu);
    int64_t bytes = 0;
    check(fsx_slab_export(h_, gpu, handle64, &bytes));
    return bytes;
  }

  const SidecarConfig& config() const { return config_; }
  void set_failure_handler(FailureHandler fn) { failure_handler_ = std::move(fn); }
  fsx_fabric* handle() const { return h_; }

 private:
  // A delivered chunk waiting for its turn: envelope, slab offset, and the
  // small-message ticket (fsx_put_small) whose read-back it owns, or -1.
  // Chunk flags of a placement still in flight (n_chunks 0: landed).
  struct Landing {
    int64_t flag_base = 0;
    int32_t n_chunks = 0;
    uint64_t token = 0;
  };

  struct Parked {
    Envelope env;
    int64_t off = -1;
    int64_t ticket = -1;
    bool network = false;  // arrived as a network frame: verify the sender's checksum64
    Landing landing;       // waited for before the bytes are handed over
  };

  struct RefState {
    std::string request_id;
    int dst_gpu = -1;
    bool has_interest = false;
    ChunkCallback on_chunk;
    RawChunkCallback raw_cb;
    EarlyChunkCallback early_cb;  // handed the segment at placement, before it lands
    RefErrorCallback on_error;
    int64_t next_seq = 0;
    std::map<int64_t, Parked> parked;  // by seq
    std::shared_ptr<Error> failed;
  };

  struct Pending {
    Envelope env;
    std::vector<uint8_t> bytes;  // owned copy (backlog / network)
    const uint8_t* src = nullptr;
    bool owned = false;
    bool src_is_device = false;
    bool network = false;
    double deadline = 0;
  };

  void check(int rc) const {
    if (rc != FSX_OK) Traits::raise(rc, fsx_last_error());
  }

  static std::string key_of(const std::string& ref_id, int gpu) {
    return ref_id + "@" + std::to_string(gpu);
  }

  // ForwardEnvelope::location of a slab segment: "gpu<G>:off<K>"
  static std::string location_of(int gpu, int64_t off) {
    char buf[48] = {'g', 'p', 'u'};
    char* p = std::to_chars(buf + 3, buf + 16, gpu).ptr;
    std::memcpy(p, ":off", 4);
    p = std::to_chars(p + 4, buf + sizeof buf, off).ptr;
    return std::string(buf, static_cast<size_t>(p - buf));
  }

  static int device_of_pointer(const void* p) {
    int dev = -1;
    if (fsx_pointer_device(p, &dev) != FSX_OK) return -1;
    return dev;
  }

  // Bytes of a pending send on the host (network checksum / backlog copies).
  void own_bytes(Pending& ps) {
    if (ps.owned) return;
    const int64_t n = ps.env.chunk_bytes;
    ps.bytes = owned_buffer(static_cast<size_t>(n));
    if (n > 0) {
      if (ps.src_is_device) check(fsx_copy_to_host(ps.bytes.data(), ps.src, n));
      else std::memcpy(ps.bytes.data(), ps.src, static_cast<size_t>(n));
    }
    ps.owned = true;
    ps.src_is_device = false;
    ps.src = ps.bytes.data();
  }

  uint64_t checksum64_any(Pending& ps) {
    if (ps.src_is_device) own_bytes(ps);
    return checksum64(ps.src, static_cast<size_t>(ps.env.chunk_bytes));
  }

  void ensure_slab(int gpu) {
    if (std::find(slabs_.begin(), slabs_.end(), gpu) != slabs_.end()) return;
    check(fsx_slab_register(h_, gpu, config_.arena_bytes));
    slabs_.push_back(gpu);
  }

  // Allocate a segment and start moving the bytes; false when the slab is full.
  bool start_copy(Pending& ps, int64_t* off, uint64_t* token, int64_t* flag_base, int32_t* n_chunks,
                  int64_t* ticket) {
    const int dst = ps.env.dst_gpu;
    ensure_slab(dst);
    const int64_t n = ps.env.chunk_bytes;
    *ticket = -1;
    FSX_PHASE(2);
    if (n > 0 && n <= FSX_SMALL_MAX) {
      // small span (per-token hidden states, codes): segment allocated and
      // the message published on the destination's small-message lane in one
      // call -- a host span staged, a device span read in place; the lane
      // kernel digests the bytes it moves (sent) and the landed segment,
      // read at delivery
      check(fsx_put_small_alloc(h_, dst, ps.src, n, ps.src_is_device ? 1 : 0, off, ticket));
      FSX_PHASE(4);
      if (*off < 0) return false;
      if (*ticket >= 0) {
        *n_chunks = 0;
        *token = 0;
        digest_slot_ = nullptr;
        return true;
      }
    } else {
      check(fsx_slab_alloc(h_, dst, std::max<int64_t>(n, 1), off));
      FSX_PHASE(3);
      if (*off < 0) return false;
    }
    // The envelope's checksum is the producer's: dg64 set here for local
    // sends; a network arrival keeps the sender's checksum64 whatever its
    // transport tag says (sidecar.hpp:351-364 verifies the frame as sent).
    const bool local = Traits::is_local(ps.env) && !ps.network;
    int64_t cb = config_.device_chunk_bytes;
    // host spans cross PCIe: every copy costs a fixed copy-engine gap, so
    // they go in chunks of at least 32 MiB (send() waits for all of it anyway)
    if (!ps.src_is_device && cb > 0) cb = std::max<int64_t>(cb, int64_t{32} << 20);
    if (cb <= 0 || cb >= n) cb = 0;
    *n_chunks = cb ? static_cast<int32_t>((n + cb - 1) / cb) : 1;
    check(fsx_flags_alloc(h_, dst, *n_chunks, flag_base));
    *token = 0;
    if (ps.src_is_device) {
      // K1, with the dg64 digest of the source fused into the copy
      fsx_transfer t{ps.env.src_gpu, dst, ps.src, *off, n, cb, *flag_base, 0, nullptr};
      if (local) check(fsx_u64_slot(h_, ps.env.src_gpu, &t.d_digest, nullptr));
      check(fsx_forward_batch(h_, 1, &t, FSX_FWD_HOST_NOTIFY, nullptr));
      *token = t.token;
      digest_slot_ = t.d_digest;
    } else {
      // host span: staged (pageable) or DMA'd (pinned) into the slab; its
      // dg64 is computed in the same pass that stages it
      uint64_t dg = 0;
      check(fsx_forward_host_digest(h_, ps.src, dst, *off, n, cb, *flag_base, token, nullptr,
                                    local ? &dg : nullptr));
      if (local) ps.env.checksum = dg;
      digest_slot_ = nullptr;
    }
    return true;
  }

  void wait_landed(int dst, int64_t flag_base, int32_t n_chunks, uint64_t token) {
    check(fsx_wait(h_, dst, flag_base, n_chunks, token, config_.wait_timeout_us));
  }

  // dg64 of a delivered slab segment, recomputed on the consumer GPU.
  uint64_t slab_digest(int gpu, int64_t off, int64_t n) {
    uint64_t* slot = nullptr;
    check(fsx_u64_slot(h_, gpu, &slot, nullptr));
    void* p = nullptr;
    check(fsx_slab_ptr(h_, gpu, off, &p));
    check(fsx_digest(h_, gpu, p, n, slot, nullptr));
    uint64_t v = 0;
    check(fsx_read_u64(h_, gpu, slot, &v, nullptr));
    return v;
  }

  // sidecar.hpp:465-483: place now, notify after the modeled latency.
  bool place_local(Pending& ps) {
    int64_t off = -1, flag_base = 0, ticket = -1;
    uint64_t token = 0;
    int32_t n_chunks = 1;
    if (!start_copy(ps, &off, &token, &flag_base, &n_chunks, &ticket)) return false;
    // The source is borrowed (caller span) or owned by a Pending about to be
    // dropped.  Where the GPU still reads it after the copy call -- a device
    // span under K1, a pinned host span under DMA -- the copy completes before
    // we return, like the reference's memcpy into the arena (sidecar.hpp:470).
    // A pageable host span has been copied out of by then (fsx_forward_host
    // stages it), and a small message sits in the pinned mailbox: send()
    // returns at once and the delivery waits for the landing instead.
    Landing landing{flag_base, ticket < 0 ? n_chunks : 0, token};
    // a staged small host span is copied out already; a small device span is
    // read by the lane kernel after this call
    const bool still_read = ticket >= 0 ? ps.src_is_device && !config_.async_borrowed_sources
                                        : source_still_read(ps);
    if (still_read) {
      if (ticket >= 0)
        check(fsx_ticket_wait(h_, ticket, nullptr, nullptr));  // the lane has read the device span
      else
        wait_landed(ps.env.dst_gpu, flag_base, n_chunks, token);
      landing.n_chunks = 0;
    }
    if (digest_slot_) check(fsx_read_u64(h_, ps.env.src_gpu, digest_slot_, &ps.env.checksum, nullptr));
    ps.env.location = location_of(ps.env.dst_gpu, off);
    const double lat = config_.latency_ms(Transport::LocalBuffer, ps.env.chunk_bytes);
    added_latency_ms_ += lat;
    if (any_early_ && hand_over_early(ps.env, off, ticket, landing)) return true;
    // the Pending is dropped once placed (send / place_backlog): move its envelope
    FSX_PHASE(5);
    auto env = std::make_shared<Envelope>(std::move(ps.env));
    Traits::schedule(kernel_, Traits::now(kernel_) + lat, "sidecar.deliver",
                     [this, env, off, ticket, landing] { deliver(std::move(*env), off, ticket, false, landing); });
    FSX_PHASE(6);
    return true;
  }

  // Does the GPU read the sender's bytes after the copy call returned?
  bool source_still_read(const Pending& ps) const {
    if (config_.async_borrowed_sources || ps.env.chunk_bytes == 0) return false;
    if (ps.src_is_device) return true;
    if (ps.owned) return false;  // our own pageable copy (backlog / network)
    int kind = 0;
    return fsx_pointer_kind(ps.src, &kind) == FSX_OK && kind == 1;  // pinned: DMA reads it
  }

  // An early-start consumer takes the segment at placement (see
  // register_interest_early); false when the ref has none.
  bool hand_over_early(const Envelope& env, int64_t off, int64_t ticket, const Landing& landing) {
    auto it = refs_.find(key_of(env.ref_id, env.dst_gpu));
    if (it == refs_.end() || !it->second.early_cb) return false;
    RefState& st = it->second;
    if (st.request_id.empty()) st.request_id = env.request_id;
    Envelope e = env;
    if (ticket >= 0) {  // a small message: in the slab once the lane served it
      uint64_t sent = 0;
      check(fsx_ticket_digests(h_, ticket, &sent, nullptr));
      if (Traits::is_local(e)) e.checksum = sent;
      drop_ticket(ticket);
    }
    ChunkFlags cf{landing.flag_base, landing.n_chunks, landing.token,
                  landing.n_chunks > 1 ? std::min<int64_t>(config_.device_chunk_bytes, e.chunk_bytes)
                                       : e.chunk_bytes};
    ++transfers_;
    bytes_forwarded_ += e.chunk_bytes;
    raw_held_.insert({e.dst_gpu, off});
    st.early_cb(e, off, cf);
    return true;
  }

  // sidecar.hpp:487-496: stage a network arrival into the slab, deliver now.
  bool stage_network(Pending& ps) {
    int64_t off = -1, flag_base = 0, ticket = -1;
    uint64_t token = 0;
    int32_t n_chunks = 1;
    if (!start_copy(ps, &off, &token, &flag_base, &n_chunks, &ticket)) return false;
    ps.env.location = location_of(ps.env.dst_gpu, off);
    if (ticket < 0) wait_landed(ps.env.dst_gpu, flag_base, n_chunks, token);
    deliver(ps.env, off, ticket, /*network=*/true);
    return true;
  }

  // sidecar.hpp:498-525
  void deliver(Envelope env, int64_t off, int64_t ticket = -1, bool network = false,
               Landing landing = {}) {
    FSX_PHASE(8);
    const std::string key = key_of(env.ref_id, env.dst_gpu);
    RefState& st = refs_[key];
    FSX_PHASE(9);
    if (st.request_id.empty()) st.request_id = env.request_id;
    if (st.failed) {
      drop_ticket(ticket);
      settle(landing, env.dst_gpu);  // no segment is reused while bytes still land in it
      release_segment(env.dst_gpu, off);
      place_backlog(env.dst_gpu);
      return;
    }
    const int64_t seq = env.seq;
    st.parked.emplace(seq, Parked{std::move(env), off, ticket, network, landing});
    if (st.has_interest) {
      drain(st);
      return;
    }
    Traits::schedule(kernel_, Traits::now(kernel_) + config_.orphan_timeout_ms, "sidecar.orphan",
                     [this, key, seq] { reclaim_orphan(key, seq); });
  }

  void reclaim_orphan(const std::string& key, int64_t seq) {
    auto it = refs_.find(key);
    if (it == refs_.end() || it->second.has_interest) return;
    auto p = it->second.parked.find(seq);
    if (p == it->second.parked.end()) return;
    const int slab = p->second.env.dst_gpu;
    drop_ticket(p->second.ticket);
    settle(p->second.landing, slab);
    release_segment(slab, p->second.off);
    it->second.parked.erase(p);
    ++orphan_reclaims_;
    place_backlog(slab);
  }

  // sidecar.hpp:527-563: in-order delivery of parked chunks.
  void drain(RefState& st) {
    for (auto it = st.parked.find(st.next_seq); it != st.parked.end();
         it = st.parked.find(st.next_seq)) {
      Envelope env = std::move(it->second.env);  // erased next
      const int64_t off = it->second.off;
      const int64_t ticket = it->second.ticket;
      const bool network = it->second.network;
      const Landing landing = it->second.landing;
      st.parked.erase(it);
      if (st.early_cb) {  // early interest registered after the placement
        if (ticket >= 0 && Traits::is_local(env) && !network) {
          uint64_t sent = 0;
          check(fsx_ticket_digests(h_, ticket, &sent, nullptr));
          env.checksum = sent;
        }
        drop_ticket(ticket);
        ++transfers_;
        bytes_forwarded_ += env.chunk_bytes;
        ++st.next_seq;
        raw_held_.insert({env.dst_gpu, off});
        ChunkFlags cf{landing.flag_base, landing.n_chunks, landing.token,
                      landing.n_chunks > 1 ? std::min<int64_t>(config_.device_chunk_bytes, env.chunk_bytes)
                                           : env.chunk_bytes};
        st.early_cb(env, off, cf);
        continue;
      }
      // a send that returned before its bytes landed: the delivery waits
      settle(landing, env.dst_gpu);
      if (st.raw_cb) {
        FSX_PHASE(18);
        if (ticket >= 0 && Traits::is_local(env) && !network) {
          uint64_t sent = 0;
          check(fsx_ticket_digests(h_, ticket, &sent, nullptr));
          env.checksum = sent;
        }
        drop_ticket(ticket);  // waits until the bytes are in the slab
        FSX_PHASE(19);
        ++transfers_;
        bytes_forwarded_ += env.chunk_bytes;
        ++st.next_seq;
        raw_held_.insert({env.dst_gpu, off});
        st.raw_cb(env, off);
        continue;
      }
      // Verify before handing the bytes over, like sidecar.hpp:545-557: the
      // device hop is checked with dg64 recomputed on the consumer GPU over
      // the slab segment, the network hop with the reference checksum64.
      const bool local = Traits::is_local(env) && !network;
      std::vector<uint8_t> bytes;
      bool dev_ok = true;
      if (ticket >= 0) {
        // small message: the lane kernel digested the bytes it moved (the
        // producer's, as staged by send) and the segment read back from the
        // slab; the consumer gets the staged bytes
        uint64_t sent = 0, landed = 0;
        bytes.resize(static_cast<size_t>(env.chunk_bytes));
        FSX_PHASE(10);
        check(fsx_ticket_take(h_, ticket, bytes.data(), env.chunk_bytes, &sent, &landed));
        FSX_PHASE(11);
        if (local) env.checksum = sent;
        dev_ok = landed == sent;
      } else {
        bytes = owned_buffer(static_cast<size_t>(env.chunk_bytes));
        dev_ok = !local || slab_digest(env.dst_gpu, off, env.chunk_bytes) == env.checksum;
        if (env.chunk_bytes > 0)
          check(fsx_slab_read(h_, env.dst_gpu, off, bytes.data(), env.chunk_bytes, nullptr));
      }
      const bool ok = local ? dev_ok : checksum64(bytes.data(), bytes.size()) == env.checksum;
      release_segment(env.dst_gpu, off);
      place_backlog(env.dst_gpu);
      if (!ok) {
        ++integrity_errors_;
        Error err = Traits::make_error(status::kIntegrity, "checksum mismatch on ref " + env.ref_id +
                                                               " seq " + std::to_string(env.seq));
        st.failed = std::make_shared<Error>(err);
        if (st.on_error) st.on_error(err);
        if (failure_handler_) failure_handler_(env.request_id, env.ref_id, err);
        return;
      }
      ++transfers_;
      bytes_forwarded_ += env.chunk_bytes;
      ++st.next_seq;
      FSX_PHASE(12);
      if (st.on_chunk) st.on_chunk(env, std::move(bytes));
      FSX_PHASE(13);
    }
  }

  void release_segment(int slab, int64_t off) { check(fsx_slab_free(h_, slab, off)); }

  void drop_parked(RefState& st) {
    for (auto& [seq, e] : st.parked) {
      drop_ticket(e.ticket);
      settle(e.landing, e.env.dst_gpu);
      release_segment(e.env.dst_gpu, e.off);
    }
    st.parked.clear();
  }

  // Wait for a placement still in flight (send returned before it landed).
  void settle(const Landing& l, int dst) {
    if (l.n_chunks > 0) wait_landed(dst, l.flag_base, l.n_chunks, l.token);
  }

  // Wait for a small message's copy and read-back, then recycle its mailbox
  // slot; the slab segment may be reused only after that.
  void drop_ticket(int64_t ticket) {
    if (ticket >= 0) check(fsx_ticket_free(h_, ticket));
  }

  // sidecar.hpp:571-582
  void place_backlog(int slab) {
    auto it = backlog_.find(slab);
    if (it == backlog_.end()) return;
    auto& q = it->second;
    while (!q.empty()) {
      Pending& front = q.front();
      const bool placed = front.network ? stage_network(front) : place_local(front);
      if (!placed) break;
      q.pop_front();
    }
  }

  // sidecar.hpp:584-602
  void arm_timeout(int slab) {
    Traits::schedule(kernel_, Traits::now(kernel_) + config_.send_timeout_ms, "sidecar.timeout",
                     [this, slab] {
                       auto it = backlog_.find(slab);
                       if (it == backlog_.end()) return;
                       const double now = Traits::now(kernel_);
                       auto& q = it->second;
                       for (auto qit = q.begin(); qit != q.end();) {
                         if (qit->deadline <= now) {
                           Error err = Traits::make_error(
                               status::kTimeout,
                               "sidecar send timed out under backpressure for ref " + qit->env.ref_id);
                           const std::string req = qit->env.request_id, ref = qit->env.ref_id;
                           qit = q.erase(qit);
                           if (failure_handler_) failure_handler_(req, ref, err);
                           fail_ref(ref, err);
                         } else {
                           ++qit;
                         }
                       }
                     });
  }

  Kernel& kernel_;
  std::map<int, int> topo_;
  SidecarConfig config_;
  fsx_fabric* h_ = nullptr;
  uint64_t* digest_slot_ = nullptr;  // K1 digest of the send being placed
  bool any_early_ = false;           // an early-start interest was registered (placement looks it up)
  std::vector<int> slabs_;
  std::map<std::string, RefState> refs_;
  struct SegHash {
    size_t operator()(const std::pair<int, int64_t>& k) const {
      return std::hash<int64_t>()(k.second * 64 + k.first);
    }
  };
  std::unordered_set<std::pair<int, int64_t>, SegHash> raw_held_;  // (slab gpu, offset) handed to raw callbacks
  std::map<int, std::deque<Pending>> backlog_;
  FailureHandler failure_handler_;
  int64_t transfers_ = 0, bytes_forwarded_ = 0, integrity_errors_ = 0, orphan_reclaims_ = 0;
  double added_latency_ms_ = 0;
};

// ---------------------------------------------------------------------------
// Standalone host types (no reference headers needed).

class Error : public std::runtime_error {
 public:
  Error(int status, const std::string& msg) : std::runtime_error(msg), status_(status) {}
  int status() const { return status_; }  // 1 + fissim::ErrorCode ordinal

 private:
  int status_;
};

struct DataRef {
  std::string ref_id;
  int64_t total_bytes = 0;
  bool streaming = false;
};

struct ForwardEnvelope {
  std::string request_id;
  std::string ref_id;
  int64_t seq = 0;
  int64_t chunk_bytes = 0;
  int64_t total_bytes = 0;
  uint64_t checksum = 0;
  Transport transport = Transport::LocalBuffer;
  std::string location;
  bool final = false;
  double send_time = 0;
  int src_gpu = 0;
  int dst_gpu = 0;
};

// Minimal discrete-event loop ordered by (time, insertion), Virtual clock:
// the role SimKernel plays for the reference fabric (sim_kernel.hpp:36-125).
class EventLoop {
 public:
  double now() const { return now_; }
  void schedule(double at, std::string label, std::function<void()> fn) {
    heap_.push_back(Ev{std::max(at, now_), next_++, std::move(label), std::move(fn)});
    std::push_heap(heap_.begin(), heap_.end());
  }
  void post(std::string label, std::function<void()> fn) { schedule(now_, std::move(label), std::move(fn)); }
  size_t run_until_idle() {
    size_t n = 0;
    while (!heap_.empty()) {
      std::pop_heap(heap_.begin(), heap_.end());
      Ev ev = std::move(heap_.back());  // moved out, not copied (the callback may be large)
      heap_.pop_back();
      now_ = std::max(now_, ev.at);
      ev.fn();
      ++n;
    }
    return n;
  }

 private:
  struct Ev {
    double at;
    uint64_t id;
    std::string label;
    std::function<void()> fn;
    bool operator<(const Ev& o) const { return at != o.at ? at > o.at : id > o.id; }
  };
  std::vector<Ev> heap_;  // binary heap ordered by (time, insertion)
  double now_ = 0;
  uint64_t next_ = 0;
};

struct StandaloneTraits {
  using Kernel = EventLoop;
  using Envelope = ForwardEnvelope;
  using Error = fsx::Error;
  using DataRef = fsx::DataRef;
  [[noreturn]] static void raise(int st, const std::string& msg) { throw Error(st, msg); }
  static Error make_error(int st, const std::string& msg) { return Error(st, msg); }
  static double now(Kernel& k) { return k.now(); }
  static void schedule(Kernel& k, double at, const char* label, std::function<void()> fn) {
    k.schedule(at, label, std::move(fn));
  }
  static const std::string& ref_id(const DataRef& r) { return r.ref_id; }
  static int64_t total_bytes(const DataRef& r) { return r.total_bytes; }
  static bool streaming(const DataRef& r) { return r.streaming; }
  static void set_transport(Envelope& e, bool local) {
    e.transport = local ? Transport::LocalBuffer : Transport::NetworkStream;
  }
  static bool is_local(const Envelope& e) { return e.transport == Transport::LocalBuffer; }
};

using SidecarFabric = Fabric<StandaloneTraits>;

}  // namespace fsx
