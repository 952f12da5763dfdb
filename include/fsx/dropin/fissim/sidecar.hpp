// Drop-in replacement for the reference's fissim/sidecar.hpp
// (/root/reference/proj/include/fissim/sidecar.hpp), backed by libfsx.
//
// Put include/fsx/dropin AHEAD of the reference include directory and link
// libfsx.so:  every `#include "fissim/sidecar.hpp"` in the reference
// (executor_sim.hpp:19, control_plane.hpp, tests) then resolves here, and
// ExecutorEnv.sidecar / Cluster / the tests get a fabric whose bytes live in
// per-GPU device slabs on B200s instead of a host shm arena.  The public
// surface (types, callbacks, SidecarPort virtuals, SidecarFabric methods) keeps
// the reference names and signatures (sidecar.hpp:32-100, 209-238, 240-430);
// differences are listed in INTEGRATION.md:
//   * one receive slab per destination GPU (the reference: one arena per node),
//     so ForwardEnvelope::location reads "gpu<G>:off<K>" and ack_raw() takes
//     the slab's GPU;
//   * LocalBuffer envelopes carry the lane-parallel dg64 digest (fused into K1)
//     instead of the serial checksum64; NetworkStream envelopes keep checksum64;
//   * arena(n).shm_name() is empty (device slabs are not shm segments).
#pragma once

#include <span>
#include <string>
#include <vector>

#include "fissim/invocation_graph.hpp"
#include "fissim/net.hpp"
#include "fissim/sim_kernel.hpp"
#include "fsx/fabric.hpp"

namespace fissim {

using Transport = fsx::Transport;
inline const char* to_string(Transport t) { return fsx::transport_name(t); }

using SidecarConfig = fsx::SidecarConfig;
using SidecarStats = fsx::SidecarStats;

// Wire envelope, field names as docs/formats.md:253-287 (sidecar.hpp:59-100).
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
  TimeMs send_time = 0;
  int src_gpu = 0;
  int dst_gpu = 0;

  json to_json() const {
    json j;
    j["request_id"] = request_id;
    j["ref_id"] = ref_id;
    j["seq"] = seq;
    j["chunk_bytes"] = chunk_bytes;
    j["total_bytes"] = total_bytes;
    j["checksum"] = checksum;
    j["transport"] = to_string(transport);
    j["location"] = location;
    j["final"] = final;
    j["send_time"] = send_time;
    j["src_gpu"] = src_gpu;
    j["dst_gpu"] = dst_gpu;
    return j;
  }

  static ForwardEnvelope from_json(const json& j) {
    ForwardEnvelope e;
    e.request_id = j.at("request_id").get<std::string>();
    e.ref_id = j.at("ref_id").get<std::string>();
    e.seq = j.value("seq", int64_t{0});
    e.chunk_bytes = j.value("chunk_bytes", int64_t{0});
    e.total_bytes = j.value("total_bytes", int64_t{0});
    e.checksum = j.value("checksum", uint64_t{0});
    e.transport = j.value("transport", std::string("local_buffer")) == "network_stream"
                      ? Transport::NetworkStream
                      : Transport::LocalBuffer;
    e.location = j.value("location", std::string());
    e.final = j.value("final", false);
    e.send_time = j.value("send_time", 0.0);
    e.src_gpu = j.value("src_gpu", 0);
    e.dst_gpu = j.value("dst_gpu", 0);
    return e;
  }
};

using ChunkCallback = std::function<void(const ForwardEnvelope& env, std::vector<uint8_t> bytes)>;
using RefErrorCallback = std::function<void(const Error& err)>;
using RawChunkCallback = std::function<void(const ForwardEnvelope& env, int64_t offset)>;

// The executor-facing surface (sidecar.hpp:230-238), unchanged.
class SidecarPort {
 public:
  virtual ~SidecarPort() = default;
  virtual void register_interest(int gpu, const std::string& ref_id, ChunkCallback on_chunk,
                                 RefErrorCallback on_error = {}) = 0;
  virtual void send(const std::string& request_id, const DataRef& ref, int src_gpu, int dst_gpu,
                    std::span<const uint8_t> payload, int64_t seq, bool final_chunk) = 0;
  virtual void fail_ref(const std::string& ref_id, const Error& err) = 0;
};

namespace fsx_dropin {

struct Traits {
  using Kernel = SimKernel;
  using Envelope = ForwardEnvelope;
  using Error = fissim::Error;
  using DataRef = fissim::DataRef;
  [[noreturn]] static void raise(int status, const std::string& msg) {
    throw Error(static_cast<ErrorCode>(status - 1), msg);
  }
  static Error make_error(int status, const std::string& msg) {
    return Error(static_cast<ErrorCode>(status - 1), msg);
  }
  static double now(Kernel& k) { return k.now(); }
  static void schedule(Kernel& k, double at, const char* label, std::function<void()> fn) {
    k.schedule(at, label, std::move(fn));
  }
  static const std::string& ref_id(const DataRef& r) { return r.ref_id; }
  static int64_t total_bytes(const DataRef& r) { return r.desc.total_bytes(); }
  static bool streaming(const DataRef& r) { return r.streaming; }
  static void set_transport(Envelope& e, bool local) {
    e.transport = local ? Transport::LocalBuffer : Transport::NetworkStream;
  }
  static bool is_local(const Envelope& e) { return e.transport == Transport::LocalBuffer; }
};

}  // namespace fsx_dropin

// Stand-in for the reference NodeArena accessor (sidecar.hpp:106-205, 419):
// device slabs have no shm name; usage comes from the slab allocator.
class SlabArenaView {
 public:
  SlabArenaView(fsx_fabric* h, int gpu) : h_(h), gpu_(gpu) {}
  int node_id() const { return gpu_; }
  const std::string& shm_name() const { return empty_; }
  int64_t capacity() const { return usage(3); }
  size_t segments_in_use() const { return static_cast<size_t>(usage(0)); }
  int64_t bytes_in_use() const { return usage(1); }
  int64_t peak_bytes() const { return usage(2); }

 private:
  int64_t usage(int which) const {
    int64_t v[4] = {0, 0, 0, 0};
    if (fsx_slab_usage(h_, gpu_, &v[0], &v[1], &v[2], &v[3]) != FSX_OK) return 0;
    return v[which];
  }
  fsx_fabric* h_;
  int gpu_;
  std::string empty_;
};

class SidecarFabric : public SidecarPort {
 public:
  SidecarFabric(SimKernel& kernel, std::map<int, int> gpu_to_node, SidecarConfig config = {})
      : engine_(kernel, std::move(gpu_to_node), config) {}

  Transport route(int src_gpu, int dst_gpu) const { return engine_.route(src_gpu, dst_gpu); }
  int node_of(int gpu) const { return engine_.node_of(gpu); }

  void register_interest(int gpu, const std::string& ref_id, ChunkCallback on_chunk,
                         RefErrorCallback on_error = {}) override {
    engine_.register_interest(gpu, ref_id, std::move(on_chunk), std::move(on_error));
  }
  void register_interest_raw(int gpu, const std::string& ref_id, RawChunkCallback on_chunk,
                             RefErrorCallback on_error = {}) {
    engine_.register_interest_raw(gpu, ref_id, std::move(on_chunk), std::move(on_error));
  }
  void ack_raw(int slab_gpu, int64_t offset) { engine_.ack_raw(slab_gpu, offset); }
  void cancel_interest(const std::string& ref_id, int gpu) { engine_.cancel_interest(ref_id, gpu); }

  void send(const std::string& request_id, const DataRef& ref, int src_gpu, int dst_gpu,
            std::span<const uint8_t> payload, int64_t seq, bool final_chunk) override {
    engine_.send(request_id, ref, src_gpu, dst_gpu, payload, seq, final_chunk);
  }
  void send_payload(const std::string& request_id, const DataRef& ref, int src_gpu, int dst_gpu,
                    std::span<const uint8_t> payload) {
    engine_.send_payload(request_id, ref, src_gpu, dst_gpu, payload);
  }

  void handle_network_frame(const Frame& frame) {
    engine_.handle_network(ForwardEnvelope::from_json(frame.header.at("envelope")), frame.payload);
  }

  void fail_ref(const std::string& ref_id, const Error& err) override { engine_.fail_ref(ref_id, err); }
  void purge_request(const std::string& request_id) { engine_.purge_request(request_id); }
  SidecarStats stats() const { return engine_.stats(); }
  const SidecarConfig& config() const { return engine_.config(); }

  SlabArenaView& arena(int node) {
    auto it = views_.find(node);
    if (it == views_.end()) it = views_.emplace(node, SlabArenaView(engine_.handle(), node)).first;
    return it->second;
  }

  void set_failure_handler(std::function<void(const std::string& request_id,
                                              const std::string& ref_id, const Error&)> fn) {
    engine_.set_failure_handler(std::move(fn));
  }

  // fsx additions for the multi-process boundary (dropin executor_worker.hpp).
  int64_t export_slab(int gpu, void* handle64) { return engine_.export_slab(gpu, handle64); }
  fsx_fabric* native_handle() const { return engine_.handle(); }

  // Zero-copy view for raw consumers (fsx addition).
  void* slab_ptr(int gpu, int64_t offset) { return engine_.slab_ptr(gpu, offset); }

  static Frame envelope_frame(const ForwardEnvelope& env) {
    return Frame{json{{"type", "sidecar_envelope"}, {"envelope", env.to_json()}}, {}};
  }

 private:
  fsx::Fabric<fsx_dropin::Traits> engine_;
  std::map<int, SlabArenaView> views_;
};

}  // namespace fissim
