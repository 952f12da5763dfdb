// Drop-in replacement for the reference's fissim/executor_worker.hpp
// (/root/reference/proj/include/fissim/executor_worker.hpp), the multi-process
// executor boundary, on B200 device memory.
//
// The reference parent keeps every intermediate tensor in a host shm arena:
// the handshake carries the arena's shm name (executor_worker.hpp:63-87), the
// worker mmaps it (MappedArena :210-227) and memcpys each delivered segment
// out (notify-then-read, :264-282), and a worker's own send() copies its
// payload into a TCP frame that the parent copies again into the arena
// (:245-256, :138-149).  Here:
//   * the handshake carries a CUDA IPC handle of each receive slab the worker
//     may read (one per GPU of the replica), and the worker maps them
//     (fsx_slab_import); a notification names (gpu, offset) and the worker
//     reads the segment out of device memory, acks, and verifies the dg64
//     digest the parent's K1 fused into the copy;
//   * a worker's send() stages the payload once in its own device outbox slab
//     (exported to the parent right after the spawn) and ships only the
//     envelope fields; the parent maps the outbox (fsx_ipc_open) and calls
//     SidecarFabric::send with that device span, so K1 pushes the bytes from
//     the worker's memory straight into the consumer slab (NVLink when the
//     GPUs differ), then hands the outbox segment back.  When the outbox is
//     full the payload travels inline in the frame as in the reference.
// The classes and entry points keep the reference names and signatures
// (MultiProcessHost, multiprocess_host_factory, worker_detail::WorkerSidecar,
// host_factory_for, run_executor_worker), so control_plane.hpp's Cluster and
// the reference's tests/test_worker.cpp build against it unchanged.
// Put include/fsx/dropin ahead of the reference include directory.
#pragma once

#include <sys/wait.h>
#include <unistd.h>

#include <atomic>
#include <cstdlib>
#include <mutex>
#include <set>
#include <thread>

#include "fissim/control_plane.hpp"
#include "fsx.h"
#include "fsx/envelope_codec.hpp"

namespace fissim {

namespace fsx_worker {

inline std::string to_hex(const uint8_t* p, size_t n) {
  static const char* kDigits = "0123456789abcdef";
  std::string s(2 * n, '0');
  for (size_t i = 0; i < n; ++i) {
    s[2 * i] = kDigits[p[i] >> 4];
    s[2 * i + 1] = kDigits[p[i] & 15];
  }
  return s;
}

inline void from_hex(const std::string& s, uint8_t* out, size_t n) {
  if (s.size() != 2 * n) fail(ErrorCode::Protocol, "bad IPC handle length in worker handshake");
  auto nib = [](char c) -> int {
    if (c >= '0' && c <= '9') return c - '0';
    if (c >= 'a' && c <= 'f') return c - 'a' + 10;
    fail(ErrorCode::Protocol, "bad IPC handle digit in worker handshake");
  };
  for (size_t i = 0; i < n; ++i) out[i] = static_cast<uint8_t>(nib(s[2 * i]) << 4 | nib(s[2 * i + 1]));
}

inline void check(int rc) {
  if (rc != FSX_OK) throw Error(static_cast<ErrorCode>(rc - 1), fsx_last_error());
}

// ReplicaSpec over the wire (both ends are this header, so the layout is ours;
// the fields are the reference's, executor_sim.hpp:105-117).
inline json spec_to_json(const ReplicaSpec& spec) {
  json stages = json::object();
  for (const auto& [name, prof] : spec.stage_profiles) stages[name] = prof.to_json();
  json j;
  j["replica_id"] = spec.replica_id;
  j["task_digest"] = spec.task_digest;
  j["unit"] = spec.unit.to_json();
  j["profile_name"] = spec.profile.name;
  j["profile"] = spec.profile.to_json();
  j["stage_profiles"] = std::move(stages);
  j["shapes"] = spec.shapes.to_json();
  j["gpus"] = spec.gpus;
  j["tp"] = spec.tp;
  j["activation_budget_per_gpu"] = spec.activation_budget_per_gpu;
  return j;
}

inline ReplicaSpec spec_from_json(const json& j) {
  ReplicaSpec spec;
  spec.replica_id = j.at("replica_id").get<std::string>();
  spec.task_digest = j.at("task_digest").get<std::string>();
  spec.unit = UnitTaskSpec::from_json(j.at("unit"));
  spec.profile = ComponentProfile::from_json(j.value("profile_name", std::string("worker")), j.at("profile"));
  for (const auto& [name, prof] : j.value("stage_profiles", json::object()).items())
    spec.stage_profiles[name] = ComponentProfile::from_json(name, prof);
  spec.shapes = ShapeRules::from_json(j.at("shapes"));
  spec.gpus = j.at("gpus").get<std::vector<int>>();
  spec.tp = j.value("tp", 1);
  spec.activation_budget_per_gpu = j.value("activation_budget_per_gpu", int64_t{1} << 62);
  return spec;
}

// Worker outbox size: FSX_WORKER_OUTBOX_BYTES, default 256 MiB of device memory.
inline int64_t outbox_bytes() {
  const char* e = std::getenv("FSX_WORKER_OUTBOX_BYTES");
  const int64_t v = e ? std::atoll(e) : (int64_t{256} << 20);
  return v > 0 ? v : (int64_t{256} << 20);
}

// Parent-process counters over every MultiProcessHost (tests, metrics).
struct HostCounters {
  std::atomic<int64_t> outbox_sends{0};  // worker payloads K1-pushed from its device outbox
  std::atomic<int64_t> outbox_bytes{0};
  std::atomic<int64_t> inline_sends{0};  // worker payloads that came inside the frame
};
inline HostCounters& host_counters() {
  static HostCounters c;
  return c;
}

}  // namespace fsx_worker

// -----------------------------------------------------------------------------
// Parent side (executor_worker.hpp:55-196)

class MultiProcessHost : public ExecutorHost {
 public:
  MultiProcessHost(const ExecutorEnv& env, const ReplicaSpec& spec, const std::string& worker_exe)
      : env_(env), spec_(spec) {
    fabric_ = dynamic_cast<SidecarFabric*>(env_.sidecar);
    if (!fabric_) fail(ErrorCode::Config, "multi-process executors require the in-process fabric");
    TcpListener listener(0);
    spawn_child(worker_exe, listener.bound_port());
    sock_ = listener.accept();

    // Handshake: the replica spec, its GPUs' nodes and an IPC handle of every
    // receive slab the worker reads notifications from.
    json topology = json::object();
    json slabs = json::object();
    for (int g : spec_.gpus) {
      topology[std::to_string(g)] = fabric_->node_of(g);
      uint8_t h[64];
      const int64_t cap = fabric_->export_slab(g, h);
      slabs[std::to_string(g)] = json{{"ipc", fsx_worker::to_hex(h, sizeof(h))}, {"capacity", cap}};
    }
    send_frame(Frame{json{{"type", "spawn"},
                          {"spec", fsx_worker::spec_to_json(spec_)},
                          {"topology", topology},
                          {"slabs", slabs}},
                     {}});
    reader_ = std::make_unique<FrameReader>(
        sock_, [this](Frame f) { on_child_frame(std::move(f)); }, [this] { child_gone_ = true; });
  }

  ~MultiProcessHost() override {
    // Unmap the worker's outbox before the worker frees it.
    if (outbox_) fsx_ipc_close(fabric_->native_handle(), outbox_);
    try {
      std::lock_guard lk(send_m_);
      if (sock_.valid()) sock_.send_frame(Frame{json{{"type", "shutdown"}}, {}});
    } catch (...) {
    }
    sock_.shutdown_both();
    if (reader_) reader_->join();
    sock_.close_fd();
    if (child_pid_ > 0) {
      int status = 0;
      ::waitpid(child_pid_, &status, 0);
    }
  }

  void deliver(const Frame& f) override { send_frame(f); }

 private:
  void send_frame(const Frame& f) {
    std::lock_guard lk(send_m_);
    if (sock_.valid() && !child_gone_) sock_.send_frame(f);
  }

  void spawn_child(const std::string& worker_exe, int port) {
    child_pid_ = ::fork();
    if (child_pid_ < 0) fail(ErrorCode::Internal, "fork failed");
    if (child_pid_ == 0) {
      const std::string port_s = std::to_string(port);
      ::execl(worker_exe.c_str(), worker_exe.c_str(), "executor-worker", "--host", "127.0.0.1", "--port",
              port_s.c_str(), static_cast<char*>(nullptr));
      ::_exit(127);
    }
  }

  // Reader thread: everything that touches the fabric is posted to the kernel
  // thread (sidecar.hpp:299-301).
  void on_child_frame(Frame f) {
    const std::string type = f.header.value("type", "");
    if (type == "status" || type == "chunk") {
      env_.kernel->post("worker.result", [this, f = std::move(f)] { env_.to_dispatcher(f); });
    } else if (type == "worker_outbox") {
      env_.kernel->post("worker.outbox", [this, f = std::move(f)] { map_outbox(f.header); });
    } else if (type == "sidecar_send") {
      env_.kernel->post("worker.sidecar_send", [this, f = std::move(f)] { on_send(f); });
    } else if (type == "sidecar_interest") {
      const std::string ref_id = f.header.value("ref_id", "");
      const int gpu = f.header.value("gpu", 0);
      env_.kernel->post("worker.interest", [this, ref_id, gpu] { on_interest(ref_id, gpu); });
    } else if (type == "sidecar_ack") {
      const int gpu = f.header.value("gpu", 0);
      const int64_t offset = f.header.value("offset", int64_t{0});
      env_.kernel->post("worker.ack", [this, gpu, offset] { fabric_->ack_raw(gpu, offset); });
    } else if (type == "sidecar_fail") {
      const std::string ref_id = f.header.value("ref_id", "");
      const std::string msg = f.header.value("message", "worker failure");
      env_.kernel->post("worker.fail",
                        [this, ref_id, msg] { fabric_->fail_ref(ref_id, Error(ErrorCode::Internal, msg)); });
    }
  }

  void map_outbox(const json& h) {
    uint8_t raw[64];
    fsx_worker::from_hex(h.at("ipc").get<std::string>(), raw, sizeof(raw));
    outbox_gpu_ = h.value("gpu", spec_.home_gpu());
    fsx_worker::check(fsx_ipc_open(fabric_->native_handle(), outbox_gpu_, raw, &outbox_));
    outbox_capacity_ = h.at("capacity").get<int64_t>();
  }

  // A worker send: the payload is either in the worker's outbox (device) or
  // inline in the frame (outbox full).  K1 moves outbox bytes device to
  // device; fabric_->send returns once they are placed (or owned by the
  // backlog), after which the outbox segment goes back to the worker.
  void on_send(const Frame& f) {
    const DataRef ref = DataRef::from_json(f.header.at("ref"));
    const std::string request_id = f.header.value("request_id", "");
    const int src = f.header.value("src_gpu", 0), dst = f.header.value("dst_gpu", 0);
    const int64_t seq = f.header.value("seq", int64_t{0});
    const bool fin = f.header.value("final", false);
    const int64_t off = f.header.value("outbox_off", int64_t{-1});
    if (off < 0) {
      ++fsx_worker::host_counters().inline_sends;
      fabric_->send(request_id, ref, src, dst, std::span<const uint8_t>(f.payload.data(), f.payload.size()),
                    seq, fin);
      return;
    }
    const int64_t n = f.header.value("bytes", int64_t{0});
    struct Release {
      MultiProcessHost* h;
      int64_t off;
      // runs during unwinding too (a failed send): never let the socket
      // error escape the destructor (std::terminate); a worker that is gone
      // no longer needs its outbox range back
      ~Release() {
        try {
          h->send_frame(Frame{json{{"type", "outbox_free"}, {"offset", off}}, {}});
        } catch (...) {
        }
      }
    } release{this, off};
    if (!outbox_ || off + n > outbox_capacity_)
      fail(ErrorCode::Protocol, "worker send names an unmapped outbox range");
    ++fsx_worker::host_counters().outbox_sends;
    fsx_worker::host_counters().outbox_bytes += n;
    const uint8_t* p = static_cast<const uint8_t*>(outbox_) + off;
    fabric_->send(request_id, ref, src, dst, std::span<const uint8_t>(p, static_cast<size_t>(n)), seq, fin);
  }

  void on_interest(const std::string& ref_id, int gpu) {
    fabric_->register_interest_raw(
        gpu, ref_id,
        [this](const ForwardEnvelope& env, int64_t offset) {
          // notify-then-read: the worker reads (gpu, offset) of the mapped
          // slab; the envelope travels in its binary form (envelope_codec.hpp)
          // followed by the slab offset
          std::vector<uint8_t> body;
          if (!fsx::encode_envelope(env, body)) {
            send_frame(Frame{json{{"type", "sidecar_envelope"},
                                  {"envelope", env.to_json()},
                                  {"offset", offset},
                                  {"gpu", env.dst_gpu}},
                             {}});
            return;
          }
          fsx::codec_detail::put<int64_t>(body, offset);
          send_frame(Frame{json{{"type", "sidecar_envelope_bin"}}, std::move(body)});
        },
        [this, ref_id](const Error& e) {
          send_frame(Frame{json{{"type", "sidecar_error"},
                                {"ref_id", ref_id},
                                {"code", to_string(e.code())},
                                {"message", e.what()}},
                           {}});
        });
  }

  ExecutorEnv env_;
  ReplicaSpec spec_;
  SidecarFabric* fabric_ = nullptr;
  pid_t child_pid_ = -1;
  TcpSocket sock_;
  std::mutex send_m_;
  std::unique_ptr<FrameReader> reader_;
  std::atomic<bool> child_gone_{false};
  void* outbox_ = nullptr;
  int outbox_gpu_ = 0;
  int64_t outbox_capacity_ = 0;
};

inline ExecutorHostFactory multiprocess_host_factory(std::string worker_exe) {
  return [worker_exe](const ExecutorEnv& env, const ReplicaSpec& spec) {
    return std::unique_ptr<ExecutorHost>(new MultiProcessHost(env, spec, worker_exe));
  };
}

// -----------------------------------------------------------------------------
// Worker side (executor_worker.hpp:204-304)

namespace worker_detail {

// SidecarPort inside the worker: interests and envelopes are frames to the
// parent; delivered bytes are read from the parent's receive slabs (CUDA IPC)
// and the worker's own payloads are staged in its exported device outbox.
// Every method runs on the worker's kernel thread.
class WorkerSidecar : public SidecarPort {
 public:
  WorkerSidecar(TcpSocket& sock, std::mutex& send_m) : sock_(sock), send_m_(send_m) {}

  ~WorkerSidecar() override {
    if (in_) fsx_close(in_);
    if (out_) fsx_close(out_);
  }

  // Spawn handshake: map the parent's slabs, create and export the outbox.
  void attach(const json& topology, const json& slabs, int home_gpu) {
    std::vector<int> ids, nodes, devs;
    for (const auto& [g, n] : topology.items()) {
      ids.push_back(std::stoi(g));
      nodes.push_back(n.get<int>());
      devs.push_back(-1);
    }
    fsx_worker::check(fsx_open(static_cast<int>(ids.size()), ids.data(), nodes.data(), devs.data(), &in_));
    for (const auto& [g, info] : slabs.items()) {
      uint8_t raw[64];
      fsx_worker::from_hex(info.at("ipc").get<std::string>(), raw, sizeof(raw));
      fsx_worker::check(fsx_slab_import(in_, std::stoi(g), raw, info.at("capacity").get<int64_t>()));
    }
    // The outbox lives in a second handle: the same logical GPU id already
    // names the imported receive slab in the first.
    home_ = home_gpu;
    int node = 0;
    fsx_worker::check(fsx_open(1, &home_, &node, nullptr, &out_));
    fsx_worker::check(fsx_slab_register(out_, home_, fsx_worker::outbox_bytes()));
    uint8_t raw[64];
    int64_t cap = 0;
    fsx_worker::check(fsx_slab_export(out_, home_, raw, &cap));
    send_frame(Frame{json{{"type", "worker_outbox"},
                          {"gpu", home_},
                          {"ipc", fsx_worker::to_hex(raw, sizeof(raw))},
                          {"capacity", cap}},
                     {}});
  }

  void register_interest(int gpu, const std::string& ref_id, ChunkCallback on_chunk,
                         RefErrorCallback on_error = {}) override {
    interests_[ref_id] = Interest{std::move(on_chunk), std::move(on_error)};
    send_frame(Frame{json{{"type", "sidecar_interest"}, {"ref_id", ref_id}, {"gpu", gpu}}, {}});
  }

  void send(const std::string& request_id, const DataRef& ref, int src_gpu, int dst_gpu,
            std::span<const uint8_t> payload, int64_t seq, bool final_chunk) override {
    json h{{"type", "sidecar_send"},
           {"request_id", request_id},
           {"ref", ref.to_json()},
           {"src_gpu", src_gpu},
           {"dst_gpu", dst_gpu},
           {"seq", seq},
           {"final", final_chunk}};
    const int64_t n = static_cast<int64_t>(payload.size());
    int64_t off = -1;
    if (out_ && n > 0) fsx_worker::check(fsx_slab_alloc(out_, home_, n, &off));
    if (off >= 0) {
      // one copy into device memory (host->device, or device->device when the
      // executor's payload already lives on a GPU); the frame carries no bytes
      fsx_worker::check(fsx_slab_write(out_, home_, off, payload.data(), n, nullptr));
      h["outbox_off"] = off;
      h["bytes"] = n;
      ++outbox_sends_;
      send_frame(Frame{std::move(h), {}});
      return;
    }
    // empty payload or outbox full: inline, as the reference does
    ++inline_sends_;
    send_frame(Frame{std::move(h), std::vector<uint8_t>(payload.begin(), payload.end())});
  }

  void fail_ref(const std::string& ref_id, const Error& err) override {
    send_frame(Frame{json{{"type", "sidecar_fail"}, {"ref_id", ref_id}, {"message", err.what()}}, {}});
  }

  // Parent notification: read the segment out of device memory, release it,
  // verify, deliver (executor_worker.hpp:264-282).
  void on_envelope(const Frame& f) {
    ForwardEnvelope env;
    int gpu = 0;
    int64_t offset = 0;
    if (f.header.value("type", "") == "sidecar_envelope_bin") {
      const size_t used = fsx::decode_envelope(f.payload.data(), f.payload.size(), &env);
      if (used == 0 || f.payload.size() - used != sizeof(int64_t))
        fail(ErrorCode::Protocol, "malformed binary sidecar envelope");
      std::memcpy(&offset, f.payload.data() + used, sizeof(int64_t));
      gpu = env.dst_gpu;
    } else {
      env = ForwardEnvelope::from_json(f.header.at("envelope"));
      gpu = f.header.value("gpu", env.dst_gpu);
      offset = f.header.value("offset", int64_t{0});
    }
    if (!in_) fail(ErrorCode::Internal, "worker has no slab mappings");
    std::vector<uint8_t> bytes(static_cast<size_t>(env.chunk_bytes));
    if (env.chunk_bytes > 0)
      fsx_worker::check(fsx_slab_read(in_, gpu, offset, bytes.data(), env.chunk_bytes, nullptr));
    send_frame(Frame{json{{"type", "sidecar_ack"}, {"gpu", gpu}, {"offset", offset}}, {}});
    auto it = interests_.find(env.ref_id);
    if (it == interests_.end()) return;
    // LocalBuffer envelopes carry dg64 (fused into K1 by the parent), network
    // envelopes the reference checksum64
    const uint64_t sum = env.transport == Transport::LocalBuffer ? fsx::digest64(bytes.data(), bytes.size())
                                                                 : fsx::checksum64(bytes.data(), bytes.size());
    if (sum != env.checksum) {
      ++integrity_errors_;
      if (it->second.on_error)
        it->second.on_error(Error(ErrorCode::Integrity, "checksum mismatch on " + env.ref_id));
      return;
    }
    ++delivered_;
    it->second.on_chunk(env, std::move(bytes));
  }

  void on_outbox_free(const Frame& f) {
    if (out_) fsx_worker::check(fsx_slab_free(out_, home_, f.header.value("offset", int64_t{0})));
  }

  void on_error_frame(const Frame& f) {
    auto it = interests_.find(f.header.value("ref_id", ""));
    if (it != interests_.end() && it->second.on_error)
      it->second.on_error(Error(ErrorCode::Internal, f.header.value("message", "sidecar error")));
  }

  int64_t outbox_sends() const { return outbox_sends_; }
  int64_t inline_sends() const { return inline_sends_; }
  int64_t delivered() const { return delivered_; }
  int64_t integrity_errors() const { return integrity_errors_; }

 private:
  void send_frame(const Frame& f) {
    std::lock_guard lk(send_m_);
    sock_.send_frame(f);
  }

  struct Interest {
    ChunkCallback on_chunk;
    RefErrorCallback on_error;
  };
  TcpSocket& sock_;
  std::mutex& send_m_;
  std::map<std::string, Interest> interests_;
  fsx_fabric* in_ = nullptr;   // imported receive slabs of the parent
  fsx_fabric* out_ = nullptr;  // this worker's outbox slab
  int home_ = 0;
  int64_t outbox_sends_ = 0, inline_sends_ = 0, delivered_ = 0, integrity_errors_ = 0;
};

}  // namespace worker_detail

// In-process by default, worker processes when the config says so
// (executor_worker.hpp:308-315).
inline ExecutorHostFactory host_factory_for(const ClusterConfig& config) {
  if (config.executor_mode != ClusterConfig::ExecutorMode::MultiProcess) return {};
  std::string exe = config.worker_exe;
  if (exe.empty()) exe = "/proc/self/exe";
  return multiprocess_host_factory(exe);
}

// `executor-worker` entry point (executor_worker.hpp:317-380): blocks until
// the parent sends shutdown or the connection drops.
inline int run_executor_worker(const std::string& host, int port) {
  TcpSocket sock = tcp_connect(host, port);
  std::mutex send_m;
  SimKernel kernel(ClockMode::RealTime);
  kernel.start();
  auto sidecar = std::make_unique<worker_detail::WorkerSidecar>(sock, send_m);
  std::unique_ptr<ExecutorBase> executor;
  std::atomic<bool> done{false};

  ExecutorEnv env;
  env.kernel = &kernel;
  env.sidecar = sidecar.get();
  env.to_dispatcher = [&sock, &send_m](Frame f) {
    std::lock_guard lk(send_m);
    sock.send_frame(f);
  };

  FrameReader reader(
      sock,
      [&](Frame f) {
        const std::string type = f.header.value("type", "");
        if (type == "spawn") {
          kernel.post("worker.spawn", [&, f = std::move(f)] {
            ReplicaSpec spec = fsx_worker::spec_from_json(f.header.at("spec"));
            sidecar->attach(f.header.value("topology", json::object()), f.header.value("slabs", json::object()),
                            spec.home_gpu());
            executor = make_executor(env, spec);
          });
        } else if (type == "shutdown") {
          done = true;
          sock.shutdown_both();
        } else if (type == "sidecar_envelope" || type == "sidecar_envelope_bin") {
          kernel.post("worker.envelope", [&, f = std::move(f)] { sidecar->on_envelope(f); });
        } else if (type == "outbox_free") {
          kernel.post("worker.outbox_free", [&, f = std::move(f)] { sidecar->on_outbox_free(f); });
        } else if (type == "sidecar_error") {
          kernel.post("worker.sidecar_error", [&, f = std::move(f)] { sidecar->on_error_frame(f); });
        } else {
          // invocation / cancel frames from the dispatcher
          kernel.post("worker.frame", [&, f = std::move(f)] {
            if (executor) executor->handle_frame(f);
          });
        }
      },
      [&] { done = true; });

  while (!done) std::this_thread::sleep_for(std::chrono::milliseconds(5));
  reader.join();
  kernel.stop();
  executor.reset();
  sidecar.reset();
  return 0;
}

}  // namespace fissim
