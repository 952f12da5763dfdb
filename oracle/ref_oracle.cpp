// ref_oracle.cpp -- C-ABI shim over the UNMODIFIED reference headers.
// TEST INFRASTRUCTURE ONLY: built by oracle/Makefile from
// $(FISSIM_REF_INCLUDE)/fissim/*.hpp (default /root/reference/proj/include)
// into oracle/_ref/libref_oracle.so.  No reference source is copied: the
// headers are only #included.  Used to
//   * pin the C restatement (oracle/fsx_oracle.c) and generate tests/golden/,
//   * time the reference CPU forwarding path (bench.py --impl reference and
//     the cpu_baseline leg), which is SidecarFabric::send_payload ->
//     SimKernel::run_until_idle (sidecar.hpp:302-347, 465-563) on 1 core.
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "fissim/executor_sim.hpp"
#include "fissim/profiles.hpp"
#include "fissim/record_replay.hpp"
#include "fissim/sidecar.hpp"
#include "fissim/task_dispatcher.hpp"
#include "fissim/task_model.hpp"
#include "fissim/workload.hpp"

extern "C" {
#include "fsx_oracle.h"
}

using namespace fissim;

namespace {

// ExecutorBase::payload_seed is protected (executor_sim.hpp:231-233); expose
// the reference's own implementation through a do-nothing subclass.
struct SeedProbe : ExecutorBase {
  SeedProbe() : ExecutorBase(ExecutorEnv{}, ReplicaSpec{}) {}
  void on_invocation(InvocationMessage) override {}
  uint64_t seed(const std::string& ref, int64_t seq) const { return payload_seed(ref, seq); }
};

std::map<int, int> topo_8x2() {
  std::map<int, int> t;
  for (int g = 0; g < 8; ++g) t[g] = g < 4 ? 0 : 1;  // tests/test_sidecar.cpp:15-20
  return t;
}

thread_local std::string g_err;

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_checksum64(const uint8_t* p, size_t n) { return checksum64(p, n); }
void ref_synth_payload_into(uint64_t seed, uint8_t* out, size_t n) {
  if (n) synth_payload_into(seed, out, n);
}
uint64_t ref_fnv1a64(const char* s, size_t n) { return fnv1a64(std::string_view(s, n)); }
uint64_t ref_splitmix64(uint64_t* st) { return splitmix64(*st); }
uint64_t ref_payload_seed(const char* s, size_t n, int64_t seq) {
  static SeedProbe probe;
  return probe.seed(std::string(s, n), seq);
}

// ShapeRules::item_tokens / embed_desc (profiles.hpp:256-283) on JSON inputs.
int64_t ref_item_tokens(const char* rules_json, const char* item_json) {
  try {
    ShapeRules r = ShapeRules::from_json(json::parse(rules_json));
    return r.item_tokens(json::parse(item_json));
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
int64_t ref_embed_bytes(const char* rules_json, const char* item_json) {
  try {
    ShapeRules r = ShapeRules::from_json(json::parse(rules_json));
    return r.embed_desc(json::parse(item_json)).total_bytes();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// NodeArena (sidecar.hpp:106-205), the reference allocator itself.
void* ref_arena_new(int64_t cap) {
  try {
    return new NodeArena(0, cap);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void ref_arena_delete(void* a) { delete static_cast<NodeArena*>(a); }
int64_t ref_arena_alloc(void* a, int64_t len) {
  auto off = static_cast<NodeArena*>(a)->alloc(len);
  return off ? *off : -1;
}
int ref_arena_free(void* a, int64_t off) {
  try {
    static_cast<NodeArena*>(a)->free_seg(off);
    return 0;
  } catch (const Error&) {
    return -2;
  }
}
int64_t ref_arena_segments_in_use(void* a) {
  return (int64_t) static_cast<NodeArena*>(a)->segments_in_use();
}
int64_t ref_arena_bytes_in_use(void* a) { return static_cast<NodeArena*>(a)->bytes_in_use(); }

// One single-shot transfer through the reference SidecarFabric on the 8-GPU
// two-node topology; the delivered bytes (the vector handed to the
// ChunkCallback, sidecar.hpp:543-561) are copied to `out`.
// stats_out[7] = {transfers, bytes_forwarded, integrity_errors, orphan_reclaims,
//                 segments_in_use, bytes_in_use, delivered_chunks}.
int ref_forward(int src_gpu, int dst_gpu, const char* ref_id, const uint8_t* payload, size_t n,
                uint8_t* out, int64_t* stats_out) {
  try {
    SimKernel k(ClockMode::Virtual);
    SidecarConfig cfg;
    cfg.arena_bytes = std::max<int64_t>(int64_t{64} << 20, 2 * static_cast<int64_t>(n) + 4096);
    SidecarFabric fabric(k, topo_8x2(), cfg);
    DataRef ref;
    ref.ref_id = ref_id;
    ref.producer = "p";
    ref.desc = {{static_cast<int64_t>(n)}, 1};
    int64_t chunks = 0;
    fabric.register_interest(dst_gpu, ref.ref_id,
                             [&](const ForwardEnvelope&, std::vector<uint8_t> bytes) {
                               if (bytes.size() == n && n) std::memcpy(out, bytes.data(), n);
                               ++chunks;
                             });
    k.post("send", [&] {
      fabric.send_payload("req", ref, src_gpu, dst_gpu, std::span<const uint8_t>(payload, n));
    });
    k.run_until_idle();
    auto s = fabric.stats();
    int64_t v[7] = {s.transfers,          s.bytes_forwarded,   s.integrity_errors,
                    s.orphan_reclaims,    (int64_t)s.segments_in_use, s.bytes_in_use, chunks};
    std::memcpy(stats_out, v, sizeof(v));
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1 + static_cast<int>(ErrorCode::Internal);
  }
}

// Reference CPU forwarding throughput: `iters` single-shot sends of `bytes`
// from gpu 0 to `dst_gpu` (1 = LocalBuffer, 4 = NetworkStream), each drained
// with run_until_idle (Virtual clock: modeled latency costs no wall time).
// Returns wall seconds for the timed iterations (2 warm-ups excluded).
double ref_forward_bench(size_t bytes, int iters, int dst_gpu) {
  SimKernel k(ClockMode::Virtual);
  SidecarConfig cfg;
  cfg.arena_bytes = std::max<int64_t>(int64_t{64} << 20, 2 * static_cast<int64_t>(bytes) + 4096);
  SidecarFabric fabric(k, topo_8x2(), cfg);
  auto payload = synth_payload(fnv1a64("req/r0"), bytes);
  size_t sink = 0;
  auto one = [&](int i) {
    DataRef ref;
    ref.ref_id = "bench/r" + std::to_string(i);
    ref.producer = "p";
    ref.desc = {{static_cast<int64_t>(bytes)}, 1};
    fabric.register_interest(dst_gpu, ref.ref_id,
                             [&](const ForwardEnvelope&, std::vector<uint8_t> b) { sink += b.size(); });
    k.post("send", [&, ref] { fabric.send_payload("bench", ref, 0, dst_gpu, payload); });
    k.run_until_idle();
  };
  for (int i = 0; i < 2; ++i) one(-1 - i);
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < iters; ++i) one(i);
  auto t1 = std::chrono::steady_clock::now();
  if (sink == 0 && bytes) return -1;
  return std::chrono::duration<double>(t1 - t0).count();
}

// One pass of the reference data plane over a batch: every item payload is
// forwarded producer gpu -> consumer gpu through SidecarFabric (single shot,
// as executor_sim.hpp:321-336 emits it), the consumer callback keeps the
// delivered bytes, then the derived merge (or_merge, the reference has none)
// writes them into the placeholder rows.  ref_ids[i] names item i.
// Returns wall seconds of the pass, or a negative value on error.
double ref_dataplane_pass(int32_t num_requests, int32_t num_items, int64_t row_bytes,
                          int32_t placeholder_id, uint8_t* embeds, const int32_t* token_ids,
                          const int64_t* req_row_off, const int64_t* req_item_off,
                          const uint8_t* const* item_payload, const int64_t* item_rows,
                          const char* const* ref_ids, int src_gpu, int dst_gpu, int merge_threads,
                          int32_t* status) {
  try {
    auto t0 = std::chrono::steady_clock::now();
    SimKernel k(ClockMode::Virtual);
    int64_t total = 0, biggest = 0;
    for (int32_t i = 0; i < num_items; ++i) {
      total += item_rows[i] * row_bytes;
      biggest = std::max(biggest, item_rows[i] * row_bytes);
    }
    SidecarConfig cfg;  // default 1 GiB arena, grown if the batch needs more
    cfg.arena_bytes = std::max<int64_t>(cfg.arena_bytes, total + 64 * (num_items + 1));
    SidecarFabric fabric(k, topo_8x2(), cfg);
    std::vector<std::vector<uint8_t>> got(num_items);
    for (int32_t i = 0; i < num_items; ++i) {
      fabric.register_interest(dst_gpu, ref_ids[i],
                               [&got, i](const ForwardEnvelope&, std::vector<uint8_t> b) {
                                 got[i] = std::move(b);
                               });
    }
    k.post("send", [&] {
      for (int32_t i = 0; i < num_items; ++i) {
        DataRef ref;
        ref.ref_id = ref_ids[i];
        ref.producer = "encoder";
        ref.desc = {{item_rows[i], row_bytes / 2}, 2};
        std::string rid(ref.ref_id.substr(0, ref.ref_id.find('/')));
        fabric.send_payload(rid, ref, src_gpu, dst_gpu,
                            std::span<const uint8_t>(item_payload[i], item_rows[i] * row_bytes));
      }
    });
    k.run_until_idle();
    std::vector<const uint8_t*> src(num_items);
    for (int32_t i = 0; i < num_items; ++i) {
      if (static_cast<int64_t>(got[i].size()) != item_rows[i] * row_bytes) {
        g_err = "item " + std::to_string(i) + " not delivered";
        return -2;
      }
      src[i] = got[i].data();
    }
    or_merge(num_requests, row_bytes, placeholder_id, embeds, token_ids, req_row_off, req_item_off,
             src.data(), item_rows, status, merge_threads);
    auto t1 = std::chrono::steady_clock::now();
    (void)biggest;
    return std::chrono::duration<double>(t1 - t0).count();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// The same pass on all host threads the reference can use: the reference
// fabric is single-threaded by construction (sim_kernel.hpp:147-183), so the
// requests are split into `fwd_threads` contiguous groups and every thread
// runs its own SimKernel + SidecarFabric (one reference sidecar per core)
// forwarding its group, then merges its group's requests.  Returns wall
// seconds of the whole pass, or a negative value on error.
double ref_dataplane_pass_mt(int32_t num_requests, int32_t num_items, int64_t row_bytes,
                             int32_t placeholder_id, uint8_t* embeds, const int32_t* token_ids,
                             const int64_t* req_row_off, const int64_t* req_item_off,
                             const uint8_t* const* item_payload, const int64_t* item_rows,
                             const char* const* ref_ids, int src_gpu, int dst_gpu, int fwd_threads,
                             int32_t* status) {
  const int T = std::max(1, std::min<int>(fwd_threads, num_requests));
  std::vector<std::thread> pool;
  std::vector<double> err(T, 0.0);
  std::vector<std::string> msg(T);
  auto t0 = std::chrono::steady_clock::now();
  for (int t = 0; t < T; ++t) {
    pool.emplace_back([&, t] {
      const int32_t r0 = static_cast<int32_t>(int64_t{num_requests} * t / T);
      const int32_t r1 = static_cast<int32_t>(int64_t{num_requests} * (t + 1) / T);
      const int64_t i0 = req_item_off[r0], i1 = req_item_off[r1];
      try {
        SimKernel k(ClockMode::Virtual);
        int64_t total = 0;
        for (int64_t i = i0; i < i1; ++i) total += item_rows[i] * row_bytes;
        SidecarConfig cfg;
        cfg.arena_bytes = std::max<int64_t>(cfg.arena_bytes, total + 64 * (i1 - i0 + 1));
        SidecarFabric fabric(k, topo_8x2(), cfg);
        std::vector<std::vector<uint8_t>> got(static_cast<size_t>(i1 - i0));
        for (int64_t i = i0; i < i1; ++i)
          fabric.register_interest(dst_gpu, ref_ids[i], [&got, i, i0](const ForwardEnvelope&, std::vector<uint8_t> b) {
            got[static_cast<size_t>(i - i0)] = std::move(b);
          });
        k.post("send", [&] {
          for (int64_t i = i0; i < i1; ++i) {
            DataRef ref;
            ref.ref_id = ref_ids[i];
            ref.producer = "encoder";
            ref.desc = {{item_rows[i], row_bytes / 2}, 2};
            std::string rid(ref.ref_id.substr(0, ref.ref_id.find('/')));
            fabric.send_payload(rid, ref, src_gpu, dst_gpu,
                                std::span<const uint8_t>(item_payload[i], item_rows[i] * row_bytes));
          }
        });
        k.run_until_idle();
        // the merge of this group (item pointers indexed globally)
        std::vector<const uint8_t*> src(static_cast<size_t>(num_items), nullptr);
        for (int64_t i = i0; i < i1; ++i) {
          if (static_cast<int64_t>(got[i - i0].size()) != item_rows[i] * row_bytes) {
            err[t] = -2;
            msg[t] = "item " + std::to_string(i) + " not delivered";
            return;
          }
          src[i] = got[i - i0].data();
        }
        or_merge(r1 - r0, row_bytes, placeholder_id, embeds, token_ids, req_row_off + r0, req_item_off + r0,
                 src.data(), item_rows, status + r0, 1);
      } catch (const std::exception& e) {
        err[t] = -1;
        msg[t] = e.what();
      }
    });
  }
  for (auto& th : pool) th.join();
  for (int t = 0; t < T; ++t)
    if (err[t] < 0) {
      g_err = msg[t];
      return err[t];
    }
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Reference small-message streaming (config C): `streams` streaming refs (one
// per request) each receive one `row_bytes` chunk per decode step with
// seq = step, final on the last step, exactly as LlmEngineExecutor::emit_token
// sends hidden states (executor_sim.hpp:540-564).  Every step's sends are
// posted and drained with run_until_idle (Virtual clock).  Returns wall
// seconds for all steps; delivered chunks are checked for count and order.
double ref_stream_bench(int64_t row_bytes, int streams, int steps) {
  try {
    SimKernel k(ClockMode::Virtual);
    SidecarFabric fabric(k, topo_8x2());
    std::vector<int64_t> next(streams, 0);
    int64_t bad = 0;
    std::vector<DataRef> refs(streams);
    std::vector<std::vector<uint8_t>> rows(streams);
    for (int s = 0; s < streams; ++s) {
      char id[64];
      std::snprintf(id, sizeof(id), "req-%06d/r0001", s);
      refs[s].ref_id = id;
      refs[s].producer = "thinker";
      refs[s].desc = {{steps, row_bytes / 2}, 2};
      refs[s].streaming = true;
      fabric.register_interest(1, id, [&, s](const ForwardEnvelope& env, std::vector<uint8_t> b) {
        if (env.seq != next[s]++ || static_cast<int64_t>(b.size()) != row_bytes) ++bad;
      });
    }
    // payload synthesis is the producer's work, not forwarding: outside the timer
    for (int s = 0; s < streams; ++s)
      rows[s] = synth_payload(fnv1a64(refs[s].ref_id), static_cast<size_t>(row_bytes));
    auto t0 = std::chrono::steady_clock::now();
    for (int step = 0; step < steps; ++step) {
      k.post("llm.step", [&, step] {
        for (int s = 0; s < streams; ++s)
          fabric.send("req", refs[s], 0, 1, rows[s], step, step + 1 == steps);
      });
      k.run_until_idle();
    }
    auto t1 = std::chrono::steady_clock::now();
    for (int s = 0; s < streams; ++s)
      if (next[s] != steps) ++bad;
    if (bad) {
      g_err = "stream delivery out of order or incomplete";
      return -1;
    }
    return std::chrono::duration<double>(t1 - t0).count();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// ---------------------------------------------------------------------------
// Merge inputs and placement, from the reference's own record / dispatch.
//
// The merge's slot order and row counts, and the config-D producer->consumer
// placement, are derived from record() (record_replay.hpp:510-528) with the
// built-in composite bodies invoke_mllm / invoke_omni (:404-454) and from
// TaskDispatcher::dispatch (task_dispatcher.hpp:178-266).  These shims run
// that code unmodified so tests can pin the repo's layout (trace.layout) and
// fan-out plan (fanout.plan) to it.

namespace {

CompositeTaskSpec make_composite(const char* kind, const char* config_json) {
  return CompositeLibrary::instance().make(kind, json::parse(config_json));
}

// The consumer of the encoder embeddings: the "llm" child of an mllm
// composite, the "thinker" of an omni one (task_model.hpp:259-330).
std::string consumer_digest(const CompositeTaskSpec& c) {
  const char* name = c.children.count("thinker") ? "thinker" : "llm";
  return canonical_hash(std::get<UnitTaskSpec>(c.children.at(name)));
}

std::map<std::string, std::string> child_of_digest(const CompositeTaskSpec& c) {
  std::map<std::string, std::string> out;
  for (const auto& [name, child] : c.children)
    if (const auto* u = std::get_if<UnitTaskSpec>(&child)) out[canonical_hash(*u)] = name;
  return out;
}

}  // namespace

// record() of one request: {"graph": InvocationGraph::to_json(), "consumer":
// invocation id of the embedding consumer, "children": {invocation id: child
// task name}}.  The pointer stays valid until the next call on this thread.
const char* ref_record(const char* kind, const char* config_json, const char* request_json,
                       const char* rules_json, const char* request_id) {
  static thread_local std::string out;
  try {
    CompositeTaskSpec comp = make_composite(kind, config_json);
    ShapeRules shapes = ShapeRules::from_json(json::parse(rules_json));
    RecordOutcome rec = record(comp, json::parse(request_json), shapes, request_id);
    const std::string cdig = consumer_digest(comp);
    auto names = child_of_digest(comp);
    json children = json::object();
    std::string consumer;
    for (const auto& [id, inv] : rec.graph.nodes) {
      children[id] = names.at(inv.task_digest);
      if (inv.task_digest == cdig) consumer = id;
    }
    out = json{{"graph", rec.graph.to_json()}, {"consumer", consumer}, {"children", children}}.dump();
    return out.c_str();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// TaskDispatcher::dispatch over a batch of requests, all dispatched before any
// completes (the gateway dispatches each request as it arrives; executors
// complete later).  Replicas: one per GPU listed for each child task, added
// in list order (add_replica, task_dispatcher.hpp:101-103), replica ids
// "<child>/<k>".  Returns, per request in order, {"request_id", "assign":
// {invocation id: [child, replica ordinal, home gpu]}, "routes": {invocation
// id: [[output index, [dest gpus]], ...]}} with the routes read back from the
// invocation frames the dispatcher delivered (:224-266).
const char* ref_dispatch(const char* kind, const char* config_json, const char* requests_json,
                         const char* rules_json, const char* replica_gpus_json) {
  static thread_local std::string out;
  try {
    CompositeTaskSpec comp = make_composite(kind, config_json);
    ShapeRules shapes = ShapeRules::from_json(json::parse(rules_json));
    json gpus = json::parse(replica_gpus_json);  // {child: [gpu, ...]}
    auto names = child_of_digest(comp);
    SimKernel k(ClockMode::Virtual);
    std::map<int, int> topo;
    for (int g = 0; g < 8; ++g) topo[g] = 0;  // one 8-GPU box
    SidecarConfig cfg;
    cfg.arena_bytes = 1 << 20;
    SidecarFabric fabric(k, topo, cfg);
    TaskDispatcher disp(k, fabric);
    std::vector<Frame> delivered;
    std::map<std::string, std::pair<std::string, int>> replica_info;  // id -> (child, ordinal)
    for (const auto& [digest, child] : names) {
      if (!gpus.contains(child)) continue;
      int ordinal = 0;
      for (int g : gpus.at(child).get<std::vector<int>>()) {
        ReplicaEndpoint ep;
        ep.replica_id = child + "/" + std::to_string(ordinal);
        ep.task_digest = digest;
        ep.home_gpu = g;
        ep.gpus = {g};
        ep.deliver = [&delivered](const Frame& f) { delivered.push_back(f); };
        replica_info[ep.replica_id] = {child, ordinal++};
        disp.add_replica(std::move(ep));
      }
    }
    json reqs = json::parse(requests_json);  // [[request_id, request], ...]
    json result = json::array();
    std::vector<std::shared_ptr<DispatchHandle>> handles;
    for (const auto& pair : reqs) {
      std::string rid = pair.at(0).get<std::string>();
      RecordOutcome rec = record(comp, pair.at(1), shapes, rid);
      // the gateway->dispatcher hop carries the JSON graph (control_plane.hpp:772-774)
      InvocationGraph wire = InvocationGraph::from_json(rec.graph.to_json());
      handles.push_back(disp.dispatch(wire, pair.at(1)));
    }
    k.run_until_idle();  // runs the "dispatch.deliver" events: frames captured
    std::map<std::string, json> routes;
    for (const auto& f : delivered) {
      InvocationMessage m = InvocationMessage::from_frame(f);
      json r = json::array();
      for (const auto& o : m.outputs) r.push_back(json::array({o.ref.output_index, o.dest_gpus}));
      routes[m.invocation_id] = r;
    }
    for (const auto& h : handles) {
      json assign = json::object(), rts = json::object();
      for (const auto& [inv, rep] : h->record().assignments) {
        const auto& info = replica_info.at(rep);
        int home = gpus.at(info.first).at(info.second).get<int>();
        assign[inv] = json::array({info.first, info.second, home});
        rts[inv] = routes.at(inv);
      }
      result.push_back(json{{"request_id", h->request_id()}, {"assign", assign}, {"routes", rts}});
    }
    out = result.dump();
    return out.c_str();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// generate_workload (workload.hpp:196-242) on a mix file: the reference's own
// seeded sampler, returned as a JSON array of {arrival_ms, class, request}.
// The returned pointer stays valid until the next call on this thread.
const char* ref_generate_workload(const char* mix_path, double rate_per_s, double duration_s,
                                  uint64_t seed) {
  static thread_local std::string out;
  try {
    auto mix = WorkloadMix::load(mix_path);
    auto reqs = generate_workload(mix, rate_per_s, duration_s, seed);
    json arr = json::array();
    for (const auto& r : reqs)
      arr.push_back(json{{"arrival_ms", r.arrival_ms}, {"class", r.class_name}, {"request", r.request}});
    out = arr.dump();
    return out.c_str();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

}  // extern "C"
