// fsx tests of the multi-process executor boundary on device memory
// (include/fsx/dropin/fissim/executor_worker.hpp), in the
// style of the reference's tests/test_worker.cpp but with embeddings up to
// 12.8 MB and counters that prove which path the bytes took:
//   * worker encoders stage each embedding in their device outbox and the
//     parent's K1 pushes it into the LLM's receive slab (no payload in the
//     frame), the LLM worker reads the slab segment through CUDA IPC and
//     verifies the dg64 digest K1 fused into the copy;
//   * with a 4 KiB outbox every payload falls back to the inline frame path
//     and the requests still complete;
//   * no slab segment is left held afterwards.
// Built against the reference's control plane (unmodified) + the drop-in
// headers; FSX_WORKER_BIN / FSX_REFDATA come from the Makefile.
#include <catch_amalgamated.hpp>

#include <cstdlib>
#include <fstream>

#include "fissim/executor_worker.hpp"

using namespace fissim;

namespace {

json load(const std::string& rel) {
  std::ifstream in(std::string(FSX_REFDATA) + "/" + rel);
  REQUIRE(in.good());
  json j;
  in >> j;
  return j;
}

struct Run {
  int ok = 0, failed = 0, chunks = 0;
  int64_t embed_bytes = 0;
};

Run serve_images(const std::vector<std::pair<int, int>>& images) {
  ClusterConfig config;
  config.nodes.push_back({0, 2, int64_t{80} * 1000 * 1000 * 1000});
  config.clock = ClockMode::RealTime;
  config.executor_mode = ClusterConfig::ExecutorMode::MultiProcess;
  config.worker_exe = FSX_WORKER_BIN;
  config.profile_files = {std::string(FSX_REFDATA) + "/profiles/mllm.json"};
  Cluster cluster(config, host_factory_for(config));
  cluster.start();
  auto& gw = cluster.gateway();
  gw.register_app(AppManifest::from_json(load("apps/mllm-gemma.json")));
  Run r;
  for (auto [w, h] : images) {
    json request{{"text", "describe"},
                 {"items", {{{"modality", "image"}, {"width", w}, {"height", h}}}},
                 {"gen", {{"input_tokens", 8}, {"output_tokens", 3}, {"chunks", 0}}}};
    auto live = gw.invoke("mllm-gemma", request);
    REQUIRE(live.channels.size() == 1);
    auto stream = std::get<2>(live.channels[0]);
    while (auto c = stream->pop()) ++r.chunks;
    auto trace = live.trace.get();
    if (trace.failed) ++r.failed;
    else ++r.ok;
    // mllm.json shape_rules: ceil(w*h / 1024) tokens x 1024 x 2 B
    r.embed_bytes += (int64_t{w} * h + 1023) / 1024 * 1024 * 2;
  }
  CHECK(cluster.fabric().stats().segments_in_use == 0);
  fsx_stats st{};
  REQUIRE(fsx_get_stats(cluster.fabric().native_handle(), &st) == FSX_OK);
  CHECK(st.bytes_forwarded >= r.embed_bytes);
  gw.deregister_app("mllm-gemma", true);
  cluster.stop();
  return r;
}

const std::vector<std::pair<int, int>> kImages = {
    {448, 448}, {896, 896}, {1792, 1792}, {1000, 701}, {2508, 2508}, {64, 48}};

}  // namespace

TEST_CASE("worker embeddings travel device to device: outbox -> K1 -> slab -> IPC read") {
  auto& c = fsx_worker::host_counters();
  const int64_t out0 = c.outbox_sends, inl0 = c.inline_sends, bytes0 = c.outbox_bytes;
  Run r = serve_images(kImages);
  CHECK(r.failed == 0);
  CHECK(r.ok == static_cast<int>(kImages.size()));
  CHECK(r.chunks == 3 * static_cast<int>(kImages.size()));
  CHECK(c.outbox_sends - out0 == static_cast<int64_t>(kImages.size()));
  CHECK(c.inline_sends - inl0 == 0);
  CHECK(c.outbox_bytes - bytes0 == r.embed_bytes);
}

TEST_CASE("a full worker outbox falls back to the inline frame path") {
  ::setenv("FSX_WORKER_OUTBOX_BYTES", "4096", 1);  // inherited by the workers
  auto& c = fsx_worker::host_counters();
  const int64_t out0 = c.outbox_sends, inl0 = c.inline_sends;
  Run r = serve_images({{448, 448}, {896, 896}});
  ::unsetenv("FSX_WORKER_OUTBOX_BYTES");
  CHECK(r.failed == 0);
  CHECK(r.ok == 2);
  CHECK(c.inline_sends - inl0 == 2);
  CHECK(c.outbox_sends - out0 == 0);
}
