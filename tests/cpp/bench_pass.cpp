// The data-plane pass driven from C++ (include/fsx/dataplane.hpp, no Python):
// config B (4 Qwen2.5-VL videos, 16 x 1024 x 3584 bf16 each, 7 MiB flagged
// chunks) and an A-like batch (64 requests x one 256 x 4096 bf16 image),
// intra-device forward + merge per pass, stream-ordered or as the colocated
// pass (K1 || early-start merge, DataPlanePass::run_colocated), as the tee
// (DataPlanePass::run_tee: one kernel), or direct placement
// (DataPlanePass::run_place: no slab).  Prints one JSON line
// per batch: device time per pass, host time per pass, payload GB/s; then
// checks the merged prompt embeddings byte for byte against the oracle
// restatement (test infrastructure: inputs built and checked with
// oracle/fsx_oracle.c, never measured).
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "fsx/dataplane.hpp"

extern "C" {
#include "fsx_oracle.h"
}

namespace {

constexpr int32_t kPlaceholder = 151655;
constexpr int32_t kTextVocab = 151643;

void cuda(cudaError_t e) {
  if (e != cudaSuccess) {
    std::fprintf(stderr, "cuda: %s\n", cudaGetErrorString(e));
    std::exit(2);
  }
}

struct Case {
  const char* name;
  int requests;
  int64_t item_rows, input_tokens, row_bytes, chunk_rows;
  bool colocated;  // K1 || early-start merge (DataPlanePass::run_colocated)
  bool graph = false;  // stream-ordered pass replayed as a CUDA graph (run_graph)
  bool place = false;  // direct placement, no slab (run_place)
  bool tee = false;    // forward + merge as one kernel (run_tee)
};

int run_case(fsx_fabric* f, const Case& c, int passes) {
  cudaStream_t st, mst;
  int lo = 0, hi = 0;
  cuda(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cuda(cudaStreamCreateWithPriority(&mst, cudaStreamNonBlocking, hi));
  cudaEvent_t join;
  cuda(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
  const int64_t item_bytes = c.item_rows * c.row_bytes;
  uint8_t* src = nullptr;
  cuda(cudaMalloc(&src, item_bytes * c.requests));
  std::vector<fsx::DataPlanePass::Request> reqs(c.requests);
  std::vector<std::string> rids(c.requests), refs(c.requests);
  for (int r = 0; r < c.requests; ++r) {
    char buf[32];
    std::snprintf(buf, sizeof(buf), "req-%06d", r);
    rids[r] = buf;
    refs[r] = rids[r] + "/r0000";
    const uint64_t seed = or_payload_seed(refs[r].data(), refs[r].size(), 0);
    if (fsx_synth_payload(f, 0, seed, src + r * item_bytes, item_bytes, st) != FSX_OK) return 2;
    reqs[r].token_ids.resize(c.input_tokens + c.item_rows);
    or_prompt_tokens(rids[r].data(), rids[r].size(), c.input_tokens, 1, &c.item_rows, kPlaceholder, kTextVocab,
                     reqs[r].token_ids.data());
    reqs[r].items.push_back({src + r * item_bytes, c.item_rows});
  }
  fsx::DataPlanePass pass(f, 0, 1, c.row_bytes, kPlaceholder, c.chunk_rows, reqs);
  if (c.graph) pass.capture(st);
  auto one = [&]() -> bool {
    if (c.graph) return pass.run_graph(st);
    if (c.place) return pass.run_place(st);
    if (c.tee) return pass.run_tee(st);
    return c.colocated ? pass.run_colocated(st, mst) : pass.run(st);
  };
  // prompt rows pre-filled like the Python batch (synth_payload(fnv1a64(id + "/text")))
  for (int r = 0, row = 0; r < c.requests; ++r) {
    const std::string key = rids[r] + "/text";
    const int64_t rows = c.input_tokens + c.item_rows;
    if (fsx_synth_payload(f, 1, or_fnv1a64(key.data(), key.size()), pass.embeds() + row * c.row_bytes,
                          rows * c.row_bytes, st) != FSX_OK)
      return 2;
    row += static_cast<int>(rows);
  }
  cuda(cudaStreamSynchronize(st));
  for (int i = 0; i < 5; ++i) one();
  cuda(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double host_s = 0;
  cudaEventRecord(e0, st);
  for (int i = 0; i < passes; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    if (!one()) return 3;
    host_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  cuda(cudaEventRecord(join, mst));  // the last merge (colocated) ends the timed region
  cuda(cudaStreamWaitEvent(st, join, 0));
  cudaEventRecord(e1, st);
  cuda(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double per = ms / passes;
  // check: the oracle merge of the same inputs, byte for byte
  std::vector<uint8_t> got(pass.total_rows() * c.row_bytes), want(got.size());
  cuda(cudaMemcpy(got.data(), pass.embeds(), got.size(), cudaMemcpyDeviceToHost));
  std::vector<int32_t> tok;
  std::vector<int64_t> req_row_off{0}, req_item_off{0}, item_rows;
  std::vector<std::vector<uint8_t>> items(c.requests);
  std::vector<const uint8_t*> item_src;
  for (int r = 0, row = 0; r < c.requests; ++r) {
    const std::string key = rids[r] + "/text";
    const int64_t rows = c.input_tokens + c.item_rows;
    or_synth_payload_into(or_fnv1a64(key.data(), key.size()), want.data() + row * c.row_bytes,
                          rows * c.row_bytes);
    row += static_cast<int>(rows);
    tok.insert(tok.end(), reqs[r].token_ids.begin(), reqs[r].token_ids.end());
    req_row_off.push_back(req_row_off.back() + rows);
    req_item_off.push_back(r + 1);
    items[r].resize(item_bytes);
    or_synth_payload_into(or_payload_seed(refs[r].data(), refs[r].size(), 0), items[r].data(), item_bytes);
    item_src.push_back(items[r].data());
    item_rows.push_back(c.item_rows);
  }
  std::vector<int32_t> st_host(c.requests);
  or_merge(c.requests, c.row_bytes, kPlaceholder, want.data(), tok.data(), req_row_off.data(),
           req_item_off.data(), item_src.data(), item_rows.data(), st_host.data(), 8);
  std::vector<int32_t> dev_status(c.requests);
  cuda(cudaMemcpy(dev_status.data(), pass.status(), c.requests * sizeof(int32_t), cudaMemcpyDeviceToHost));
  bool ok = got == want;
  for (int r = 0; r < c.requests; ++r) ok = ok && dev_status[r] == 0 && st_host[r] == 0;
  std::printf("{\"batch\": \"%s\", \"requests\": %d, \"payload_bytes\": %lld, \"passes\": %d, "
              "\"device_ms_per_pass\": %.4f, \"host_us_per_pass\": %.1f, \"payload_gbs\": %.1f, "
              "\"bit_exact_vs_oracle\": %s}\n",
              c.name, c.requests, (long long)pass.payload_bytes(), passes, per, host_s / passes * 1e6,
              pass.payload_bytes() / (per * 1e-3) / 1e9, ok ? "true" : "false");
  cuda(cudaDeviceSynchronize());
  cudaFree(src);
  cudaStreamDestroy(st);
  cudaStreamDestroy(mst);
  return ok ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
  const int passes = argc > 1 ? std::atoi(argv[1]) : 50;
  int gpus[2] = {0, 1}, nodes[2] = {0, 0}, devs[2] = {0, 0};
  fsx_fabric* f = nullptr;
  if (fsx_open(2, gpus, nodes, devs, &f) != FSX_OK) {
    std::fprintf(stderr, "fsx_open: %s\n", fsx_last_error());
    return 2;
  }
  if (fsx_slab_register(f, 1, int64_t{1} << 30) != FSX_OK) return 2;
  int rc = 0;
  rc |= run_case(f, Case{"B, tee (fsx_forward_merge: forward + merge in one kernel)", 4, 16384, 1800, 7168,
                          1024, false, false, false, true},
                 passes);
  rc |= run_case(f, Case{"A-like, tee", 64, 256, 500, 8192, 0, false, false, false, true}, passes);
  rc |= run_case(f, Case{"B: Qwen2.5-VL video, 7 MiB chunks", 4, 16384, 1800, 7168, 1024, false}, passes);
  rc |= run_case(f, Case{"B, colocated pass", 4, 16384, 1800, 7168, 1024, true}, passes);
  rc |= run_case(f, Case{"A-like: 64 x one 256-row 4096-d image", 64, 256, 500, 8192, 0, false}, passes);
  rc |= run_case(f, Case{"A-like, colocated pass", 64, 256, 500, 8192, 64, true}, passes);
  rc |= run_case(f, Case{"A-like, stream-ordered pass as a CUDA graph", 64, 256, 500, 8192, 0, false, true},
                 passes);
  rc |= run_case(f, Case{"B, stream-ordered pass as a CUDA graph", 4, 16384, 1800, 7168, 1024, false, true},
                 passes);
  rc |= run_case(f, Case{"B, direct placement (forward fused with the merge, no slab)", 4, 16384, 1800, 7168,
                          1024, false, false, true},
                 passes);
  rc |= run_case(f, Case{"A-like, direct placement", 64, 256, 500, 8192, 0, false, false, true}, passes);
  fsx_close(f);
  return rc;
}
