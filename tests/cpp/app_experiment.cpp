// Whole serving experiments of the reference's own bench harness
// (bench_harness.hpp run_experiment: cluster, planner, dispatcher, executors
// and the sidecar, Virtual clock), built twice from this one file:
//   build/app_experiment_ref  against the reference's fissim/sidecar.hpp
//                             (the reference headers, unmodified), and
//   build/app_experiment_fsx  against the fsx drop-in (include/fsx/dropin).
// Per experiment it prints the report's JSON digest (the report is the
// reference's own: throughput, latency percentiles, completions, failures --
// identical digests mean the drop-in changed nothing the application sees),
// the sidecar's transfer and byte counts, and the wall time of the run.
//   build/app_experiment_{ref,fsx} [experiment ...]   (mllm | omni)
// Each experiment runs twice in the process: the first run pays the one-time
// setup (for fsx: CUDA context, slabs, pinned staging), the second is warm.
#include <chrono>
#include <cstdio>
#include <fstream>
#include <string>

#include "fissim/bench_harness.hpp"

using namespace fissim;

namespace {

std::string repo(const std::string& rel) { return std::string(FISSIM_REPO_ROOT) + "/" + rel; }

json load_json(const std::string& rel) {
  std::ifstream in(repo(rel));
  if (!in.good()) throw std::runtime_error("missing " + repo(rel));
  json j;
  in >> j;
  return j;
}

uint64_t fnv(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
  return h;
}

ExperimentConfig experiment(const std::string& name) {
  ExperimentConfig cfg;
  cfg.cluster.clock = ClockMode::Virtual;
  if (name == "mllm") {  // InternVL3-style image->text chat (config A's app)
    cfg.cluster.nodes.push_back({0, 2, int64_t{80} * 1000 * 1000 * 1000});
    cfg.cluster.profile_files = {repo("profiles/mllm.json")};
    cfg.app = AppManifest::from_json(load_json("apps/mllm-gemma.json"));
    cfg.mix = WorkloadMix::from_json(load_json("mixes/mllm-chat.json"));
    cfg.rate_per_s = 2.0;
    cfg.duration_s = 60;
    cfg.seed = 42;
  } else {  // omni: thinker -> talker -> generator (config C's app)
    cfg.cluster.nodes.push_back({0, 8, int64_t{80} * 1000 * 1000 * 1000});
    cfg.cluster.profile_files = {repo("profiles/qwen25-omni.json")};
    cfg.app = AppManifest::from_json(load_json("apps/omni-qwen25.json"));
    cfg.mix = WorkloadMix::from_json(load_json("mixes/qwen25-audio-chat.json"));
    cfg.rate_per_s = 1.0;
    cfg.duration_s = 60;
    cfg.seed = 5;
  }
  return cfg;
}

}  // namespace

int main(int argc, char** argv) {
#ifdef FSX_DROPIN
  const char* impl = "fsx";
#else
  const char* impl = "reference";
#endif
  std::vector<std::string> names;
  for (int i = 1; i < argc; ++i) names.push_back(argv[i]);
  if (names.empty()) names = {"mllm", "omni"};
  for (const auto& name : names) {
    for (int run = 0; run < 2; ++run) {
      auto cfg = experiment(name);
      const auto t0 = std::chrono::steady_clock::now();
      BenchReport report = run_experiment(cfg);
      const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      const std::string js = report.to_json().dump();
      std::printf("{\"experiment\": \"%s\", \"impl\": \"%s\", \"run\": \"%s\", \"wall_s\": %.3f, "
                  "\"report_fnv1a\": \"%016llx\", \"completed\": %lld, \"failed\": %lld, \"p50_ms\": %.3f, "
                  "\"achieved_throughput\": %.4f}\n",
                  name.c_str(), impl, run ? "warm" : "first", wall, (unsigned long long)fnv(js),
                  (long long)report.completed, (long long)report.failed, report.p50_ms, report.achieved_throughput);
      std::fflush(stdout);
    }
  }
  return 0;
}
