// Worker executable for multi-process executors on the fsx drop-in: the
// `executor-worker --host H --port P` subcommand of the reference CLI
// (tools/fissim_cli.cpp:378-397), which cannot be built here (CLI11 absent),
// reduced to that one subcommand.  The parent (MultiProcessHost in
// include/fsx/dropin/fissim/executor_worker.hpp) execs it per replica.
#include <cstring>
#include <iostream>
#include <string>

#include "fissim/executor_worker.hpp"

int main(int argc, char** argv) {
  std::string host = "127.0.0.1";
  int port = 0;
  if (argc < 2 || std::strcmp(argv[1], "executor-worker") != 0) {
    std::cerr << "usage: " << argv[0] << " executor-worker --host H --port P\n";
    return 1;
  }
  for (int i = 2; i + 1 < argc; i += 2) {
    if (std::strcmp(argv[i], "--host") == 0) host = argv[i + 1];
    else if (std::strcmp(argv[i], "--port") == 0) port = std::atoi(argv[i + 1]);
  }
  if (port <= 0) {
    std::cerr << "--port is required\n";
    return 1;
  }
  try {
    return fissim::run_executor_worker(host, port);
  } catch (const fissim::Error& e) {
    std::cerr << e.to_json().dump() << "\n";
    return e.code() == fissim::ErrorCode::Internal ? 2 : 1;
  }
}
