// Phase breakdown of the config-C small-message path (32 host-span rows per
// decode step into ChunkCallback consumers): what each C-ABI step and each
// host-side piece of fsx::Fabric::send / deliver costs on its own, so the
// per-step total of build/bench_fabric can be attributed.  One JSON line per
// phase, microseconds per step (32 messages).
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#include "fsx/fabric.hpp"

using clk = std::chrono::steady_clock;

static double us_since(clk::time_point a) {
  return std::chrono::duration<double, std::micro>(clk::now() - a).count();
}

int main(int argc, char** argv) {
  const int row = argc > 1 ? std::atoi(argv[1]) : 7168;
  const int batch = 32, steps = 400;
  int ids[2] = {0, 1}, nodes[2] = {0, 0}, devs[2] = {-1, -1};
  fsx_fabric* f = nullptr;
  if (fsx_open(2, ids, nodes, devs, &f) != FSX_OK) {
    std::fprintf(stderr, "fsx_open: %s\n", fsx_last_error());
    return 2;
  }
  fsx_slab_register(f, 1, int64_t{64} << 20);
  std::vector<uint8_t> rowbuf(row, 7);
  auto line = [&](const char* phase, double us_total) {
    std::printf("{\"phase\": \"%s\", \"row_bytes\": %d, \"rows_per_step\": %d, \"us_per_step\": %.2f}\n", phase,
                row, batch, us_total / steps);
  };
  auto run = [&](const char* phase, auto&& body) {
    for (int s = 0; s < 20; ++s) body();
    const auto a = clk::now();
    for (int s = 0; s < steps; ++s) body();
    line(phase, us_since(a));
  };
  run("pointer_device_x32", [&] {
    int d = 0;
    for (int r = 0; r < batch; ++r) fsx_pointer_device(rowbuf.data(), &d);
  });
  run("pointer_kind_x32", [&] {
    int k = 0;
    for (int r = 0; r < batch; ++r) fsx_pointer_kind(rowbuf.data(), &k);
  });
  volatile uint64_t sink = 0;
  run("host_digest64_x32", [&] {
    for (int r = 0; r < batch; ++r) sink = sink + fsx::digest64(rowbuf.data(), rowbuf.size());
  });
  run("slab_alloc_free_x32", [&] {
    int64_t off[32];
    for (int r = 0; r < batch; ++r) fsx_slab_alloc(f, 1, row, &off[r]);
    for (int r = 0; r < batch; ++r) fsx_slab_free(f, 1, off[r]);
  });
  std::vector<uint8_t> out(row);
  run("put_small_flush_wait_free_x32", [&] {
    int64_t off[32], t[32];
    for (int r = 0; r < batch; ++r) fsx_slab_alloc(f, 1, row, &off[r]);
    for (int r = 0; r < batch; ++r) fsx_put_small(f, 1, off[r], rowbuf.data(), row, &t[r]);
    for (int r = 0; r < batch; ++r) {
      const void* m = nullptr;
      uint64_t dg = 0;
      fsx_ticket_wait(f, t[r], &m, &dg);
      std::memcpy(out.data(), m, row);
      fsx_ticket_free(f, t[r]);
    }
    for (int r = 0; r < batch; ++r) fsx_slab_free(f, 1, off[r]);
  });
  // only the staging part (no flush) and only the device round trip
  {
    double stage = 0, trip = 0;
    for (int s = 0; s < steps + 20; ++s) {
      int64_t off[32], t[32];
      for (int r = 0; r < batch; ++r) fsx_slab_alloc(f, 1, row, &off[r]);
      const auto a = clk::now();
      for (int r = 0; r < batch; ++r) fsx_put_small(f, 1, off[r], rowbuf.data(), row, &t[r]);
      const double st = us_since(a);
      const auto b = clk::now();
      fsx_flush_small(f);
      const void* m = nullptr;
      uint64_t dg = 0;
      fsx_ticket_wait(f, t[batch - 1], &m, &dg);
      const double tr = us_since(b);
      if (s >= 20) {
        stage += st;
        trip += tr;
      }
      for (int r = 0; r < batch; ++r) fsx_ticket_free(f, t[r]);
      for (int r = 0; r < batch; ++r) fsx_slab_free(f, 1, off[r]);
    }
    line("put_small_stage_x32", stage);
    line("mailbox_flush_and_wait", trip);
  }
  run("owned_vector_assign_x32", [&] {
    for (int r = 0; r < batch; ++r) {
      std::vector<uint8_t> v(rowbuf.begin(), rowbuf.end());
      sink = sink + v[0];
    }
  });
  run("event_loop_schedule_run_x32", [&] {
    fsx::EventLoop k;
    for (int r = 0; r < batch; ++r) {
      auto env = std::make_shared<fsx::ForwardEnvelope>();
      env->ref_id = "req-" + std::to_string(r) + "/r0001";
      k.schedule(1.0, "sidecar.deliver", [env] { (void)env; });
    }
    k.run_until_idle();
  });
  fsx_close(f);
  return 0;
}
