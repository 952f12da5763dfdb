// Binary envelope codec (include/fsx/envelope_codec.hpp):
// round trips of the standalone and the drop-in (fissim) envelope, rejection
// of truncated / foreign records, and the per-envelope cost next to the
// reference's JSON route (ForwardEnvelope::to_json -> dump -> parse ->
// from_json, sidecar.hpp:59-100 / 474-479).  CPU only.
#include <catch_amalgamated.hpp>

#include <chrono>
#include <cstdio>

#include "fissim/sidecar.hpp"  // the drop-in (include/fsx/dropin first on the path)
#include "fsx/envelope_codec.hpp"

namespace {

fissim::ForwardEnvelope sample() {
  fissim::ForwardEnvelope e;
  e.request_id = "req-000123";
  e.ref_id = "req-000123/r0001";
  e.seq = 4711;
  e.chunk_bytes = 7168;
  e.total_bytes = 0;
  e.checksum = 0x9e3779b97f4a7c15ull;
  e.transport = fsx::Transport::LocalBuffer;
  e.location = "gpu1:off1048576";
  e.final = false;
  e.send_time = 12.5;
  e.src_gpu = 0;
  e.dst_gpu = 1;
  return e;
}

bool same(const fissim::ForwardEnvelope& a, const fissim::ForwardEnvelope& b) {
  return a.to_json() == b.to_json();
}

}  // namespace

TEST_CASE("binary envelope round-trips every field") {
  for (int variant = 0; variant < 4; ++variant) {
    auto e = sample();
    e.final = variant & 1;
    e.transport = (variant & 2) ? fsx::Transport::NetworkStream : fsx::Transport::LocalBuffer;
    e.location = (variant & 2) ? "" : e.location;
    std::vector<uint8_t> buf;
    REQUIRE(fsx::encode_envelope(e, buf));
    fissim::ForwardEnvelope d;
    CHECK(fsx::decode_envelope(buf.data(), buf.size(), &d) == buf.size());
    CHECK(same(e, d));
  }
  // the standalone engine's envelope type uses the same codec
  fsx::ForwardEnvelope s;
  s.request_id = "r";
  s.ref_id = "r/x";
  s.seq = -1;
  s.final = true;
  std::vector<uint8_t> buf;
  REQUIRE(fsx::encode_envelope(s, buf));
  fsx::ForwardEnvelope t;
  CHECK(fsx::decode_envelope(buf.data(), buf.size(), &t) == buf.size());
  CHECK(t.ref_id == "r/x");
  CHECK(t.seq == -1);
  CHECK(t.final);
}

TEST_CASE("truncated, foreign and oversized records are rejected") {
  auto e = sample();
  std::vector<uint8_t> buf;
  REQUIRE(fsx::encode_envelope(e, buf));
  fissim::ForwardEnvelope d;
  for (size_t cut = 0; cut < buf.size(); ++cut) CHECK(fsx::decode_envelope(buf.data(), cut, &d) == 0);
  auto bad = buf;
  bad[0] ^= 0xff;  // magic
  CHECK(fsx::decode_envelope(bad.data(), bad.size(), &d) == 0);
  bad = buf;
  bad[4] = 9;  // version
  CHECK(fsx::decode_envelope(bad.data(), bad.size(), &d) == 0);
  e.ref_id.assign(70000, 'x');
  std::vector<uint8_t> big;
  CHECK_FALSE(fsx::encode_envelope(e, big));
}

TEST_CASE("binary envelope cost next to the reference JSON route") {
  const auto e = sample();
  const int n = 200000;
  uint64_t sink = 0;
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i) {
    const std::string wire = e.to_json().dump();
    const auto d = fissim::ForwardEnvelope::from_json(fissim::json::parse(wire));
    sink += static_cast<uint64_t>(d.seq) + wire.size();
  }
  auto t1 = std::chrono::steady_clock::now();
  std::vector<uint8_t> buf;
  for (int i = 0; i < n; ++i) {
    buf.clear();
    fsx::encode_envelope(e, buf);
    fissim::ForwardEnvelope d;
    sink += fsx::decode_envelope(buf.data(), buf.size(), &d) + static_cast<uint64_t>(d.seq);
  }
  auto t2 = std::chrono::steady_clock::now();
  const double json_ns = std::chrono::duration<double, std::nano>(t1 - t0).count() / n;
  const double bin_ns = std::chrono::duration<double, std::nano>(t2 - t1).count() / n;
  std::printf("{\"json_ns_per_envelope\": %.0f, \"binary_ns_per_envelope\": %.0f, \"json_bytes\": %zu, "
              "\"binary_bytes\": %zu, \"sink\": %llu}\n",
              json_ns, bin_ns, e.to_json().dump().size(), buf.size(), (unsigned long long)sink);
  CHECK(bin_ns < json_ns);
}
