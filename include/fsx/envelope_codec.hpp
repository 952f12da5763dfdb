// fsx/envelope_codec.hpp -- binary form of the sidecar envelope (SURVEY.md
// 8f-4, second half).
//
// The reference serialises every ForwardEnvelope as a ~300-byte JSON object
// (sidecar.hpp:59-100, docs/formats.md:253-287) and round-trips it through the
// frame codec even in memory (sidecar.hpp:474-479); for config C's per-token
// messages that JSON dump/parse is most of the per-message cost.  The fsx
// engine keeps envelopes as structs in process; where an envelope does cross
// a process boundary (the multi-process worker protocol, dropin
// executor_worker.hpp) it travels as this fixed little-endian record:
//
//   u32 magic 'FSXE' | u16 version | u16 flags (bit0 final, bit1 network)
//   i64 seq | i64 chunk_bytes | i64 total_bytes | u64 checksum | f64 send_time
//   i32 src_gpu | i32 dst_gpu
//   u16 len + bytes: request_id, ref_id, location
//
// Header-only, templated on the envelope type (fsx::ForwardEnvelope or the
// drop-in fissim::ForwardEnvelope: same field names, fsx::Transport).
#pragma once

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "fsx/fabric.hpp"  // fsx::Transport

namespace fsx {

constexpr uint32_t kEnvelopeMagic = 0x45585346u;  // "FSXE" little-endian
constexpr uint16_t kEnvelopeVersion = 1;
constexpr size_t kEnvelopeFixedBytes = 4 + 2 + 2 + 8 * 5 + 4 * 2;

namespace codec_detail {

template <class T>
inline void put(std::vector<uint8_t>& out, T v) {
  const size_t at = out.size();
  out.resize(at + sizeof(T));
  std::memcpy(out.data() + at, &v, sizeof(T));  // little-endian host (x86-64 / aarch64)
}

inline bool put_str(std::vector<uint8_t>& out, const std::string& s) {
  if (s.size() > 0xffff) return false;
  put<uint16_t>(out, static_cast<uint16_t>(s.size()));
  out.insert(out.end(), s.begin(), s.end());
  return true;
}

struct Reader {
  const uint8_t* p;
  size_t n, at = 0;
  template <class T>
  bool get(T* v) {
    if (n - at < sizeof(T)) return false;
    std::memcpy(v, p + at, sizeof(T));
    at += sizeof(T);
    return true;
  }
  bool get_str(std::string* s) {
    uint16_t len = 0;
    if (!get(&len) || n - at < len) return false;
    s->assign(reinterpret_cast<const char*>(p + at), len);
    at += len;
    return true;
  }
};

}  // namespace codec_detail

// Appends the binary envelope to `out`; false if a string field exceeds 64 KiB.
template <class Env>
inline bool encode_envelope(const Env& e, std::vector<uint8_t>& out) {
  using namespace codec_detail;
  out.reserve(out.size() + kEnvelopeFixedBytes + 6 + e.request_id.size() + e.ref_id.size() +
              e.location.size());
  put<uint32_t>(out, kEnvelopeMagic);
  put<uint16_t>(out, kEnvelopeVersion);
  const uint16_t flags = static_cast<uint16_t>((e.final ? 1u : 0u) |
                                               (e.transport == Transport::NetworkStream ? 2u : 0u));
  put<uint16_t>(out, flags);
  put<int64_t>(out, e.seq);
  put<int64_t>(out, e.chunk_bytes);
  put<int64_t>(out, e.total_bytes);
  put<uint64_t>(out, e.checksum);
  put<double>(out, static_cast<double>(e.send_time));
  put<int32_t>(out, e.src_gpu);
  put<int32_t>(out, e.dst_gpu);
  return put_str(out, e.request_id) && put_str(out, e.ref_id) && put_str(out, e.location);
}

// Decodes one envelope from [p, p + n); returns the bytes consumed, 0 on a
// malformed or foreign record (wrong magic / version, truncated).
template <class Env>
inline size_t decode_envelope(const uint8_t* p, size_t n, Env* e) {
  codec_detail::Reader r{p, n};
  uint32_t magic = 0;
  uint16_t version = 0, flags = 0;
  double send_time = 0;
  if (!r.get(&magic) || magic != kEnvelopeMagic || !r.get(&version) || version != kEnvelopeVersion ||
      !r.get(&flags) || !r.get(&e->seq) || !r.get(&e->chunk_bytes) || !r.get(&e->total_bytes) ||
      !r.get(&e->checksum) || !r.get(&send_time) || !r.get(&e->src_gpu) || !r.get(&e->dst_gpu) ||
      !r.get_str(&e->request_id) || !r.get_str(&e->ref_id) || !r.get_str(&e->location))
    return 0;
  e->final = (flags & 1u) != 0;
  e->transport = (flags & 2u) ? Transport::NetworkStream : Transport::LocalBuffer;
  e->send_time = send_time;
  return r.at;
}

}  // namespace fsx
