// Host dg64 of include/fsx/fabric.hpp (digest64: four accumulators;
// digest64_par: word ranges on several threads) against the oracle C
// restatement or_digest64 (oracle/fsx_oracle.c, test infrastructure), over
// empty, tail-only, odd and multi-MiB sizes incl. the threaded range.  CPU only.
#include <cstdio>
#include <vector>

#include "fsx/fabric.hpp"

extern "C" {
#include "fsx_oracle.h"
}

int main() {
  const size_t big = (size_t{48} << 20) + 13;
  std::vector<uint8_t> buf(big);
  or_synth_payload_into(0x5eedull, buf.data(), buf.size());
  const size_t sizes[] = {0, 1, 7, 8, 9, 31, 32, 33, 63, 64, 65, 4095, 7168, 7171, size_t{1} << 20,
                          (size_t{16} << 20) + 7, (size_t{32} << 20), big};
  int failed = 0, cases = 0;
  for (size_t n : sizes)
    for (size_t shift : {size_t{0}, size_t{3}}) {
      if (n + shift > buf.size()) continue;
      const uint8_t* p = buf.data() + shift;
      const uint64_t want = or_digest64(p, n);
      ++cases;
      if (fsx::digest64(p, n) != want || fsx::digest64_par(p, n) != want) {
        std::printf("MISMATCH n=%zu shift=%zu\n", n, shift);
        ++failed;
      }
    }
  std::printf("%d digest cases, %d failed\n", cases, failed);
  return failed ? 1 : 0;
}
