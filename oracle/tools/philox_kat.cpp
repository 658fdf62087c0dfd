// Generates tests/golden/philox_kat.json from PyTorch's header-only
// at::Philox4_32 (ATen/core/PhiloxRNGEngine.h), an independent Philox4x32-10
// implementation, to pin oracle/gsb_oracle.c:gso_philox4x32_10.
// Build/run: oracle/tools/make_philox_kat.sh  (test infrastructure only)
#include <ATen/core/PhiloxRNGEngine.h>
#include <cstdint>
#include <cstdio>

int main() {
  // at::Philox4_32(seed, subsequence, offset): key = (lo32 seed, hi32 seed),
  // counter = (lo32 offset, hi32 offset, lo32 subseq, hi32 subseq); operator()
  // returns the 4 output words in order, then advances the offset.
  const uint64_t seeds[] = {0ull, 1ull, 0xFFFFFFFFFFFFFFFFull, 0x299f31d0a4093822ull,
                            4439793921019041103ull, 11420144667590826704ull};
  const uint64_t subs[] = {0ull, 1ull, 0x0000000100000002ull, 0xFFFFFFFFFFFFFFFFull,
                           0x1370734413198a2eull};
  const uint64_t offs[] = {0ull, 5ull, 0x85a308d3243f6a88ull, 0xFFFFFFFFFFFFFFFFull};
  std::printf("{\"source\": \"torch at::Philox4_32 (ATen/core/PhiloxRNGEngine.h)\",\n \"cases\": [\n");
  bool first = true;
  for (uint64_t s : seeds)
    for (uint64_t q : subs)
      for (uint64_t o : offs) {
        at::Philox4_32 eng(s, q, o);
        uint32_t out[4];
        for (int i = 0; i < 4; i++) out[i] = eng();
        std::printf("%s  {\"ctr\": [%u, %u, %u, %u], \"key\": [%u, %u], \"out\": [%u, %u, %u, %u]}",
                    first ? "" : ",\n", (uint32_t)o, (uint32_t)(o >> 32), (uint32_t)q,
                    (uint32_t)(q >> 32), (uint32_t)s, (uint32_t)(s >> 32), out[0], out[1], out[2],
                    out[3]);
        first = false;
      }
  std::printf("\n ]}\n");
  return 0;
}
