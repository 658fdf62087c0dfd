// gsb_device.cuh -- device-side RNG primitives shared by the sweep kernels.
//
//  * Philox4x32-10 (counter-based; checkerboard engine).  Pinned against
//    torch's at::Philox4_32 and the Random123 KATs (tests/golden/philox_kat.json).
//  * numpy PCG64 emulation (reference engine): SeedSequence seeding, XSL-RR
//    output, next32 half-buffering and O(log k) jump-ahead.  Mirrors what
//    gsetbench.solvers.run_trial consumes through np.random.default_rng
//    (solvers.py:94, :96, :110, :118); restated from numpy's published
//    algorithms, pinned by tests/golden/rng_kat.json.
#pragma once
#include <cstdint>

namespace gsb {

// ------------------------------------------------------------------ Philox
struct P4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ void mulwide(uint32_t a, uint32_t b, uint32_t &hi, uint32_t &lo) {
  hi = __umulhi(a, b);
  lo = a * b;
}

__device__ __forceinline__ P4 philox10(P4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    uint32_t hi0, lo0, hi1, lo1;
    mulwide(0xD2511F53u, c.x, hi0, lo0);
    mulwide(0xCD9E8D57u, c.z, hi1, lo1);
    P4 n;
    n.x = hi1 ^ c.y ^ k0;
    n.y = lo1;
    n.z = hi0 ^ c.w ^ k1;
    n.w = lo0;
    c = n;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// ------------------------------------------------------------------ PCG64
typedef unsigned __int128 u128;

__host__ __device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

__host__ __device__ __forceinline__ uint64_t pcg_out(u128 s) {
  uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  unsigned rot = (unsigned)(s >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// SeedSequence(seed).generate_state(4, uint64) -> pcg64_set_seed
__host__ __device__ inline void pcg_seed(uint64_t seed, u128 &state, u128 &inc) {
  uint32_t ent0 = (uint32_t)seed, ent1 = (uint32_t)(seed >> 32);
  int nent = (seed >> 32) ? 2 : 1;
  uint32_t pool[4];
  uint32_t hc = 0x43b0d7e5u;
  for (int i = 0; i < 4; i++) {
    uint32_t v = i == 0 ? ent0 : (i == 1 && nent == 2 ? ent1 : 0u);
    v ^= hc;
    hc *= 0x931e8875u;
    v *= hc;
    v ^= v >> 16;
    pool[i] = v;
  }
  for (int s = 0; s < 4; s++)
    for (int d = 0; d < 4; d++)
      if (s != d) {
        uint32_t v = pool[s];
        v ^= hc;
        hc *= 0x931e8875u;
        v *= hc;
        v ^= v >> 16;
        uint32_t r = 0xca01f9ddu * pool[d] - 0x4973f715u * v;
        r ^= r >> 16;
        pool[d] = r;
      }
  uint32_t words[8];
  uint32_t hb = 0x8b51f9ddu;
  for (int i = 0; i < 8; i++) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= 0x58f38dedu;
    v *= hb;
    v ^= v >> 16;
    words[i] = v;
  }
  uint64_t val[4];
  for (int i = 0; i < 4; i++) val[i] = (uint64_t)words[2 * i] | ((uint64_t)words[2 * i + 1] << 32);
  u128 s = ((u128)val[0] << 64) | val[1];
  u128 q = ((u128)val[2] << 64) | val[3];
  inc = (q << 1) | 1u;
  u128 st = 0;
  st = st * pcg_mult() + inc;
  st += s;
  st = st * pcg_mult() + inc;
  state = st;
}

// (A, C) such that step^k(s) = A*s + C
__host__ __device__ inline void pcg_jump_coeffs(uint64_t k, u128 inc, u128 &A, u128 &C) {
  u128 am = 1, ap = 0, cm = pcg_mult(), cp = inc;
  while (k) {
    if (k & 1) {
      am *= cm;
      ap = ap * cm + cp;
    }
    cp = (cm + 1) * cp;
    cm *= cm;
    k >>= 1;
  }
  A = am;
  C = ap;
}

}  // namespace gsb
