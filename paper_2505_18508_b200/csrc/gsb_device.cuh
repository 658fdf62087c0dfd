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

// Philox4x32-10 of a counter (wi, t, q, 1) from round 2 on.  Rounds 0-1 of
// such a counter split into a part that depends only on (wi, q) and the key
// (PhiloxPre, per trial) and a part that depends only on (t, q) and the key
// (PhiloxUni, per sweep and plane pair, uniform over words):
//   round 0: x1 = hi(M1 q) ^ t ^ k0, y1 = lo(M1 q), z1 = hi(M0 wi) ^ 1 ^ k1,
//            w1 = lo(M0 wi)
//   round 1: x2 = hi(M1 z1) ^ y1 ^ k0', y2 = lo(M1 z1),
//            z2 = hi(M0 x1) ^ w1 ^ k1', w2 = lo(M0 x1)
//   round 2: (hi0, lo0) = M0 x2  -- (wi, q) only: pre.hi / pre.lo
//            x3 = hi(M1 z2) ^ y2 ^ k0'', y3 = lo(M1 z2),
//            z3 = hi0 ^ w2 ^ k1'', w3 = lo0
// so a block costs one multiply and three XORs for rounds 0-2 instead of six
// and six.  Same outputs as philox10 (checked in tests through the kernels).
constexpr uint32_t kPhiloxM0 = 0xD2511F53u, kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u, kPhiloxW1 = 0xBB67AE85u;

struct PhiloxWord {  // per (trial, wi): c1 = w1 ^ k1', c2 = y2 ^ k0''
  uint32_t c1, c2;
};

__device__ __forceinline__ PhiloxWord philox_word(uint32_t wi, uint32_t k0, uint32_t k1,
                                                  uint32_t &h1z) {
  const uint32_t h0 = __umulhi(kPhiloxM0, wi), l0 = kPhiloxM0 * wi;
  const uint32_t z1 = h0 ^ 1u ^ k1;
  h1z = __umulhi(kPhiloxM1, z1);
  return PhiloxWord{l0 ^ (k1 + kPhiloxW1), (kPhiloxM1 * z1) ^ (k0 + 2u * kPhiloxW0)};
}

// per (trial, wi, q): M0 * x2 as (hi, lo)
__device__ __forceinline__ void philox_pre(uint32_t h1z, uint32_t q, uint32_t k0, uint32_t &hi,
                                           uint32_t &lo) {
  const uint32_t x2 = h1z ^ (kPhiloxM1 * q) ^ (k0 + kPhiloxW0);
  hi = __umulhi(kPhiloxM0, x2);
  lo = kPhiloxM0 * x2;
}

// per (trial, t, q), uniform over words: u1 = hi(M0 x1), v = lo(M0 x1) ^ k1''
__device__ __forceinline__ void philox_uni(uint32_t t, uint32_t q, uint32_t k0, uint32_t k1,
                                           uint32_t &u1, uint32_t &v) {
  const uint32_t x1 = __umulhi(kPhiloxM1, q) ^ t ^ k0;
  u1 = __umulhi(kPhiloxM0, x1);
  v = (kPhiloxM0 * x1) ^ (k1 + 2u * kPhiloxW1);
}

__device__ __forceinline__ P4 philox10_from2(const PhiloxWord &pw, uint32_t pre_hi,
                                             uint32_t pre_lo, uint32_t u1, uint32_t v,
                                             uint32_t k0, uint32_t k1) {
  const uint32_t z2 = u1 ^ pw.c1;
  P4 c{__umulhi(kPhiloxM1, z2) ^ pw.c2, kPhiloxM1 * z2, pre_hi ^ v, pre_lo};
  k0 += 3u * kPhiloxW0;
  k1 += 3u * kPhiloxW1;
#pragma unroll
  for (int r = 3; r < 10; r++) {
    uint32_t hi0, lo0, hi1, lo1;
    mulwide(kPhiloxM0, c.x, hi0, lo0);
    mulwide(kPhiloxM1, c.z, hi1, lo1);
    P4 n;
    n.x = hi1 ^ c.y ^ k0;
    n.y = lo1;
    n.z = hi0 ^ c.w ^ k1;
    n.w = lo0;
    c = n;
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
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
