// checker_common.cuh -- per-word pieces of the checkerboard sweep shared by the
// shared-memory engine (checker.cu) and the HBM-tiled engine (checker_hbm.cu).
// Bit layout and contract: see checker.cu / DESIGN.md.
#pragma once
#include <cstdint>

#include "gsb_device.cuh"

namespace gsb {

// lop3.b32 with an explicit truth table (a = 0xF0, b = 0xCC, c = 0xAA): nvcc
// splits some 3-input functions into two LOP3s, this keeps them one.
template <uint32_t LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
  return d;
}

__device__ __forceinline__ uint32_t shifted_nb(const uint32_t *__restrict__ o, uint32_t same,
                                               uint32_t cidx, uint32_t cinfo) {
  const uint32_t src = cinfo & 31u, dst = (cinfo >> 5) & 31u;
  const uint32_t carry = ((o[cidx] >> src) & 1u) << dst;
  return ((cinfo >> 10) & 1u) ? ((same >> 1) | carry) : ((same << 1) | carry);
}

// cut contribution of a colour-0 word: sum over its 4 edges of w*[differ]
__device__ __forceinline__ int word_cut(uint32_t s, uint32_t same, uint32_t sh, uint32_t up,
                                        uint32_t dn, uint4 m, uint32_t v) {
  int c = 0;
  uint32_t x;
  x = (s ^ same) & v;
  c += __popc(x & ~m.x) - __popc(x & m.x);
  x = (s ^ sh) & v;
  c += __popc(x & ~m.y) - __popc(x & m.y);
  x = (s ^ up) & v;
  c += __popc(x & ~m.z) - __popc(x & m.z);
  x = (s ^ dn) & v;
  c += __popc(x & ~m.w) - __popc(x & m.w);
  return c;
}

// Delta classes of a word (bit-sliced counts of the 4 positive-term planes)
struct Classes {
  uint32_t ge2, k3, k4, km2, km4;
};

__device__ __forceinline__ Classes classes(uint32_t Sw, uint32_t same, uint32_t sh, uint32_t up,
                                           uint32_t dn, uint4 m, uint32_t V) {
  const uint32_t P0 = ~(Sw ^ same ^ m.x);
  const uint32_t P1 = ~(Sw ^ sh ^ m.y);
  const uint32_t P2 = ~(Sw ^ up ^ m.z);
  const uint32_t P3 = ~(Sw ^ dn ^ m.w);
  const uint32_t x01 = P0 ^ P1, c01 = P0 & P1, x23 = P2 ^ P3, c23 = P2 & P3;
  const uint32_t ones = x01 ^ x23;
  Classes c;
  c.ge2 = (c01 | c23 | (x01 & x23)) & V;  // Delta >= 0
  c.k4 = c01 & c23 & V;                    // Delta = +4
  c.k3 = ((c01 | c23) & ones) & V;         // Delta = +2
  const uint32_t any = P0 | P1 | P2 | P3;
  c.km2 = any & ~c.ge2 & V;  // Delta = -2
  c.km4 = ~any & V;          // Delta = -4
  return c;
}

// Shifted neighbour word with its padding bits cleared (V = valid bits): the
// input classes_pad() expects.
__device__ __forceinline__ uint32_t shifted_nb_v(const uint32_t *__restrict__ o, uint32_t same,
                                                 uint32_t cidx, uint32_t cinfo, uint32_t V) {
  const uint32_t src = cinfo & 31u, dst = (cinfo >> 5) & 31u;
  const uint32_t carry = ((o[cidx] >> src) & 1u) << dst;
  const uint32_t t = ((cinfo >> 10) & 1u) ? (same >> 1) : (same << 1);
  return lop3<0xA8>(t, carry, V);  // (t | carry) & V
}

// word at a byte offset into the shared spin copy
__device__ __forceinline__ uint32_t word_at(const uint32_t *base, uint32_t off) {
  return *(const uint32_t *)((const char *)base + off);
}

// Shifted neighbour from the per-colour table of checker_geo2_kernel:
// ga = {up, down, carry offsets, V}, gb = {VG, r, a, b}.  4 ALU ops.
__device__ __forceinline__ uint32_t shifted_nb2(const uint32_t *st, uint32_t same, uint4 ga,
                                                uint4 gb) {
  const uint32_t rot = __funnelshift_l(same, same, gb.y);  // rotate left by r
  const uint32_t carry = (word_at(st, ga.z) << gb.z) >> gb.w;
  return lop3<0xEA>(rot, gb.x, carry);  // (rot & VG) | carry
}

// Delta classes in 11 LOP3s, using the padding convention of
// checker_masks_kernel (coupling planes NU/ND set, NS/NSH clear on padding
// bits) and padding-free spin/neighbour words: a padding site then has
// exactly two positive terms (Delta = 0), so k3/k4/km2/km4 never contain it
// and only ge2 must be masked with V by the caller.
//   a+b+c = 2*c1 + s1 (full adder), #positive = 2*c1 + s1 + d
__device__ __forceinline__ Classes classes_pad(uint32_t Sw, uint32_t same, uint32_t sh, uint32_t up,
                                               uint32_t dn, uint4 m) {
  const uint32_t a = lop3<0x69>(Sw, same, m.x);  // ~(x ^ y ^ z)
  const uint32_t b = lop3<0x69>(Sw, sh, m.y);
  const uint32_t c = lop3<0x69>(Sw, up, m.z);
  const uint32_t d = lop3<0x69>(Sw, dn, m.w);
  const uint32_t s1 = lop3<0x96>(a, b, c);  // a ^ b ^ c
  const uint32_t c1 = lop3<0xE8>(a, b, c);  // majority
  Classes r;
  r.ge2 = lop3<0xF8>(c1, s1, d);  // c1 | (s1 & d): >= 2 positive   (Delta >= 0, unmasked)
  r.k4 = lop3<0x80>(c1, s1, d);   // c1 & s1 & d:     4 positive     (Delta = +4)
  r.k3 = lop3<0x60>(c1, s1, d);   // c1 & (s1 ^ d):   3 positive     (Delta = +2)
  r.km4 = lop3<0x01>(c1, s1, d);  // ~(c1 | s1 | d):  0 positive     (Delta = -4)
  r.km2 = lop3<0x06>(c1, s1, d);  // ~c1 & (s1 ^ d):  1 positive     (Delta = -2)
  return r;
}

// Bit-sliced comparison of the uniforms' top 8 bits with the thresholds, as a
// borrow chain over the planes LSB-first (plane 7 = uniform bit 24 first,
// plane 0 = bit 31 last).  c2 = class -2 sites (threshold K2), other pending
// sites use K4; ma/mb = all-ones iff the plane's bit of K2/K4 is set (per
// sweep, uniform).  lt becomes [u_hi < K_hi] (strict), eq keeps the pending
// sites whose 8 bits all equal K_hi.  3 LOP3 per plane.
__device__ __forceinline__ void cmp_plane_lsb(uint32_t R, uint32_t c2, uint32_t ma, uint32_t mb,
                                              uint32_t &eq, uint32_t &lt) {
  const uint32_t tb = lop3<0xCA>(c2, ma, mb);  // c2 ? ma : mb
  lt = lop3<0xB2>(tb, R, lt);                  // tb ? (~R | lt) : (~R & lt)
  eq = lop3<0x90>(eq, R, tb);                  // eq & ~(R ^ tb)
}

// Leading planes in which both thresholds' top bytes are 0 (per sweep,
// uniform): 8 when K2, K4 < 2^24, 4 when K2, K4 < 2^28, else 0.  On the
// default schedule (3.0 -> 0.05) that is 48 % / 17 % / 35 % of the sweeps.
__device__ __forceinline__ int zero_planes(uint32_t K2, uint32_t K4) {
  const uint32_t khi = (K2 | K4) >> 24;
  return khi == 0u ? 8 : (khi >> 4) == 0u ? 4 : 0;
}

// The top-8-bit comparison of a word's pending sites, planes r0 = uniform bits
// 31..28 (x..w), r1 = bits 27..24.  eq = pending sites whose 8 bits equal
// K_hi (undecided, go to the tail), lt = pending sites with u_hi < K_hi
// (accepted).  With L leading planes where both K_hi bits are 0 a set bit
// there already means u_hi > K_hi, so those planes collapse to one OR
// (L = 8: 4 LOP3 instead of 25; L = 4: 16).  Same results for every L.
template <int L>
__device__ __forceinline__ void cmp_planes(const P4 &r0, const P4 &r1, uint32_t c2, uint32_t pend,
                                           uint32_t K2, uint32_t K4, uint32_t &eq, uint32_t &lt) {
  static_assert(L == 0 || L == 4 || L == 8, "L is 0, 4 or 8");
  if (L == 8) {
    uint32_t z = lop3<0xFE>(r0.x, r0.y, r0.z);  // OR3
    z = lop3<0xFE>(z, r0.w, r1.x);
    z = lop3<0xFE>(z, r1.y, r1.z);
    eq = lop3<0x10>(pend, z, r1.w);  // pend & ~(z | w)
    lt = 0u;
    return;
  }
  // plane masks: all-ones iff bit 31-j of K2 / K4 is set (uniform)
  uint32_t ma[8], mb[8];
#pragma unroll
  for (int j = L; j < 8; j++) {
    ma[j] = (uint32_t)((int32_t)(K2 << j) >> 31);
    mb[j] = (uint32_t)((int32_t)(K4 << j) >> 31);
  }
  uint32_t q = pend, l = 0;
  cmp_plane_lsb(r1.w, c2, ma[7], mb[7], q, l);
  cmp_plane_lsb(r1.z, c2, ma[6], mb[6], q, l);
  cmp_plane_lsb(r1.y, c2, ma[5], mb[5], q, l);
  cmp_plane_lsb(r1.x, c2, ma[4], mb[4], q, l);
  if (L == 4) {
    const uint32_t z = lop3<0xFE>(r0.x, r0.y, r0.z);
    const uint32_t keep = lop3<0x10>(pend, z, r0.w);  // pending and planes 0-3 all 0
    eq = q & keep;
    lt = l & keep;
    return;
  }
  cmp_plane_lsb(r0.w, c2, ma[3], mb[3], q, l);
  cmp_plane_lsb(r0.z, c2, ma[2], mb[2], q, l);
  cmp_plane_lsb(r0.y, c2, ma[1], mb[1], q, l);
  cmp_plane_lsb(r0.x, c2, ma[0], mb[0], q, l);
  eq = q;
  lt = l & pend;
}

// 8-bit mask of the non-zero nibbles of x (bit g <-> nibble g)
__device__ __forceinline__ uint32_t nibmask8(uint32_t x) {
  x |= x >> 1;
  x |= x >> 2;
  x &= 0x11111111u;
  x = (x | (x >> 3)) & 0x03030303u;
  x = (x | (x >> 6)) & 0x000F000Fu;
  x = (x | (x >> 12)) & 0xFFu;
  return x;
}

}  // namespace gsb
