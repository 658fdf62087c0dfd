// checker_common.cuh -- per-word pieces of the checkerboard sweep shared by the
// shared-memory engine (checker.cu) and the HBM-tiled engine (checker_hbm.cu).
// Bit layout and contract: see checker.cu / DESIGN.md.
#pragma once
#include <cstdint>

#include "gsb_device.cuh"

namespace gsb {

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

// Bit-sliced comparison of the uniforms' top 8 bits with the thresholds, as a
// borrow chain over the planes LSB-first (plane 7 = uniform bit 24 first,
// plane 0 = bit 31 last).  c2 = class -2 sites (threshold K2), other pending
// sites use K4; ma/mb = all-ones iff the plane's bit of K2/K4 is set (per
// sweep, uniform).  lt becomes [u_hi < K_hi] (strict), eq keeps the pending
// sites whose 8 bits all equal K_hi.  3 LOP3 per plane.
__device__ __forceinline__ void cmp_plane_lsb(uint32_t R, uint32_t c2, uint32_t ma, uint32_t mb,
                                              uint32_t &eq, uint32_t &lt) {
  const uint32_t tb = (c2 & ma) | (~c2 & mb);
  lt = (tb & (~R | lt)) | (~tb & ~R & lt);
  eq &= ~(R ^ tb);
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
