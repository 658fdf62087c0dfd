// rscan2.cu -- random-scan engine (kinds *_random_scan), contract v2.
//
// The reference sweep (solvers.py:107-127) visits every site once in a fresh
// uniformly random order and updates it from its current neighbours.  Here
// the order of sweep t is the sites sorted by (priority, id), priorities
// i.i.d. 32-bit Philox values, and a site's acceptance uniform is its own
// Philox value (executable form
// oracle/gsb_oracle.c:trial_rscan).  Any order that visits each site after
// the neighbours that precede it leaves the same spins after every visit, so
// the engine visits by rounds: a site is ready once every preceding
// neighbour has been visited, and all ready sites of a word update with one
// bit-sliced instruction sequence (two ready sites are never neighbours).
// The best-so-far of the sequential priority-order scan is recovered
// exactly at the end of each sweep (below).
//
// Layout (contract words): WPR = ceil(cols / 32) words per row, word
// wi = r*WPR + (c >> 5) holds sites (r, 32k + b) at bit b; padding bits 0.
// Team = one CTA of NW warps per trial (persistent over trials).  A warp
// holds BPW = 32 / WPR row blocks, lane = (block, word column); a lane owns
// one word column of RB (or RB - 1) consecutive rows and keeps every plane of
// those words in registers (slot j = row start + j).  Neighbours:
//   left / right   the same slot of the lanes of the adjacent word columns
//                  (one SHFL per plane; the row wraps from the last column);
//   up / down      slot j -+ 1 of the same lane, or, at the block edges, the
//                  adjacent block's edge row through a shared-memory
//                  exchange (double-buffered, one barrier per round).
// Per sweep:
//   1. priority planes 0..7 (2 Philox blocks per word) to shared memory and,
//      for SA, the acceptance planes A2 / A4 = [u < K(-2)] / [u < K(-4)]
//      (2 blocks: the uniform's top 8 bits compared with the thresholds; a
//      site whose top byte equals K's draws its low 24 bits);
//   2. precedence planes: Pr = right neighbour precedes, Pd = down neighbour
//      precedes (8-plane comparators; equal top bytes compare the low 24
//      bits, then the ids), Pl and Pu from the neighbours' Pr / Pd (the
//      order is strict and total);
//   3. rounds: ready = unvisited & no unvisited preceding neighbour; Delta
//      classes from the 4 positive-term planes; flip = ready & (Delta >= 0 |
//      accepted); slots update in order, so a chain down a lane's rows can
//      advance several levels in one round;
//   4. best-so-far of the sequential scan: each flipped site's Delta at its
//      visit is recomputed from the end-of-sweep spins (a preceding
//      neighbour's final spin, a following neighbour's initial one).  The
//      running cut in priority order is cur0 + the prefix sums of those
//      Deltas.  If cur0 + (sum of positive Deltas) cannot beat best, nothing
//      to do; else the Deltas are binned by their priority's top byte (256
//      buckets: sum, positive sum), and only buckets whose prefix + positive
//      sum can beat best are sorted exactly ((priority, id) order) and
//      scanned.  The snapshot is S0 ^ (flips with key <= the key where the
//      maximum was first reached).
#include <climits>
#include <cstdint>

#include "checker_common.cuh"
#include "gsb_device.cuh"
#include "gsb_internal.h"

namespace gsb {

constexpr uint32_t RS2_TAG = 5u;
constexpr int RS2_CAP = 256;  // events of one candidate bucket sorted at once

struct Rs2Args {
  int rows, cols, n, WPR;
  int NBu, nbig, lastvalid;  // row blocks used, blocks with RB rows, valid bits of the last column
  const int8_t *w;
  const uint64_t *table;
  int sweeps;
  const uint64_t *seeds;
  int T;
  int64_t *best_cut;
  int32_t *sweeps_exec;
  uint8_t *best_bits;
  int nbytes, nstream;  // output bytes per trial, 32-bit words of the staged bitstring
  int *err;
  unsigned long long *stats;  // [0] rounds, [1] gated sweeps, [2] candidate buckets, [3] ties
};

struct Rs2Entry {
  uint32_t key, id;
  int d;
};

// per-CTA shared memory carve-up (sizes from the host, see rs2_smem)
struct Rs2Smem {
  uint4 *planes;     // [RB][NT][2] priority planes 0-3, 4-7 of every slot
  uint4 *ev;         // [RB][NT] flipped sites by Delta at visit: +4, +2, -2, -4
  uint32_t *bs;      // [RB][NT] best snapshot
  uint32_t *s0;      // [RB][NT] spins at the start of the sweep
  uint2 *xtop;       // [2][NT] (S, U) of each lane's first row
  uint2 *xbot;       // [2][NT] (S, U) of each lane's last real row
  uint32_t *xpd;     // [NT] Pd of the last real row (Pu of the block below)
  unsigned long long *bucket;  // [256]
  Rs2Entry *list;    // [2][RS2_CAP]
  uint32_t *stream;  // [nstream] best bitstring staging
  int *red;          // [2][NW][4] reduction scratch
  int *misc;         // [16]
  unsigned long long *mm;  // [NW] minimum-extraction scratch
  int *md;           // [NW]
};

__device__ __forceinline__ uint32_t word_of(const P4 &p, int i) {
  return i == 0 ? p.x : i == 1 ? p.y : i == 2 ? p.z : p.w;
}

// per (trial, wi) Philox precomputation for counters (wi, t, q, tag)
__device__ __forceinline__ PhiloxWord philox_word_tag(uint32_t wi, uint32_t tag, uint32_t k0,
                                                      uint32_t k1, uint32_t &h1z) {
  const uint32_t h0 = __umulhi(kPhiloxM0, wi), l0 = kPhiloxM0 * wi;
  const uint32_t z1 = h0 ^ tag ^ k1;
  h1z = __umulhi(kPhiloxM1, z1);
  return PhiloxWord{l0 ^ (k1 + kPhiloxW1), (kPhiloxM1 * z1) ^ (k0 + 2u * kPhiloxW0)};
}

__device__ __forceinline__ P4 philox_block(const PhiloxWord &pw, uint32_t h1z, uint32_t q,
                                           uint32_t u1, uint32_t v, uint32_t k0, uint32_t k1) {
  uint32_t hi, lo;
  philox_pre(h1z, q, k0, hi, lo);
  return philox10_from2(pw, hi, lo, u1, v, k0, k1);
}

// low 24 bits of the priority (q0 = 2) or uniform (q0 = 12) of site (wi, b)
__device__ __forceinline__ uint32_t rs2_low24(uint32_t wi, uint32_t t, uint32_t q0, int b,
                                              uint32_t k0, uint32_t k1) {
  const P4 o = philox10(P4{wi, t, q0 + (uint32_t)(b >> 2), RS2_TAG}, k0, k1);
  return word_of(o, b & 3) >> 8;
}

// top byte (planes 0..7, plane 0 = MSB) of bit b
__device__ __forceinline__ uint32_t gather8(const uint4 &a, const uint4 &b, int bit) {
  return (((a.x >> bit) & 1u) << 7) | (((a.y >> bit) & 1u) << 6) | (((a.z >> bit) & 1u) << 5) |
         (((a.w >> bit) & 1u) << 4) | (((b.x >> bit) & 1u) << 3) | (((b.y >> bit) & 1u) << 2) |
         (((b.z >> bit) & 1u) << 1) | ((b.w >> bit) & 1u);
}

// LSB-first borrow chain: lt = [a < b] over planes, neq = any plane differs
__device__ __forceinline__ void cmp_step(uint32_t a, uint32_t b, uint32_t &lt, uint32_t &neq) {
  lt = lop3<0x8E>(a, b, lt);    // (~a & b) | (~(a ^ b) & lt)
  neq = lop3<0xBE>(a, b, neq);  // neq | (a ^ b)
}

// [x < y] over the 8 planes (x0..x7 vs y0..y7, plane 0 = MSB) and the tie mask
__device__ __forceinline__ void cmp8(const uint32_t *x, const uint32_t *y, uint32_t &lt,
                                     uint32_t &tie) {
  uint32_t l = 0, ne = 0;
#pragma unroll
  for (int i = 7; i >= 0; i--) cmp_step(x[i], y[i], l, ne);
  lt = l;
  tie = ~ne;
}

template <int NW>
__device__ __forceinline__ void team_sync() {
  if (NW == 1)
    __syncwarp();
  else
    __syncthreads();
}

template <int NW>
__device__ __forceinline__ bool team_any(bool p) {
  if (NW == 1) {
    __syncwarp();
    return __any_sync(0xffffffffu, p);
  }
  return __syncthreads_or(p) != 0;
}

// team sum of up to 4 ints (scratch double-buffered by parity: one barrier)
template <int NW>
__device__ __forceinline__ void team_sum4(int *red, int par, int lane, int warp, int &a, int &b,
                                          int &c, int &d) {
  a = (int)__reduce_add_sync(0xffffffffu, (unsigned)a);
  b = (int)__reduce_add_sync(0xffffffffu, (unsigned)b);
  c = (int)__reduce_add_sync(0xffffffffu, (unsigned)c);
  d = (int)__reduce_add_sync(0xffffffffu, (unsigned)d);
  if (NW == 1) return;
  int *r = red + par * NW * 4;
  if (lane == 0) {
    r[warp * 4] = a;
    r[warp * 4 + 1] = b;
    r[warp * 4 + 2] = c;
    r[warp * 4 + 3] = d;
  }
  __syncthreads();
  a = b = c = d = 0;
#pragma unroll
  for (int i = 0; i < NW; i++) {
    a += r[i * 4];
    b += r[i * 4 + 1];
    c += r[i * 4 + 2];
    d += r[i * 4 + 3];
  }
}

template <int NW, int RB, bool SA>
__global__ void __launch_bounds__(NW * 32) rscan2_kernel(Rs2Args a) {
  constexpr int NT = NW * 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Rs2Smem sm;
  {
    unsigned char *p = smem_raw;
    sm.planes = (uint4 *)p;
    p += sizeof(uint4) * 2 * RB * NT;
    sm.ev = (uint4 *)p;
    p += SA ? sizeof(uint4) * RB * NT : 0;
    sm.bucket = (unsigned long long *)p;
    p += SA ? sizeof(unsigned long long) * 256 : 0;
    sm.list = (Rs2Entry *)p;
    p += SA ? sizeof(Rs2Entry) * 2 * RS2_CAP : 0;
    sm.xtop = (uint2 *)p;
    p += sizeof(uint2) * 2 * NT;
    sm.xbot = (uint2 *)p;
    p += sizeof(uint2) * 2 * NT;
    sm.bs = (uint32_t *)p;
    p += sizeof(uint32_t) * RB * NT;
    sm.s0 = (uint32_t *)p;
    p += sizeof(uint32_t) * RB * NT;
    sm.xpd = (uint32_t *)p;
    p += sizeof(uint32_t) * NT;
    sm.red = (int *)p;
    p += sizeof(int) * 2 * NW * 4;
    sm.misc = (int *)p;
    p += sizeof(int) * 16;
    sm.mm = (unsigned long long *)p;
    p += sizeof(unsigned long long) * NW;
    sm.md = (int *)p;
    p += sizeof(int) * NW;
    p = (unsigned char *)(((uintptr_t)p + 15) & ~(uintptr_t)15);
    sm.stream = (uint32_t *)p;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rows = a.rows, cols = a.cols, WPR = a.WPR;
  const int BPW = 32 / WPR;
  const int rbl = lane / WPR, c = lane - rbl * WPR;
  const int rb = warp * BPW + rbl;
  const bool act = rbl < BPW && rb < a.NBu;
  const int nr = act ? (rb < a.nbig ? RB : RB - 1) : 0;
  const int start = act ? rb * (RB - 1) + min(rb, a.nbig) : 0;
  const bool shortb = nr < RB;  // the last slot is a dummy
  const int vb = c == WPR - 1 ? a.lastvalid : 32;
  const uint32_t V = act ? (vb == 32 ? 0xFFFFFFFFu : (1u << vb) - 1u) : 0u;
  const uint32_t Vlast = shortb ? 0u : V;
  const int cpos = vb - 1;
  const uint32_t Mr = 1u << cpos;
  const int ppos = (c == 0 ? a.lastvalid : 32) - 1;
  const int rsrc = act ? rbl * WPR + (c + 1 == WPR ? 0 : c + 1) : lane;
  const int lsrc = act ? rbl * WPR + (c == 0 ? WPR - 1 : c - 1) : lane;
  auto tid_of = [&](int x) {
    const int w = x / BPW;
    return w * 32 + (x - w * BPW) * WPR + c;
  };
  const int tid_above = act ? tid_of(rb == 0 ? a.NBu - 1 : rb - 1) : tid;
  const int tid_below = act ? tid_of(rb + 1 == a.NBu ? 0 : rb + 1) : tid;
  const int col0 = 32 * c;
  const int down_row_last = act ? (start + nr == rows ? 0 : start + nr) : 0;
  auto vslot = [&](int j) -> uint32_t { return j == RB - 1 ? Vlast : V; };
  auto row_of = [&](int j) { return start + (j < nr ? j : 0); };

  // ---- couplings (instance constants): bit b of N* = weight of that edge < 0
  uint32_t Nr[RB], Nl[RB], Nd[RB], Nu0 = 0;
#pragma unroll
  for (int j = 0; j < RB; j++) {
    uint32_t nrr = 0, nll = 0, ndd = 0;
    if (act && j < nr) {
      const int r = start + j;
      for (int b = 0; b < vb; b++) {
        const int col = col0 + b, v = r * cols + col;
        const int vl = r * cols + (col == 0 ? cols - 1 : col - 1);
        nrr |= (uint32_t)(a.w[2 * v] < 0) << b;
        ndd |= (uint32_t)(a.w[2 * v + 1] < 0) << b;
        nll |= (uint32_t)(a.w[2 * vl] < 0) << b;
      }
    }
    Nr[j] = nrr;
    Nl[j] = nll;
    Nd[j] = ndd;
  }
  if (act) {
    const int ru = start == 0 ? rows - 1 : start - 1;
    for (int b = 0; b < vb; b++) Nu0 |= (uint32_t)(a.w[2 * (ru * cols + col0 + b) + 1] < 0) << b;
  }

  unsigned long long st_rounds = 0, st_gated = 0, st_cand = 0, st_ties = 0;
  int par = 0;  // exchange buffer parity

  // neighbour planes of slot j for the rounds and the cut: up / down of the
  // clean planes X (S, U or F), from the registers or the exchange values
  uint32_t S[RB], U[RB], Pr[RB], Pl[RB], Pd[RB], A2[RB], A4[RB];

  // cut of a clean spin array (right and down edges of the own words)
  auto cut_of = [&](const uint32_t *X, uint32_t xdown) -> int {
    int cc = 0;
#pragma unroll
    for (int j = 0; j < RB; j++) {
      const uint32_t rS = __shfl_sync(0xffffffffu, X[j], rsrc);
      const uint32_t R = (X[j] >> 1) + rS * Mr;
      uint32_t D;
      if (j == RB - 1)
        D = xdown;
      else if (j == RB - 2)
        D = shortb ? xdown : X[j + 1];
      else
        D = X[j + 1];
      const uint32_t vs = vslot(j);
      const uint32_t xr = (X[j] ^ R) & vs, xd = (X[j] ^ D) & vs;
      cc += __popc(xr & ~Nr[j]) - __popc(xr & Nr[j]) + __popc(xd & ~Nd[j]) - __popc(xd & Nd[j]);
    }
    return cc;
  };
  auto last_of = [&](const uint32_t *X) -> uint32_t {
    return RB >= 2 && shortb ? X[RB >= 2 ? RB - 2 : 0] : X[RB - 1];
  };

  for (int trial = blockIdx.x; trial < a.T; trial += gridDim.x) {
    const uint64_t seed = a.seeds[trial];
    const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    // ---- initial spins: bit b of word 0 of Philox(key, (wi, 0, 31, TAG))
#pragma unroll
    for (int j = 0; j < RB; j++) {
      const uint32_t wi = (uint32_t)(row_of(j) * WPR + c);
      const P4 o = philox10(P4{wi, 0u, 31u, RS2_TAG}, k0, k1);
      S[j] = o.x & vslot(j);
      sm.bs[j * NT + tid] = S[j];
    }
    sm.xtop[par * NT + tid] = make_uint2(S[0], 0u);
    team_sync<NW>();
    int cur, best, executed = 0;
    {
      int c0 = cut_of(S, sm.xtop[par * NT + tid_below].x), z1 = 0, z2 = 0, z3 = 0;
      team_sum4<NW>(sm.red, par, lane, warp, c0, z1, z2, z3);
      cur = best = c0;
    }
    par ^= 1;

    for (int t = 0; t < a.sweeps; t++) {
      // ---- per-sweep constants (uniform over the team)
      uint32_t u1q[4], vq[4];
      const uint32_t qs[4] = {0u, 1u, 10u, 11u};
#pragma unroll
      for (int i = 0; i < (SA ? 4 : 2); i++) philox_uni((uint32_t)t, qs[i], k0, k1, u1q[i], vq[i]);
      uint64_t K2f = 0, K4f = 0;
      uint32_t kb2[8], kb4[8];
      if (SA) {
        K2f = a.table[(size_t)t * 4 + 1];
        K4f = a.table[(size_t)t * 4 + 3];
#pragma unroll
        for (int i = 0; i < 8; i++) {
          kb2[i] = (uint32_t)((int32_t)((uint32_t)K2f << i) >> 31);
          kb4[i] = (uint32_t)((int32_t)((uint32_t)K4f << i) >> 31);
        }
      }
      const uint32_t all2 = K2f > 0xFFFFFFFFull ? ~0u : 0u, all4 = K4f > 0xFFFFFFFFull ? ~0u : 0u;

      // ---- 1. priority planes (shared memory) and acceptance planes
#pragma unroll
      for (int j = 0; j < RB; j++) {
        const uint32_t wi = (uint32_t)(row_of(j) * WPR + c);
        uint32_t h1z;
        const PhiloxWord pw = philox_word_tag(wi, RS2_TAG, k0, k1, h1z);
        const P4 p0 = philox_block(pw, h1z, 0u, u1q[0], vq[0], k0, k1);
        const P4 p1 = philox_block(pw, h1z, 1u, u1q[1], vq[1], k0, k1);
        sm.planes[(j * NT + tid) * 2] = make_uint4(p0.x, p0.y, p0.z, p0.w);
        sm.planes[(j * NT + tid) * 2 + 1] = make_uint4(p1.x, p1.y, p1.z, p1.w);
        if (SA) {
          const P4 q0 = philox_block(pw, h1z, 10u, u1q[2], vq[2], k0, k1);
          const P4 q1 = philox_block(pw, h1z, 11u, u1q[3], vq[3], k0, k1);
          const uint32_t up8[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
          uint32_t lt2 = 0, ne2 = 0, lt4 = 0, ne4 = 0;
#pragma unroll
          for (int i = 7; i >= 0; i--) {
            cmp_step(up8[i], kb2[i], lt2, ne2);
            cmp_step(up8[i], kb4[i], lt4, ne4);
          }
          const uint32_t vs = vslot(j);
          uint32_t t2 = ~ne2 & vs & ~all2, t4 = ~ne4 & vs & ~all4;
          uint32_t a2 = lt2 | all2, a4 = lt4 | all4;
          uint32_t tie = t2 | t4;
          while (tie) {  // top byte equal to K's: the low 24 bits decide
            const int b = __ffs(tie) - 1;
            tie &= tie - 1;
            st_ties++;
            const uint32_t lo = rs2_low24(wi, (uint32_t)t, 12u, b, k0, k1);
            a2 |= (uint32_t)(((t2 >> b) & 1u) && lo < ((uint32_t)K2f & 0xFFFFFFu)) << b;
            a4 |= (uint32_t)(((t4 >> b) & 1u) && lo < ((uint32_t)K4f & 0xFFFFFFu)) << b;
          }
          A2[j] = a2;
          A4[j] = a4;
        }
        sm.s0[j * NT + tid] = S[j];
        U[j] = vslot(j);
      }
      team_sync<NW>();

      // ---- 2. precedence planes
#pragma unroll
      for (int j = 0; j < RB; j++) {
        const uint4 pa = sm.planes[(j * NT + tid) * 2], pb = sm.planes[(j * NT + tid) * 2 + 1];
        const uint32_t P[8] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
        const int didx = (j + 1 < nr) ? (j + 1) * NT + tid : tid_below;  // slot 0 of the block below
        const uint4 da = sm.planes[didx * 2], db = sm.planes[didx * 2 + 1];
        const uint32_t D[8] = {da.x, da.y, da.z, da.w, db.x, db.y, db.z, db.w};
        uint32_t R[8];
#pragma unroll
        for (int i = 0; i < 8; i++) {
          const uint32_t x = __shfl_sync(0xffffffffu, P[i], rsrc);
          R[i] = lop3<0xD8>(P[i] >> 1, x * Mr, Mr);  // (P >> 1 & ~Mr) | (x << cpos & Mr)
        }
        uint32_t ltR, tieR, ltD, tieD;
        cmp8(R, P, ltR, tieR);
        cmp8(D, P, ltD, tieD);
        const uint32_t vs = vslot(j);
        tieR &= vs;
        tieD &= vs;
        if (tieR | tieD) {  // equal top bytes (p = 2^-8 per edge): low 24 bits, then ids
          const int r = row_of(j);
          const uint32_t wi = (uint32_t)(r * WPR + c);
          const uint32_t wir = (uint32_t)(r * WPR + (c + 1 == WPR ? 0 : c + 1));
          const int rd = j + 1 < nr ? r + 1 : down_row_last;
          const uint32_t wid = (uint32_t)(rd * WPR + c);
          uint32_t tt = tieR | tieD;
          while (tt) {
            const int b = __ffs(tt) - 1;
            tt &= tt - 1;
            st_ties++;
            const uint32_t me = rs2_low24(wi, (uint32_t)t, 2u, b, k0, k1);
            const int id = r * cols + col0 + b;
            if ((tieR >> b) & 1u) {
              const bool wrapc = b == cpos;
              const uint32_t o = rs2_low24(wrapc ? wir : wi, (uint32_t)t, 2u, wrapc ? 0 : b + 1, k0, k1);
              const int idn = r * cols + (col0 + b + 1 == cols ? 0 : col0 + b + 1);
              const bool prec = o < me || (o == me && idn < id);
              ltR = (ltR & ~(1u << b)) | ((uint32_t)prec << b);
            }
            if ((tieD >> b) & 1u) {
              const uint32_t o = rs2_low24(wid, (uint32_t)t, 2u, b, k0, k1);
              const int idn = rd * cols + col0 + b;
              const bool prec = o < me || (o == me && idn < id);
              ltD = (ltD & ~(1u << b)) | ((uint32_t)prec << b);
            }
          }
        }
        Pr[j] = ltR;
        Pd[j] = ltD;
      }
      // Pl(v) = !Pr(left(v)), Pu(v) = !Pd(up(v))
#pragma unroll
      for (int j = 0; j < RB; j++) {
        const uint32_t x = __shfl_sync(0xffffffffu, Pr[j], lsrc);
        Pl[j] = lop3<0x07>(Pr[j] * 2u, x >> ppos, 1u);  // ~((Pr << 1) | (x >> ppos & 1))
      }
      sm.xpd[tid] = last_of(Pd);
      sm.xtop[par * NT + tid] = make_uint2(S[0], U[0]);
      sm.xbot[par * NT + tid] = make_uint2(last_of(S), last_of(U));
      team_sync<NW>();
      const uint32_t Pu0 = ~sm.xpd[tid_above];

      // ---- 3. rounds
      for (int rr = 0;; rr++) {
        if (rr >= 1 << 16) {
          if (tid == 0) atomicExch(a.err, GSB_EUNSUPPORTED);
          break;
        }
        st_rounds++;
        const uint2 xu = sm.xbot[par * NT + tid_above];  // (S, U) of the row above slot 0
        const uint2 xd = sm.xtop[par * NT + tid_below];  // (S, U) of the row below the last
        uint32_t left = 0;
#pragma unroll
        for (int j = 0; j < RB; j++) {
          const uint32_t s = S[j], u = U[j];
          const uint32_t upS = j == 0 ? xu.x : S[j - 1], upU = j == 0 ? xu.y : U[j - 1];
          uint32_t dnS, dnU;
          if (j == RB - 1) {
            dnS = xd.x;
            dnU = xd.y;
          } else if (j == RB - 2) {
            dnS = shortb ? xd.x : S[j + 1];
            dnU = shortb ? xd.y : U[j + 1];
          } else {
            dnS = S[j + 1];
            dnU = U[j + 1];
          }
          const uint32_t rS = __shfl_sync(0xffffffffu, s, rsrc);
          const uint32_t rU = __shfl_sync(0xffffffffu, u, rsrc);
          const uint32_t lS = __shfl_sync(0xffffffffu, s, lsrc);
          const uint32_t lU = __shfl_sync(0xffffffffu, u, lsrc);
          const uint32_t RS = (s >> 1) + rS * Mr, RU = (u >> 1) + rU * Mr;
          const uint32_t LS = s * 2u + (lS >> ppos), LU = u * 2u + (lU >> ppos);
          uint32_t blk = Pr[j] & RU;
          blk = lop3<0xF8>(blk, Pl[j], LU);  // | (Pl & LU)
          blk = lop3<0xF8>(blk, Pd[j], dnU);
          if (j == 0)
            blk = lop3<0xF8>(blk, Pu0, upU);
          else
            blk = lop3<0xF2>(blk, Pd[j - 1], upU);  // | (~Pd[j-1] & upU)
          const uint32_t ready = u & ~blk;
          const uint32_t ta = lop3<0x69>(s, RS, Nr[j]);
          const uint32_t tb = lop3<0x69>(s, LS, Nl[j]);
          const uint32_t tc = lop3<0x69>(s, upS, j == 0 ? Nu0 : Nd[j - 1]);
          const uint32_t td = lop3<0x69>(s, dnS, Nd[j]);
          const uint32_t s1 = lop3<0x96>(ta, tb, tc), c1 = lop3<0xE8>(ta, tb, tc);
          uint32_t flip;
          if (SA) {
            const uint32_t ge2 = lop3<0xF8>(c1, s1, td);         // >= 2 positive terms
            const uint32_t mux = lop3<0xCA>(s1 ^ td, A2[j], A4[j]);  // 1 positive: A2, 0: A4
            flip = lop3<0xE0>(ready, ge2, mux);
          } else {
            flip = ready & lop3<0xE0>(c1, s1, td);  // >= 3 positive terms
          }
          S[j] = s ^ flip;
          U[j] = u ^ ready;
          left |= U[j];
        }
        par ^= 1;
        sm.xtop[par * NT + tid] = make_uint2(S[0], U[0]);
        sm.xbot[par * NT + tid] = make_uint2(last_of(S), last_of(U));
        if (!team_any<NW>(left != 0)) break;
      }

      // ---- 4. Delta of every flip at its visit, sums, best-so-far
      // F = flips of the sweep; exchange (S, F) of the edge rows
      uint32_t S0[RB];  // holds F from here on
#pragma unroll
      for (int j = 0; j < RB; j++) S0[j] = sm.s0[j * NT + tid] ^ S[j];
      sm.xtop[par * NT + tid] = make_uint2(S[0], S0[0]);
      sm.xbot[par * NT + tid] = make_uint2(last_of(S), last_of(S0));
      team_sync<NW>();
      int dsum = 0, ppos_sum = 0, anyf = 0, z = 0;
      {
        const uint2 xu = sm.xbot[par * NT + tid_above];
        const uint2 xd = sm.xtop[par * NT + tid_below];
#pragma unroll
        for (int j = 0; j < RB; j++) {
          const uint32_t s = S[j], F = S0[j], s0 = s ^ F;
          const uint32_t upS = j == 0 ? xu.x : S[j - 1], upF = j == 0 ? xu.y : S0[j - 1];
          uint32_t dnS, dnF;
          if (j == RB - 1) {
            dnS = xd.x;
            dnF = xd.y;
          } else if (j == RB - 2) {
            dnS = shortb ? xd.x : S[j + 1];
            dnF = shortb ? xd.y : S0[j + 1];
          } else {
            dnS = S[j + 1];
            dnF = S0[j + 1];
          }
          const uint32_t rS = __shfl_sync(0xffffffffu, s, rsrc);
          const uint32_t rF = __shfl_sync(0xffffffffu, F, rsrc);
          const uint32_t lS = __shfl_sync(0xffffffffu, s, lsrc);
          const uint32_t lF = __shfl_sync(0xffffffffu, F, lsrc);
          const uint32_t RS = (s >> 1) + rS * Mr, RF = (F >> 1) + rF * Mr;
          const uint32_t LS = s * 2u + (lS >> ppos), LF = F * 2u + (lF >> ppos);
          if (!SA) {
            anyf |= F != 0;
            // greedy flips have Delta > 0 only: the sum still follows the same formula
          }
          // neighbour spin at the visit: final if it precedes, else initial
          const uint32_t xr = lop3<0xB4>(RS, RF, Pr[j]);  // S ^ (F & ~P)
          const uint32_t xl = lop3<0xB4>(LS, LF, Pl[j]);
          const uint32_t xdn = lop3<0xB4>(dnS, dnF, Pd[j]);
          const uint32_t xup = j == 0 ? lop3<0xB4>(upS, upF, Pu0) : (upS ^ (upF & Pd[j - 1]));
          const uint32_t ta = lop3<0x69>(s0, xr, Nr[j]);
          const uint32_t tb = lop3<0x69>(s0, xl, Nl[j]);
          const uint32_t tc = lop3<0x69>(s0, xup, j == 0 ? Nu0 : Nd[j - 1]);
          const uint32_t td = lop3<0x69>(s0, xdn, Nd[j]);
          const uint32_t s1 = lop3<0x96>(ta, tb, tc), c1 = lop3<0xE8>(ta, tb, tc);
          const uint32_t k4 = lop3<0x80>(c1, s1, td) & F, k3 = lop3<0x60>(c1, s1, td) & F;
          const uint32_t k1 = lop3<0x06>(c1, s1, td) & F, k0m = lop3<0x01>(c1, s1, td) & F;
          const int n4 = __popc(k4), n3 = __popc(k3);
          dsum += 4 * n4 + 2 * n3 - 2 * __popc(k1) - 4 * __popc(k0m);
          ppos_sum += 4 * n4 + 2 * n3;
          if (SA) sm.ev[j * NT + tid] = make_uint4(k4, k3, k1, k0m);
        }
      }
      team_sum4<NW>(sm.red, par, lane, warp, dsum, ppos_sum, anyf, z);
      par ^= 1;
      const int cur0 = cur;
      cur += dsum;
      if (!SA) {
        executed = t + 1;
        if (anyf == 0) break;
        // Delta > 0 flips only: the cut rises monotonically, the best is the
        // end-of-sweep state
        best = cur;
#pragma unroll
        for (int j = 0; j < RB; j++) sm.bs[j * NT + tid] = S[j];
        continue;
      }
      executed = t + 1;
      if (cur0 + ppos_sum <= best) continue;

      // ---- 4b. exact best-so-far in (priority, id) order
      st_gated++;
      for (int i = tid; i < 256; i += NT) sm.bucket[i] = 0ull;
      team_sync<NW>();
#pragma unroll
      for (int j = 0; j < RB; j++) {
        const uint4 e = sm.ev[j * NT + tid];
        uint32_t any = e.x | e.y | e.z | e.w;
        if (!any) continue;
        const uint4 pa = sm.planes[(j * NT + tid) * 2], pb = sm.planes[(j * NT + tid) * 2 + 1];
        while (any) {
          const int b = __ffs(any) - 1;
          any &= any - 1;
          const uint32_t key8 = gather8(pa, pb, b);
          const int d = ((e.x >> b) & 1u) ? 4 : ((e.y >> b) & 1u) ? 2 : ((e.z >> b) & 1u) ? -2 : -4;
          atomicAdd(&sm.bucket[key8],
                    ((unsigned long long)(d > 0 ? d : 0) << 32) + (unsigned long long)(long long)d);
        }
      }
      team_sync<NW>();
      // candidate buckets (warp 0): prefix C_b = cur0 + sum of the buckets before b
      if (warp == 0) {
        int sb[8], pbk[8], tot = 0;
#pragma unroll
        for (int i = 0; i < 8; i++) {
          const unsigned long long x = sm.bucket[lane * 8 + i];
          sb[i] = (int)(uint32_t)x;
          pbk[i] = (int)((long long)(x - (unsigned long long)(long long)sb[i]) >> 32);
          tot += sb[i];
        }
        int incl = tot;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl += y;
        }
        int run = cur0 + incl - tot;
        uint32_t cm = 0;
        int cbase[8];
#pragma unroll
        for (int i = 0; i < 8; i++) {
          cbase[i] = run;
          if (run + pbk[i] > best) cm |= 1u << i;
          run += sb[i];
        }
        // candidate list in bucket order: (bucket, C_b, P_b)
        const int cnt = __popc(cm);
        int off = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, off, o);
          if (lane >= o) off += y;
        }
        off -= cnt;
        int k = 0;
#pragma unroll
        for (int i = 0; i < 8; i++)
          if ((cm >> i) & 1u) {
            Rs2Entry *L = sm.list + RS2_CAP;  // second half: candidate table
            if (off + k < RS2_CAP) L[off + k] = Rs2Entry{(uint32_t)(lane * 8 + i), (uint32_t)cbase[i], pbk[i]};
            k++;
          }
        const int ncand = __shfl_sync(0xffffffffu, off + cnt, 31);
        if (lane == 0) sm.misc[0] = ncand;
      }
      team_sync<NW>();
      const int ncand = sm.misc[0];
      st_cand += ncand;
      uint32_t kstar = 0, idstar = 0;
      bool improved = false;
      for (int ci = 0; ci < ncand; ci++) {
        const Rs2Entry ce = sm.list[RS2_CAP + ci];
        const uint32_t bkt = ce.key;
        const int Cb = (int)ce.id, Pb = ce.d;
        if (Cb + Pb <= best) continue;  // best rose in an earlier bucket
        // gather the bucket's events with their full keys
        if (tid == 0) sm.misc[1] = 0;
        team_sync<NW>();
        const uint32_t bm[8] = {(bkt & 0x80u) ? ~0u : 0u, (bkt & 0x40u) ? ~0u : 0u,
                                (bkt & 0x20u) ? ~0u : 0u, (bkt & 0x10u) ? ~0u : 0u,
                                (bkt & 0x08u) ? ~0u : 0u, (bkt & 0x04u) ? ~0u : 0u,
                                (bkt & 0x02u) ? ~0u : 0u, (bkt & 0x01u) ? ~0u : 0u};
#pragma unroll
        for (int j = 0; j < RB; j++) {
          const uint4 e = sm.ev[j * NT + tid];
          uint32_t any = e.x | e.y | e.z | e.w;
          if (!any) continue;
          const uint4 pa = sm.planes[(j * NT + tid) * 2], pb = sm.planes[(j * NT + tid) * 2 + 1];
          any &= ~(pa.x ^ bm[0]) & ~(pa.y ^ bm[1]) & ~(pa.z ^ bm[2]) & ~(pa.w ^ bm[3]) &
                 ~(pb.x ^ bm[4]) & ~(pb.y ^ bm[5]) & ~(pb.z ^ bm[6]) & ~(pb.w ^ bm[7]);
          const int r = row_of(j);
          const uint32_t wi = (uint32_t)(r * WPR + c);
          while (any) {
            const int b = __ffs(any) - 1;
            any &= any - 1;
            const int d = ((e.x >> b) & 1u) ? 4 : ((e.y >> b) & 1u) ? 2 : ((e.z >> b) & 1u) ? -2 : -4;
            const uint32_t key = (bkt << 24) | rs2_low24(wi, (uint32_t)t, 2u, b, k0, k1);
            const int slot = atomicAdd(&sm.misc[1], 1);
            if (slot < RS2_CAP) sm.list[slot] = Rs2Entry{key, (uint32_t)(r * cols + col0 + b), d};
          }
        }
        team_sync<NW>();
        const int m = sm.misc[1];
        if (warp == 0) {
          if (m <= RS2_CAP) {
            // rank sort by (key, id) into registers, then an in-order scan
            // in chunks of 32 (warp scan + first argmax)
            Rs2Entry mine[RS2_CAP / 32];
            int rk[RS2_CAP / 32];
#pragma unroll
            for (int q = 0; q < RS2_CAP / 32; q++) {
              const int i = q * 32 + lane;
              rk[q] = -1;
              if (i < m) {
                mine[q] = sm.list[i];
                int r = 0;
                for (int x = 0; x < m; x++) {
                  const Rs2Entry o = sm.list[x];
                  r += (o.key < mine[q].key || (o.key == mine[q].key && o.id < mine[q].id));
                }
                rk[q] = r;
              }
            }
            __syncwarp();
            // write sorted order into the first half (all reads done above)
#pragma unroll
            for (int q = 0; q < RS2_CAP / 32; q++)
              if (rk[q] >= 0) sm.list[rk[q]] = mine[q];
            __syncwarp();
            int carry = Cb, bst = best;
            uint32_t ks = kstar, is = idstar;
            bool imp = false;
            for (int base = 0; base < m; base += 32) {
              const int i = base + lane;
              const Rs2Entry e = i < m ? sm.list[i] : Rs2Entry{0u, 0u, 0};
              int inc = e.d;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
              }
              const int val = carry + inc;
              // max over valid lanes, lowest lane on ties
              int mv = i < m ? val : INT_MIN;
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) mv = max(mv, __shfl_xor_sync(0xffffffffu, mv, o));
              if (mv > bst) {
                const uint32_t hit = __ballot_sync(0xffffffffu, i < m && val == mv);
                const int src = __ffs(hit) - 1;
                bst = mv;
                ks = __shfl_sync(0xffffffffu, e.key, src);
                is = __shfl_sync(0xffffffffu, e.id, src);
                imp = true;
              }
              carry += __shfl_sync(0xffffffffu, inc, 31);
            }
            if (lane == 0) {
              sm.misc[2] = bst;
              sm.misc[3] = (int)ks;
              sm.misc[4] = (int)is;
              sm.misc[5] = imp ? 1 : 0;
            }
          } else if (lane == 0) {
            sm.misc[5] = -1;  // overflow: ordered extraction below
          }
        }
        team_sync<NW>();
        int flag = sm.misc[5];
        if (flag < 0) {
          // more than RS2_CAP events share this top byte: visit them in
          // (key, id) order by repeated team-wide minimum extraction
          int run = Cb, bst = best;
          uint32_t pk = 0, pid = 0;
          bool first = true, imp = false;
          uint32_t ks = kstar, is = idstar;
          for (int it = 0; it < m; it++) {
            unsigned long long mn = ~0ull;
            int md = 0;
#pragma unroll
            for (int j = 0; j < RB; j++) {
              const uint4 e = sm.ev[j * NT + tid];
              uint32_t any = e.x | e.y | e.z | e.w;
              if (!any) continue;
              const uint4 pa = sm.planes[(j * NT + tid) * 2], pb = sm.planes[(j * NT + tid) * 2 + 1];
              any &= ~(pa.x ^ bm[0]) & ~(pa.y ^ bm[1]) & ~(pa.z ^ bm[2]) & ~(pa.w ^ bm[3]) &
                     ~(pb.x ^ bm[4]) & ~(pb.y ^ bm[5]) & ~(pb.z ^ bm[6]) & ~(pb.w ^ bm[7]);
              const int r = row_of(j);
              const uint32_t wi = (uint32_t)(r * WPR + c);
              while (any) {
                const int b = __ffs(any) - 1;
                any &= any - 1;
                const uint32_t key = (bkt << 24) | rs2_low24(wi, (uint32_t)t, 2u, b, k0, k1);
                const uint32_t id = (uint32_t)(r * cols + col0 + b);
                const unsigned long long kk = ((unsigned long long)key << 32) | id;
                const unsigned long long pkk = ((unsigned long long)pk << 32) | pid;
                if ((first || kk > pkk) && kk < mn) {
                  mn = kk;
                  md = ((e.x >> b) & 1u) ? 4 : ((e.y >> b) & 1u) ? 2 : ((e.z >> b) & 1u) ? -2 : -4;
                }
              }
            }
            // team minimum (key, id) and its Delta
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              const unsigned long long y = __shfl_xor_sync(0xffffffffu, mn, o);
              const int yd = __shfl_xor_sync(0xffffffffu, md, o);
              if (y < mn) {
                mn = y;
                md = yd;
              }
            }
            if (NW > 1) {
              if (lane == 0) {
                sm.mm[warp] = mn;
                sm.md[warp] = md;
              }
              __syncthreads();
              mn = ~0ull;
              for (int i = 0; i < NW; i++)
                if (sm.mm[i] < mn) {
                  mn = sm.mm[i];
                  md = sm.md[i];
                }
              __syncthreads();
            }
            pk = (uint32_t)(mn >> 32);
            pid = (uint32_t)mn;
            first = false;
            run += md;
            if (run > bst) {
              bst = run;
              ks = pk;
              is = pid;
              imp = true;
            }
          }
          if (tid == 0) {
            sm.misc[2] = bst;
            sm.misc[3] = (int)ks;
            sm.misc[4] = (int)is;
            sm.misc[5] = imp ? 1 : 0;
          }
          team_sync<NW>();
          flag = sm.misc[5];
        }
        if (flag > 0) {
          best = sm.misc[2];
          kstar = (uint32_t)sm.misc[3];
          idstar = (uint32_t)sm.misc[4];
          improved = true;
        }
        team_sync<NW>();
      }
      if (improved) {
        // snapshot: S0 ^ (flips with (priority, id) <= (kstar, idstar))
        const uint32_t k8 = kstar >> 24, klo = kstar & 0xFFFFFFu;
        uint32_t kb[8];
#pragma unroll
        for (int i = 0; i < 8; i++) kb[i] = ((k8 >> (7 - i)) & 1u) ? ~0u : 0u;
#pragma unroll
        for (int j = 0; j < RB; j++) {
          const uint32_t F = S0[j];
          uint32_t inc = 0;
          if (F) {
            const uint4 pa = sm.planes[(j * NT + tid) * 2], pb = sm.planes[(j * NT + tid) * 2 + 1];
            const uint32_t P[8] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
            uint32_t lt, tie;
            cmp8(P, kb, lt, tie);
            inc = lt & F;
            uint32_t eqm = tie & F;
            const int r = row_of(j);
            const uint32_t wi = (uint32_t)(r * WPR + c);
            while (eqm) {
              const int b = __ffs(eqm) - 1;
              eqm &= eqm - 1;
              const uint32_t lo = rs2_low24(wi, (uint32_t)t, 2u, b, k0, k1);
              const uint32_t id = (uint32_t)(r * cols + col0 + b);
              if (lo < klo || (lo == klo && id <= idstar)) inc |= 1u << b;
            }
          }
          sm.bs[j * NT + tid] = S[j] ^ F ^ inc;
        }
      }
    }

    // ---- integrity guard (solvers.py:132-133) and outputs
    uint32_t B[RB];
#pragma unroll
    for (int j = 0; j < RB; j++) B[j] = sm.bs[j * NT + tid];
    for (int i = tid; i < a.nstream; i += NT) sm.stream[i] = 0u;
    sm.xtop[par * NT + tid] = make_uint2(B[0], 0u);
    team_sync<NW>();
    {
      int cb = cut_of(B, sm.xtop[par * NT + tid_below].x), z1 = 0, z2 = 0, z3 = 0;
      team_sum4<NW>(sm.red, par, lane, warp, cb, z1, z2, z3);
      if (tid == 0) {
        a.best_cut[trial] = best;
        a.sweeps_exec[trial] = executed;
        if (cb != best) atomicExch(a.err, GSB_EINTEGRITY);
      }
    }
    par ^= 1;
    // best spins MSB-first by site id: site v -> stream bit v
#pragma unroll
    for (int j = 0; j < RB; j++) {
      const uint32_t x = __brev(B[j] & vslot(j));
      if (x) {
        const int v0 = row_of(j) * cols + col0;
        const int W = v0 >> 5, sh = v0 & 31;
        atomicOr(&sm.stream[W], x >> sh);
        if (sh && W + 1 < a.nstream) atomicOr(&sm.stream[W + 1], x << (32 - sh));
      }
    }
    team_sync<NW>();
    uint8_t *out = a.best_bits + (size_t)trial * a.nbytes;
    for (int i = tid; i < a.nbytes; i += NT)
      out[i] = (uint8_t)(sm.stream[i >> 2] >> (24 - 8 * (i & 3)));
    team_sync<NW>();
  }
  if (a.stats) {
    st_rounds = tid == 0 ? st_rounds : 0;
    st_gated = tid == 0 ? st_gated : 0;
    st_cand = tid == 0 ? st_cand : 0;
    if (st_rounds) atomicAdd(&a.stats[0], st_rounds);
    if (st_gated) atomicAdd(&a.stats[1], st_gated);
    if (st_cand) atomicAdd(&a.stats[2], st_cand);
    if (st_ties) atomicAdd(&a.stats[3], st_ties);
  }
}

// ------------------------------------------------------------------ host
struct Rs2Shape {
  int NW, RB, NBu, nbig;
};

static size_t rs2_smem(int NW, int RB, bool sa, int nstream) {
  const size_t NT = (size_t)NW * 32;
  size_t b = sizeof(uint4) * 2 * RB * NT;
  if (sa) b += sizeof(uint4) * RB * NT + 8 * 256 + sizeof(Rs2Entry) * 2 * RS2_CAP;
  b += sizeof(uint2) * 4 * NT + sizeof(uint32_t) * 2 * RB * NT + sizeof(uint32_t) * NT;
  b += sizeof(int) * (2 * NW * 4 + 16) + (sizeof(unsigned long long) + sizeof(int)) * NW;
  b = align_up(b, 16) + sizeof(uint32_t) * (size_t)nstream;
  return align_up(b, 16);
}

// row-block counts with blocks of RB or RB - 1 rows
static bool rs2_blocks(int rows, int RB, int maxblocks, int &NBu, int &nbig) {
  for (int nb = (rows + RB - 1) / RB; nb <= maxblocks; nb++) {
    if (RB == 1) {
      if (nb == rows) {
        NBu = nb;
        nbig = nb;
        return true;
      }
      continue;
    }
    const int big = rows - nb * (RB - 1);  // blocks with RB rows
    if (big >= 1 && big <= nb) {
      NBu = nb;
      nbig = big;
      return true;
    }
    if (big < 1) break;
  }
  return false;
}

static const int kRbSet[] = {1, 2, 4, 7, 10, 13};
static const int kNwSet[] = {1, 2, 4};

// Team shape (NW warps, RB rows per lane): minimise the warp-slots a trial
// occupies (NW * RB, +15 % per extra warp for the CTA barriers) over the
// fraction of the SMs' warp slots the batch fills (8 per SM).
static bool rs2_shape(int rows, int cols, int T, int nsm, Rs2Shape &sh) {
  const int WPR = (cols + 31) / 32;
  if (WPR > 32) return false;
  const int BPW = 32 / WPR;
  bool found = false;
  double bestcost = 0;
  for (int nw : kNwSet) {
    for (int RB : kRbSet) {
      int NBu, nbig;
      if (!rs2_blocks(rows, RB, nw * BPW, NBu, nbig)) continue;
      const double warps_total = (double)T * nw;
      const double fill = warps_total >= nsm * 8.0 ? 1.0 : warps_total / (nsm * 8.0);
      const double cost = (double)RB * nw * (1.0 + 0.15 * (nw - 1)) / fill;
      if (!found || cost < bestcost - 1e-9) {
        found = true;
        bestcost = cost;
        sh = Rs2Shape{nw, RB, NBu, nbig};
      }
    }
  }
  return found;
}

bool rscan2_fits(int rows, int cols) {
  Rs2Shape sh;
  if (rows < 3 || cols < 3) return false;
  return rs2_shape(rows, cols, 1 << 20, 148, sh);
}

bool rscan2_shape(int rows, int cols, int T, int *nw, int *rb) {
  Rs2Shape sh;
  if (rows < 3 || cols < 3 || T < 1 || !rs2_shape(rows, cols, T, num_sms(), sh)) return false;
  *nw = sh.NW;
  *rb = sh.RB;
  return true;
}

template <int NW, int RB>
static int rs2_launch(Rs2Args &a, bool sa, cudaStream_t stream) {
  const size_t smem = rs2_smem(NW, RB, sa, a.nstream);
  auto kern = sa ? rscan2_kernel<NW, RB, true> : rscan2_kernel<NW, RB, false>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return set_error(GSB_ECUDA, "cudaFuncSetAttribute failed (random-scan kernel)");
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NW * 32, smem) != cudaSuccess ||
      per_sm < 1)
    return set_error(GSB_ECUDA, "random-scan kernel does not fit on an SM");
  long long grid = (long long)num_sms() * per_sm;
  if (grid > a.T) grid = a.T;
  kern<<<(int)grid, NW * 32, smem, stream>>>(a);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(GSB_ECUDA, cudaGetErrorString(e));
  return GSB_OK;
}

int rscan2_run(int rows, int cols, const int8_t *w_dev, int kind, int sweeps,
               const uint64_t *table, const uint64_t *seeds, int T, int64_t *best_cut,
               int32_t *sweeps_exec, uint8_t *best_bits, int *err_ws,
               unsigned long long *stats, cudaStream_t stream) {
  Rs2Shape sh;
  if (rows < 3 || cols < 3 || !rs2_shape(rows, cols, T, num_sms(), sh))
    return set_error(GSB_EUNSUPPORTED, "torus too large for the random-scan engine");
  Rs2Args a;
  a.rows = rows;
  a.cols = cols;
  a.n = rows * cols;
  a.WPR = (cols + 31) / 32;
  a.NBu = sh.NBu;
  a.nbig = sh.nbig;
  a.lastvalid = cols - 32 * (a.WPR - 1);
  a.w = w_dev;
  a.table = table;
  a.sweeps = sweeps;
  a.seeds = seeds;
  a.T = T;
  a.best_cut = best_cut;
  a.sweeps_exec = sweeps_exec;
  a.best_bits = best_bits;
  a.nbytes = (a.n + 7) / 8;
  a.nstream = (a.n + 31) / 32;
  a.err = err_ws;
  a.stats = stats;
  const bool sa = kind == GSB_ANNEALING;
#define RS2_CASE(nw, rb) \
  if (sh.NW == nw && sh.RB == rb) return rs2_launch<nw, rb>(a, sa, stream);
#define RS2_NW(nw) RS2_CASE(nw, 1) RS2_CASE(nw, 2) RS2_CASE(nw, 4) RS2_CASE(nw, 7) RS2_CASE(nw, 10) RS2_CASE(nw, 13)
  RS2_NW(1)
  RS2_NW(2)
  RS2_NW(4)
#undef RS2_NW
#undef RS2_CASE
  return set_error(GSB_EUNSUPPORTED, "no random-scan kernel for this team shape");
}

}  // namespace gsb
