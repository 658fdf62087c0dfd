// rscan2_kernel.cuh -- random-scan engine (kinds *_random_scan), contract v2:
// the kernel template.  Host side and shape selection: rscan2.cu; the
// instantiations are spread over rscan2_nw{1,2,4,7,8,9,13}.cu to compile in parallel.
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
// exactly at the end of each sweep (step 4b).
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
//                  exchange (one 64-bit (S, U) word per lane and edge row,
//                  stale-tolerant; one team barrier per round).
// Per sweep:
//   1. priority planes 0..7 (2 Philox blocks per word) to shared memory and,
//      for SA, the acceptance planes A2 / A4 = [u < K(-2)] / [u < K(-4)]
//      (2 blocks: the uniform's top 8 bits compared with the thresholds);
//   2. precedence planes: Pr = right neighbour precedes, Pd = down neighbour
//      precedes (8-plane comparators), Pl and Pu from the neighbours' Pr / Pd
//      (the order is strict and total);
//   2b. ties: a site whose uniform's top byte equals a threshold's, or whose
//      priority's top byte equals a neighbour's (2^-8 per comparison), is
//      decided by the low 24 bits (one Philox block per site), then the ids.
//      Ties are queued in shared memory and shared out over the whole team
//      (a lane deciding its own ties serialises a warp on ~every word);
//   3. rounds: ready = unvisited & no unvisited preceding neighbour; Delta
//      classes from the 4 positive-term planes; flip = ready & (Delta >= 0 |
//      accepted); slots update in order, so a chain down a lane's rows can
//      advance several levels in one round.  The rounds are bound by the ALU
//      pipe (LOP3/SHF), so shifts by powers of two and additions of disjoint
//      bit sets are multiply-adds with multipliers the compiler cannot fold
//      (kernel arguments m_one, m_two, m_neg, m_last): they issue on the
//      otherwise idle FMA pipe;
//   4. Delta of every flip at its visit, recomputed from the end-of-sweep
//      spins (a preceding neighbour's final spin, a following neighbour's
//      initial one); the running cut in priority order is cur0 + the prefix
//      sums of those Deltas.  If cur0 + (sum of positive Deltas) cannot beat
//      best, nothing to do; else
//   4b. the Deltas are binned by their priority's top byte (256 buckets: sum,
//      positive sum).  With E = the largest bucket-end value (an achieved
//      value), only buckets whose start + positive sum reaches
//      max(best + 1, E) can hold the first maximum; their events are gathered
//      with full keys in one pass, sorted by (priority, id) and scanned.  The
//      snapshot is S0 ^ (flips with key <= the key of the first maximum).
#pragma once
#include <climits>
#include <cstdint>

#include "checker_common.cuh"
#include "gsb_device.cuh"
#include "gsb_internal.h"

namespace gsb {

#ifndef RS2_RPB
#define RS2_RPB 1  // rounds between team barriers (step 3); 2-6 measured equal or slower
#endif
constexpr uint32_t RS2_TAG = 5u;
constexpr int RS2_CAP = 256;  // events sorted at once in step 4b

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
  int tqcap;            // tie queue capacity (items)
  int lcap;             // events sorted at once in step 4b (<= RS2_CAP; smaller in tests)
  // multipliers the compiler cannot fold (1, 2, 0xFFFFFFFF, 1 << (lastvalid - 1)): the
  // rounds are bound by the ALU pipe, so additions of disjoint bit sets and
  // shifts by these are written as multiply-adds, which issue on the FMA pipe
  uint32_t m_one, m_two, m_neg, m_last;
  // sweep slices (annealing, more trials than resident teams): the schedule is
  // cut into nslice pieces of slice_len sweeps and the teams draw (slice, trial)
  // items slice-major from sl_ctr, so every SM keeps its full set of resident
  // teams until the work runs out instead of ending on a part-filled wave.  A
  // trial's spins, best snapshot and cuts wait in sl_state between its slices;
  // sl_flag[trial] = slices finished.  Greedy launches draw whole trials (nslice == 1).
  int nslice, slice_len, sl_shift;
  int dynamic;  // items drawn from sl_ctr (more trials than teams); else strided over the grid
  uint32_t *sl_ctr, *sl_flag, *sl_state;
  int *err;
  // [0] rounds, [1] gated sweeps, [2] candidate buckets, [3] ties (queued or inline),
  // [4..9] cycles per phase (GSB_RS2_PROF builds)
  unsigned long long *stats;
};

// bytes of the per-CTA region shared by the tie queue (steps 1-2b), the
// bucket tables and event list (step 4b) and the output staging (trial end)
__host__ __device__ inline size_t rs2_union_bytes(int tqcap, int nstream) {
  size_t b = 1024 + 1024 + 8 * (size_t)RS2_CAP + 256;  // hist, cb, list, candidate ids
  if (b < 8 * (size_t)tqcap) b = 8 * (size_t)tqcap;
  if (b < 4 * (size_t)nstream) b = 4 * (size_t)nstream;
  return (b + 15) & ~(size_t)15;
}

__host__ __device__ inline size_t rs2_smem_bytes(int NW, int RB, int tqcap, int nstream) {
  const size_t NT = (size_t)NW * 32;
  size_t b = 16 * 2 * RB * NT;  // planes
  b += 16 * RB * NT;            // ev / tie fix-ups
  b += 4 * RB * NT;             // best snapshot
  b += 8 * 4 * NT;              // xtop, xbot (double-buffered)
  b += 4 * NT;                  // xpd
  b += 8 * NW + 8 * NW;         // mm, md (padded)
  b += 4 * (2 * NW * 4 + 16);   // red, misc
  b = (b + 15) & ~(size_t)15;
  return b + rs2_union_bytes(tqcap, nstream);
}

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

// top byte (planes 0..7, plane 0 = MSB) of bit b: each plane's bit is moved to
// bit 31 and funnel-shifted into the key (2 SHF per plane).  (As multiply-adds
// on the FMA pipe -- 3 per plane, one dependent chain -- it measured 3 % slower.)
__device__ __forceinline__ uint32_t gather8(const uint4 &a, const uint4 &b, int bit) {
  const int sh = 31 - bit;
  uint32_t r = 0;
  r = __funnelshift_l(a.x << sh, r, 1);
  r = __funnelshift_l(a.y << sh, r, 1);
  r = __funnelshift_l(a.z << sh, r, 1);
  r = __funnelshift_l(a.w << sh, r, 1);
  r = __funnelshift_l(b.x << sh, r, 1);
  r = __funnelshift_l(b.y << sh, r, 1);
  r = __funnelshift_l(b.z << sh, r, 1);
  r = __funnelshift_l(b.w << sh, r, 1);
  return r;
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

// ---- TMA bulk copy global -> shared, completion on an mbarrier (prologue:
// the instance's couplings are staged once per CTA)
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// flag hand-over between teams (sweep slices): release store / acquire load at GPU scope
__device__ __forceinline__ void st_release_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void tma_bulk_load(void *dst_smem, const void *src_gmem, uint32_t bytes,
                                              unsigned long long *mbar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(mbar))
      : "memory");
}

__device__ __forceinline__ void mbar_init(unsigned long long *mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long *mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@p bra DONE_%=;\n\tbra WAIT_%=;\n\tDONE_%=:\n\t}" ::"r"(smem_u32(mbar)),
      "r"(parity)
      : "memory");
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

// ---- ties (step 2b).  Item: a = me | nb << 16 with me / nb = wi | bit << 11
// (wi < 2^11: rows * WPR <= 8 warps * 32 lanes * 7 rows), b = fix index |
// kind << 12 | flags << 14; kind 0 = acceptance (flags: bit 0 = A2 ties, bit
// 1 = A4 ties), 1 = right neighbour, 2 = down neighbour.  The decision is
// OR-ed into the owner's fix-up word: .x A2, .y A4, .z Pr, .w Pd.
struct Rs2Tie {
  uint32_t t, k0, k1, K2lo, K4lo;
  int WPR, cols;
};

__device__ __forceinline__ void rs2_tie_resolve(uint2 it, const Rs2Tie &c, uint32_t *fix) {
  const uint32_t wi = it.x & 0x7FFu, b = (it.x >> 11) & 31u;
  const uint32_t kind = (it.y >> 12) & 3u, flags = it.y >> 14;
  uint32_t *f = fix + 4 * (it.y & 0xFFFu);
  if (kind == 0) {
    const uint32_t lo = rs2_low24(wi, c.t, 12u, (int)b, c.k0, c.k1);
    if ((flags & 1u) && lo < c.K2lo) atomicOr(f + 0, 1u << b);
    if ((flags & 2u) && lo < c.K4lo) atomicOr(f + 1, 1u << b);
    return;
  }
  const uint32_t win = (it.x >> 16) & 0x7FFu, bn = it.x >> 27;
  const P4 om = philox10(P4{wi, c.t, 2u + (b >> 2), RS2_TAG}, c.k0, c.k1);
  const uint32_t me = word_of(om, b & 3) >> 8;
  uint32_t o;
  if (win == wi && (bn >> 2) == (b >> 2)) {
    o = word_of(om, bn & 3) >> 8;
  } else {
    o = rs2_low24(win, c.t, 2u, (int)bn, c.k0, c.k1);
  }
  bool prec = o < me;
  if (o == me) {  // 2^-32 per edge: the ids decide
    const int r = (int)wi / c.WPR, rn = (int)win / c.WPR;
    const int id = r * c.cols + 32 * ((int)wi - r * c.WPR) + (int)b;
    const int idn = rn * c.cols + 32 * ((int)win - rn * c.WPR) + (int)bn;
    prec = idn < id;
  }
  if (prec) atomicOr(f + (kind == 1 ? 2 : 3), 1u << b);
}


// register cap: 14 resident warps per SM (144 registers) for teams of 1-2
// warps, 16 (128) for larger teams unless 7 rows per lane need more; 8 warps
// x 2 rows run 24 warps per SM at 80 registers, and 7 x 2 (config 2) four
// teams = 28 warps per SM at 72: with sweep slices keeping every seat busy the
// fourth team is worth +7 % over three at 80 (before the slices it was not;
// 96 for 4 x 5, 7 x 3, 7 x 4 buys a team more per SM and loses 4-13 % to
// spills: profiles/r02_rscan2_regcaps.txt, r02_rscan2_regcaps_sliced.txt)
constexpr int rs2_max_regs(int NW, int RB) {
  return NW <= 2 ? 144
         : NW == 4 ? (RB >= 7 ? 168 : 128)
         : RB >= 7 ? 255
         : RB == 2 ? (NW == 8 ? 80 : 72)
                   : 128;  // 7 warps and more
}

template <int NW, int RB, bool SA>
__global__ void __maxnreg__(rs2_max_regs(NW, RB)) rscan2_kernel(Rs2Args a) {
  constexpr int NT = NW * 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // ---- shared memory carve-up (sizes: rs2_smem_bytes)
  uint4 *const s_planes = (uint4 *)smem_raw;             // [RB][NT][2] priority planes 0-3, 4-7
  uint4 *const s_ev = s_planes + 2 * RB * NT;            // [RB][NT] flips by Delta: +4, +2, -2, -4
  uint32_t *const s_fix = (uint32_t *)s_ev;              //   (steps 1-2b: tie decisions)
  uint32_t *const s_bs = (uint32_t *)(s_ev + RB * NT);   // [RB][NT] best snapshot
  uint2 *const s_xtop = (uint2 *)(s_bs + RB * NT);       // [2][NT] (S, U) of each lane's first row
  uint2 *const s_xbot = s_xtop + 2 * NT;                 // [2][NT] ... last real row
  uint32_t *const s_xpd = (uint32_t *)(s_xbot + 2 * NT);  // [NT] Pd of the last real row
  unsigned long long *const s_mm = (unsigned long long *)(s_xpd + NT);  // [NW]
  int *const s_md = (int *)(s_mm + NW);                  // [2 * NW] (padded)
  int *const s_red = s_md + 2 * NW;                      // [2][NW][4]
  int *const s_misc = s_red + 2 * NW * 4;                // [16]
  unsigned char *const s_un =
      (unsigned char *)(((uintptr_t)(s_misc + 16) + 15) & ~(uintptr_t)15);
  uint32_t *const s_hist = (uint32_t *)s_un;             // [256] (pos << 16) + sum per bucket
  int *const s_cb = (int *)(s_un + 1024);                // [256] running cut at each bucket start
  unsigned long long *const s_list = (unsigned long long *)(s_un + 2048);  // [RS2_CAP]
  uint8_t *const s_cl = (uint8_t *)(s_un + 2048 + 8 * RS2_CAP);           // [256] candidates
  uint2 *const s_tq = (uint2 *)s_un;                     // [tqcap] tie queue
  uint32_t *const s_stream = (uint32_t *)s_un;           // [nstream] best bitstring staging
  // s_misc: [0] candidates, [1] list count, [2] best, [3] key*, [4] id*, [5] flag,
  //         [6] tie queue count, [7] E (largest bucket-end value)

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
  const uint32_t Mr = c == WPR - 1 ? a.m_last : 0x80000000u;  // 1 << cpos, opaque (see m_last)
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

  // ---- couplings (instance constants): bit b of N* = weight of that edge < 0.
  // The int8 array w[2n] is staged in shared memory by one TMA bulk copy when
  // it fits the plane / event regions (free before the first trial) and its
  // size is a multiple of 16 bytes; else the planes are read from global memory.
  __shared__ __align__(8) unsigned long long s_mbar;
  const int8_t *wsrc = a.w;
  {
    const uint32_t wbytes = 2u * (uint32_t)a.n;
    if (wbytes % 16u == 0u && wbytes <= (uint32_t)(48 * RB * NT) &&
        ((uintptr_t)a.w & 15u) == 0) {  // team-uniform
      if (tid == 0) mbar_init(&s_mbar, 1);
      team_sync<NW>();
      if (tid == 0) tma_bulk_load(smem_raw, a.w, wbytes, &s_mbar);
      mbar_wait(&s_mbar, 0);
      wsrc = (const int8_t *)smem_raw;
    }
  }
  uint32_t Nr[RB], Nl[RB], Nd[RB], Nu0 = 0;
#pragma unroll
  for (int j = 0; j < RB; j++) {
    uint32_t nrr = 0, nll = 0, ndd = 0;
    if (act && j < nr) {
      const int r = start + j;
      for (int b = 0; b < vb; b++) {
        const int col = col0 + b, v = r * cols + col;
        const int vl = r * cols + (col == 0 ? cols - 1 : col - 1);
        nrr |= (uint32_t)(wsrc[2 * v] < 0) << b;
        ndd |= (uint32_t)(wsrc[2 * v + 1] < 0) << b;
        nll |= (uint32_t)(wsrc[2 * vl] < 0) << b;
      }
    }
    Nr[j] = nrr;
    Nl[j] = nll;
    Nd[j] = ndd;
  }
  if (act) {
    const int ru = start == 0 ? rows - 1 : start - 1;
    for (int b = 0; b < vb; b++) Nu0 |= (uint32_t)(wsrc[2 * (ru * cols + col0 + b) + 1] < 0) << b;
  }

    team_sync<NW>();  // the staged couplings are consumed: the regions are free

unsigned long long st_rounds = 0, st_gated = 0, st_cand = 0, st_ties = 0;
#ifdef GSB_RS2_PROF
  long long pf[6] = {0, 0, 0, 0, 0, 0}, pf_t = clock64();
#define RS2_TICK(i)                   \
  do {                                \
    const long long now_ = clock64(); \
    pf[i] += now_ - pf_t;             \
    pf_t = now_;                      \
  } while (0)
#else
#define RS2_TICK(i)
#endif
  int par = 0;  // exchange buffer parity

  // S spins, U unvisited, F flips of the sweep, P* precedence, A* acceptance
  uint32_t S[RB], U[RB], F[RB], Pr[RB], Pl[RB], Pd[RB], A2[RB], A4[RB];

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

  if (tid == 0) s_misc[6] = 0;

  // items: (slice << sl_shift) + trial, 2^sl_shift >= T.  `item` stays a warp-uniform
  // value for the compiler (block index, kernel arguments, a warp reduction),
  // so the sweep loop's bounds and branches do
  const int nitems = a.nslice == 1 ? a.T : a.nslice << a.sl_shift;
  const int swords = 4 + 2 * rows * WPR;  // sl_state words per trial
  auto next_item = [&](int item) -> int {
    if (!a.dynamic) return item + (int)gridDim.x;
    if (tid == 0) s_misc[8] = (int)(atomicAdd(a.sl_ctr, 1u) + gridDim.x);
    team_sync<NW>();
    return (int)__reduce_max_sync(0xffffffffu, (unsigned)s_misc[8]);
  };
  for (int item = blockIdx.x; item < nitems;) {
    const int slice = item >> a.sl_shift;
    const int trial = item - (slice << a.sl_shift);
    if (trial >= a.T) {  // padding of the item space
      team_sync<NW>();   // s_misc[8] is read by every warp before the next draw
      item = next_item(item);
      continue;
    }
    const int t_begin = slice * a.slice_len;
    const int t_end = slice + 1 == a.nslice ? a.sweeps : t_begin + a.slice_len;
    const uint64_t seed = a.seeds[trial];
    const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    int cur, best, executed = 0;
    if (slice == 0) {
      // ---- initial spins: bit b of word 0 of Philox(key, (wi, 0, 31, TAG))
#pragma unroll
      for (int j = 0; j < RB; j++) {
        const uint32_t wi = (uint32_t)(row_of(j) * WPR + c);
        const P4 o = philox10(P4{wi, 0u, 31u, RS2_TAG}, k0, k1);
        S[j] = o.x & vslot(j);
        s_bs[j * NT + tid] = S[j];
      }
      s_xtop[par * NT + tid] = make_uint2(S[0], 0u);
      team_sync<NW>();
      {
        int c0 = cut_of(S, s_xtop[par * NT + tid_below].x), z1 = 0, z2 = 0, z3 = 0;
        team_sum4<NW>(s_red, par, lane, warp, c0, z1, z2, z3);
        cur = best = c0;
      }
      par ^= 1;
    } else {
      // ---- resume: the trial's previous slice (any team) has published its state
      // (every warp polls for itself: one broadcast load, exit by vote)
      while (!__all_sync(0xffffffffu, ld_acquire_u32(a.sl_flag + trial) >= (uint32_t)slice))
        __nanosleep(256);
      const uint32_t *st = a.sl_state + (size_t)trial * swords;
      // (broadcast through shared memory like team_sum4's results: the sweep
      // loop branches on cur and best, and read per thread from global memory
      // the compiler treats them as divergent values -- the branches and all the
      // code behind them leave the uniform datapath: +46 % instructions, configs
      // 3 and 4 a third slower)
      if (tid == 0) {
        s_misc[9] = (int)__ldcg(st);
        s_misc[10] = (int)__ldcg(st + 1);
        s_misc[11] = (int)__ldcg(st + 2);
      }
      team_sync<NW>();
      cur = s_misc[9];
      best = s_misc[10];
      executed = s_misc[11];
#pragma unroll
      for (int j = 0; j < RB; j++) {
        const bool real = act && j < nr;
        const int wi = real ? (start + j) * WPR + c : 0;
        const uint2 sb = __ldcg(reinterpret_cast<const uint2 *>(st + 4 + 2 * wi));
        S[j] = real ? sb.x : 0u;
        s_bs[j * NT + tid] = real ? sb.y : 0u;
      }
    }

    for (int t = t_begin; t < t_end; t++) {
      RS2_TICK(5);
      // ---- per-sweep constants (uniform over the team)
      uint32_t u1q[4], vq[4];
      const uint32_t qs[4] = {0u, 1u, 10u, 11u};
#pragma unroll
      for (int i = 0; i < (SA ? 4 : 2); i++) philox_uni((uint32_t)t, qs[i], k0, k1, u1q[i], vq[i]);
      uint64_t K2f = 0, K4f = 0;
      if (SA) {
        K2f = a.table[(size_t)t * 4 + 1];
        K4f = a.table[(size_t)t * 4 + 3];
      }
      // thresholds' top bytes at bits 31..24 (plane i of K = bit 31 - i)
      const uint32_t K2w = (uint32_t)K2f, K4w = (uint32_t)K4f;
      const uint32_t all2 = K2f > 0xFFFFFFFFull ? ~0u : 0u, all4 = K4f > 0xFFFFFFFFull ? ~0u : 0u;
      uint32_t fixmask = 0;  // slots whose fix-up word is in use
      auto push_tie = [&](int j, uint32_t item_a, uint32_t kind_flags) {
        if (!((fixmask >> j) & 1u)) {
          reinterpret_cast<uint4 *>(s_fix)[j * NT + tid] = make_uint4(0u, 0u, 0u, 0u);
          fixmask |= 1u << j;
        }
        st_ties++;
        const uint2 it = make_uint2(item_a, (uint32_t)(j * NT + tid) | kind_flags);
        const int slot = atomicAdd(&s_misc[6], 1);
        if (slot < a.tqcap) {
          s_tq[slot] = it;
        } else {  // queue full: decide here
          const Rs2Tie tc{(uint32_t)t, k0, k1, (uint32_t)K2f & 0xFFFFFFu, (uint32_t)K4f & 0xFFFFFFu,
                          WPR, cols};
          rs2_tie_resolve(it, tc, s_fix);
        }
      };

      // ---- 1. priority planes (shared memory) and acceptance planes
#pragma unroll
      for (int j = 0; j < RB; j++) {
        const uint32_t wi = (uint32_t)(row_of(j) * WPR + c);
        uint32_t h1z;
        const PhiloxWord pw = philox_word_tag(wi, RS2_TAG, k0, k1, h1z);
        const P4 p0 = philox_block(pw, h1z, 0u, u1q[0], vq[0], k0, k1);
        const P4 p1 = philox_block(pw, h1z, 1u, u1q[1], vq[1], k0, k1);
        s_planes[(j * NT + tid) * 2] = make_uint4(p0.x, p0.y, p0.z, p0.w);
        s_planes[(j * NT + tid) * 2 + 1] = make_uint4(p1.x, p1.y, p1.z, p1.w);
        if (SA) {
          const P4 q0 = philox_block(pw, h1z, 10u, u1q[2], vq[2], k0, k1);
          const P4 q1 = philox_block(pw, h1z, 11u, u1q[3], vq[3], k0, k1);
          const uint32_t up8[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
          uint32_t lt2 = 0, ne2 = 0, lt4 = 0, ne4 = 0;
#pragma unroll
          for (int i = 7; i >= 0; i--) {
            cmp_step(up8[i], (uint32_t)((int32_t)(K2w << i) >> 31), lt2, ne2);
            cmp_step(up8[i], (uint32_t)((int32_t)(K4w << i) >> 31), lt4, ne4);
          }
          const uint32_t vs = vslot(j);
          const uint32_t t2 = ~ne2 & vs & ~all2, t4 = ~ne4 & vs & ~all4;
          A2[j] = lt2 | all2;
          A4[j] = lt4 | all4;
          uint32_t tie = t2 | t4;
          while (tie) {  // top byte equal to K's: the low 24 bits decide (step 2b)
            const int b = __ffs(tie) - 1;
            tie &= tie - 1;
            push_tie(j, wi | ((uint32_t)b << 11),
                     (((t2 >> b) & 1u) << 14) | (((t4 >> b) & 1u) << 15));
          }
        }
        F[j] = 0u;
        U[j] = vslot(j);
      }
      team_sync<NW>();
      RS2_TICK(0);

      // ---- 2. precedence planes
#pragma unroll
      for (int j = 0; j < RB; j++) {
        const uint4 pa = s_planes[(j * NT + tid) * 2], pb = s_planes[(j * NT + tid) * 2 + 1];
        const uint32_t P[8] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
        const int didx = (j + 1 < nr) ? (j + 1) * NT + tid : tid_below;  // slot 0 of the block below
        const uint4 da = s_planes[didx * 2], db = s_planes[didx * 2 + 1];
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
        Pr[j] = ltR & ~tieR;
        Pd[j] = ltD & ~tieD;
        uint32_t tt = tieR | tieD;
        if (tt) {  // equal top bytes (2^-8 per edge): low 24 bits, then ids (step 2b)
          const int r = row_of(j);
          const uint32_t wi = (uint32_t)(r * WPR + c);
          const uint32_t wir = (uint32_t)(r * WPR + (c + 1 == WPR ? 0 : c + 1));
          const int rd = j + 1 < nr ? r + 1 : down_row_last;
          const uint32_t wid = (uint32_t)(rd * WPR + c);
          while (tt) {
            const int b = __ffs(tt) - 1;
            tt &= tt - 1;
            const uint32_t me = wi | ((uint32_t)b << 11);
            if ((tieR >> b) & 1u) {
              const bool wrapc = b == cpos;
              const uint32_t nb = (wrapc ? wir : wi) | ((uint32_t)(wrapc ? 0 : b + 1) << 11);
              push_tie(j, me | (nb << 16), 1u << 12);
            }
            if ((tieD >> b) & 1u) push_tie(j, me | ((wid | ((uint32_t)b << 11)) << 16), 2u << 12);
          }
        }
      }
      team_sync<NW>();

      // ---- 2b. ties, shared out over the team
      {
        const int cnt = min(s_misc[6], a.tqcap);
        if (cnt > 0) {
          const Rs2Tie tc{(uint32_t)t, k0, k1, (uint32_t)K2f & 0xFFFFFFu, (uint32_t)K4f & 0xFFFFFFu,
                          WPR, cols};
          for (int i = tid; i < cnt; i += NT) rs2_tie_resolve(s_tq[i], tc, s_fix);
        }
      }
      team_sync<NW>();
      if (tid == 0) s_misc[6] = 0;
      if (fixmask) {
#pragma unroll
        for (int j = 0; j < RB; j++)
          if ((fixmask >> j) & 1u) {
            const uint4 f = reinterpret_cast<const uint4 *>(s_fix)[j * NT + tid];
            if (SA) {
              A2[j] |= f.x;
              A4[j] |= f.y;
            }
            Pr[j] |= f.z;
            Pd[j] |= f.w;
          }
      }
      // Pl(v) = !Pr(left(v)), Pu(v) = !Pd(up(v))
#pragma unroll
      for (int j = 0; j < RB; j++) {
        const uint32_t x = __shfl_sync(0xffffffffu, Pr[j], lsrc);
        Pl[j] = lop3<0x07>(Pr[j] * 2u, x >> ppos, 1u);  // ~((Pr << 1) | (x >> ppos & 1))
      }
      s_xpd[tid] = last_of(Pd);
      s_xtop[par * NT + tid] = make_uint2(S[0], U[0]);
      s_xbot[par * NT + tid] = make_uint2(last_of(S), last_of(U));
      team_sync<NW>();
      const uint32_t Pu0 = ~s_xpd[tid_above];
      RS2_TICK(1);

      // ---- 3. rounds.  The edge rows (S, U) are exchanged through one 64-bit
      // word per lane, written after every round and read without waiting for
      // the other warps: a stale value only shows a neighbour as still
      // unvisited (the site then waits a round), and a site seen as visited
      // has its final spin in the same word.  The team meets at a barrier only
      // every RS2_RPB rounds (end-of-sweep test); lanes of one warp exchange
      // in step (syncwarp).  (One buffer instead of two per round: +2.5 %.
      // Fewer barriers gain nothing: the sweep then ends at a multiple of
      // RS2_RPB rounds, profiles/r02_rscan2_rounds_per_barrier.txt.)
      volatile unsigned long long *const xt = (volatile unsigned long long *)(s_xtop + par * NT);
      volatile unsigned long long *const xb = (volatile unsigned long long *)(s_xbot + par * NT);
      for (int rr = 0;; rr++) {
        if (rr >= 1 << 16) {
          if (tid == 0) atomicExch(a.err, GSB_EUNSUPPORTED);
          break;
        }
        st_rounds++;
        const unsigned long long xu64 = xb[tid_above], xd64 = xt[tid_below];
        const uint2 xu = make_uint2((uint32_t)xu64, (uint32_t)(xu64 >> 32));  // row above slot 0
        const uint2 xd = make_uint2((uint32_t)xd64, (uint32_t)(xd64 >> 32));  // row below the last
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
          // the left neighbour sends its last valid bit at bit 0 (its cpos = our ppos)
          const uint32_t lS = __shfl_sync(0xffffffffu, s >> cpos, lsrc);
          const uint32_t lU = __shfl_sync(0xffffffffu, u >> cpos, lsrc);
          const uint32_t RS = rS * Mr + (s >> 1), RU = rU * Mr + (u >> 1);
          const uint32_t LS = s * a.m_two + lS, LU = u * a.m_two + lU;
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
          F[j] = flip * a.m_one + F[j];   // disjoint bits: a site flips once per sweep
          U[j] = ready * a.m_neg + u;     // ready is a subset of u
          left |= U[j];
        }
        xt[tid] = (unsigned long long)S[0] | ((unsigned long long)U[0] << 32);
        xb[tid] = (unsigned long long)last_of(S) | ((unsigned long long)last_of(U) << 32);
        if (rr % RS2_RPB == RS2_RPB - 1) {
          if (!team_any<NW>(left != 0)) break;
        } else {
          __syncwarp();
        }
      }
      par ^= 1;

      RS2_TICK(2);
      // ---- 4. Delta of every flip at its visit, sums, best-so-far
      // exchange (S, F) of the edge rows
      s_xtop[par * NT + tid] = make_uint2(S[0], F[0]);
      s_xbot[par * NT + tid] = make_uint2(last_of(S), last_of(F));
      team_sync<NW>();
      int dsum = 0, ppos_sum = 0, anyf = 0, z = 0;
      {
        const uint2 xu = s_xbot[par * NT + tid_above];
        const uint2 xd = s_xtop[par * NT + tid_below];
#pragma unroll
        for (int j = 0; j < RB; j++) {
          const uint32_t s = S[j], f = F[j], s0 = s ^ f;
          const uint32_t upS = j == 0 ? xu.x : S[j - 1], upF = j == 0 ? xu.y : F[j - 1];
          uint32_t dnS, dnF;
          if (j == RB - 1) {
            dnS = xd.x;
            dnF = xd.y;
          } else if (j == RB - 2) {
            dnS = shortb ? xd.x : S[j + 1];
            dnF = shortb ? xd.y : F[j + 1];
          } else {
            dnS = S[j + 1];
            dnF = F[j + 1];
          }
          const uint32_t rS = __shfl_sync(0xffffffffu, s, rsrc);
          const uint32_t rF = __shfl_sync(0xffffffffu, f, rsrc);
          const uint32_t lS = __shfl_sync(0xffffffffu, s >> cpos, lsrc);
          const uint32_t lF = __shfl_sync(0xffffffffu, f >> cpos, lsrc);
          const uint32_t RS = rS * Mr + (s >> 1), RF = rF * Mr + (f >> 1);
          const uint32_t LS = s * a.m_two + lS, LF = f * a.m_two + lF;
          if (!SA) anyf |= f != 0;
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
          const uint32_t k4 = lop3<0x80>(c1, s1, td) & f, k3 = lop3<0x60>(c1, s1, td) & f;
          const uint32_t k1m = lop3<0x06>(c1, s1, td) & f, k0m = lop3<0x01>(c1, s1, td) & f;
          const int n4 = __popc(k4), n3 = __popc(k3);
          dsum += 4 * n4 + 2 * n3 - 2 * __popc(k1m) - 4 * __popc(k0m);
          ppos_sum += 4 * n4 + 2 * n3;
          if (SA) s_ev[j * NT + tid] = make_uint4(k4, k3, k1m, k0m);
        }
      }
      team_sum4<NW>(s_red, par, lane, warp, dsum, ppos_sum, anyf, z);
      par ^= 1;
      const int cur0 = cur;
      cur += dsum;
      RS2_TICK(3);
      executed = t + 1;
      if (!SA) {
        if (anyf == 0) break;
        // Delta > 0 flips only: the cut rises monotonically, the best is the
        // end-of-sweep state
        best = cur;
#pragma unroll
        for (int j = 0; j < RB; j++) s_bs[j * NT + tid] = S[j];
        continue;
      }
      if (cur0 + ppos_sum <= best) continue;

      // ---- 4b. exact best-so-far in (priority, id) order
      st_gated++;
      for (int i = tid; i < 256; i += NT) s_hist[i] = 0u;
      team_sync<NW>();
#pragma unroll
      for (int j = 0; j < RB; j++) {
        const uint4 e = s_ev[j * NT + tid];
        uint32_t any = e.x | e.y | e.z | e.w;
        if (!any) continue;
        const uint4 pa = s_planes[(j * NT + tid) * 2], pb = s_planes[(j * NT + tid) * 2 + 1];
        const uint32_t PM = e.x | e.y, M4 = e.x | e.w;
        while (any) {
          const int b = __ffs(any) - 1;
          any &= any - 1;
          const uint32_t key8 = gather8(pa, pb, b);
          const uint32_t mag = 2u + 2u * ((M4 >> b) & 1u);
          const uint32_t v = ((PM >> b) & 1u) ? mag * 0x10001u : 0u - mag;
          atomicAdd(&s_hist[key8], v);
        }
      }
      team_sync<NW>();
      // bucket starts C_b = cur0 + sum of the buckets before b, E = largest
      // bucket-end value, candidates (warp 0)
      if (warp == 0) {
        int sb[8], pbk[8], tot = 0;
#pragma unroll
        for (int i = 0; i < 8; i++) {
          const uint32_t x = s_hist[lane * 8 + i];
          sb[i] = (int)(int16_t)(uint16_t)x;
          pbk[i] = (int)((x - (uint32_t)sb[i]) >> 16);
          tot += sb[i];
        }
        int incl = tot;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl += y;
        }
        int run = cur0 + incl - tot, emax = INT_MIN;
#pragma unroll
        for (int i = 0; i < 8; i++) {
          s_cb[lane * 8 + i] = run;
          run += sb[i];
          emax = max(emax, run);
        }
        const int E = __reduce_max_sync(0xffffffffu, emax);
        const int thr = max(best + 1, E);
        uint32_t cm = 0;
#pragma unroll
        for (int i = 0; i < 8; i++)
          if (pbk[i] | sb[i]) cm |= (uint32_t)(s_cb[lane * 8 + i] + pbk[i] >= thr) << i;
        const int cnt = __popc(cm);
        int off = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, off, o);
          if (lane >= o) off += y;
        }
        const int ncand = __shfl_sync(0xffffffffu, off, 31);
        off -= cnt;
#pragma unroll
        for (int i = 0; i < 8; i++)
          if ((cm >> i) & 1u) s_cl[off++] = (uint8_t)(lane * 8 + i);
        if (lane == 0) {
          s_misc[0] = ncand;
          s_misc[7] = E;
        }
      }
      team_sync<NW>();
      const int ncand = s_misc[0], Eend = s_misc[7];
      st_cand += ncand;
      uint32_t kstar = 0, idstar = 0;
      bool improved = false;
      int g0 = 0, gs = ncand;
      while (g0 < ncand) {
        // gather the events of candidates [g0, g0 + gs) with their full keys
        const int thr = max(best + 1, Eend);
        uint32_t cmask[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
        for (int ci = g0; ci < g0 + gs; ci++) {
          const int bkt = s_cl[ci];
          const uint32_t x = s_hist[bkt];
          const int sb = (int)(int16_t)(uint16_t)x;
          const int pbk = (int)((x - (uint32_t)sb) >> 16);
          if (s_cb[bkt] + pbk >= thr) {
#pragma unroll
            for (int q = 0; q < 8; q++)
              if (q == (bkt >> 5)) cmask[q] |= 1u << (bkt & 31);
          }
        }
        if (tid == 0) s_misc[1] = 0;
        team_sync<NW>();
#pragma unroll
        for (int j = 0; j < RB; j++) {
          const uint4 e = s_ev[j * NT + tid];
          uint32_t any = e.x | e.y | e.z | e.w;
          if (!any) continue;
          const uint4 pa = s_planes[(j * NT + tid) * 2], pb = s_planes[(j * NT + tid) * 2 + 1];
          const uint32_t PM = e.x | e.y, M4 = e.x | e.w;
          const int r = row_of(j);
          const uint32_t wi = (uint32_t)(r * WPR + c);
          while (any) {
            const int b = __ffs(any) - 1;
            any &= any - 1;
            const uint32_t key8 = gather8(pa, pb, b);
            uint32_t mw = 0;
#pragma unroll
            for (int q = 0; q < 8; q++)
              if (q == (int)(key8 >> 5)) mw = cmask[q];
            if (!((mw >> (key8 & 31u)) & 1u)) continue;
            const uint32_t key = (key8 << 24) | rs2_low24(wi, (uint32_t)t, 2u, b, k0, k1);
            // Delta code 0..3 = -4, -2, +2, +4
            const uint32_t code = ((PM >> b) & 1u) * 2u + (((PM ^ ~M4) >> b) & 1u);
            const int slot = atomicAdd(&s_misc[1], 1);
            if (slot < a.lcap)
              s_list[slot] = ((unsigned long long)key << 32) |
                             ((unsigned long long)(uint32_t)(r * cols + col0 + b) << 4) | code;
          }
        }
        team_sync<NW>();
        const int m = s_misc[1];
        if (m > a.lcap && gs > 1) {  // too many events at once: fewer candidates per pass
          gs = max(1, gs / 2);
          team_sync<NW>();
          continue;
        }
        if (m <= a.lcap) {
          // rank sort by (key, id) over the team, then an in-order segmented
          // scan (segments = buckets) by warp 0
          unsigned long long mine[(RS2_CAP + NT - 1) / NT];
          int rk[(RS2_CAP + NT - 1) / NT];
#pragma unroll
          for (int q = 0; q < (RS2_CAP + NT - 1) / NT; q++) {
            const int i = q * NT + tid;
            rk[q] = -1;
            if (i < m) {
              mine[q] = s_list[i];
              int r = 0;
              for (int x = 0; x < m; x++) r += s_list[x] < mine[q];
              rk[q] = r;
            }
          }
          team_sync<NW>();
#pragma unroll
          for (int q = 0; q < (RS2_CAP + NT - 1) / NT; q++)
            if (rk[q] >= 0) s_list[rk[q]] = mine[q];
          team_sync<NW>();
          if (warp == 0) {
            int carry = 0, cbkt = -1, bst = best;
            uint32_t ks = kstar, is = idstar;
            bool imp = false;
            for (int base = 0; base < m; base += 32) {
              const int i = base + lane;
              const bool valid = i < m;
              const unsigned long long kk = valid ? s_list[i] : ~0ull;
              const int bkt = (int)(kk >> 56);
              const uint32_t code = (uint32_t)kk & 3u;
              int v = valid ? (code == 0 ? -4 : code == 1 ? -2 : code == 2 ? 2 : 4) : 0;
              const int pbk = __shfl_up_sync(0xffffffffu, bkt, 1);
              int head = lane == 0 ? bkt != cbkt : bkt != pbk;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const int pv = __shfl_up_sync(0xffffffffu, v, o);
                const int ph = __shfl_up_sync(0xffffffffu, head, o);
                if (lane >= o) {
                  if (!head) v += pv;
                  head |= ph;
                }
              }
              if (!head) v += carry;  // the segment began in an earlier chunk
              const int val = valid ? s_cb[bkt] + v : INT_MIN;
              const int mv = __reduce_max_sync(0xffffffffu, val);
              if (mv > bst) {
                const uint32_t hit = __ballot_sync(0xffffffffu, val == mv);
                const int src = __ffs(hit) - 1;
                bst = mv;
                ks = (uint32_t)(__shfl_sync(0xffffffffu, kk, src) >> 32);
                is = ((uint32_t)__shfl_sync(0xffffffffu, kk, src) >> 4) & 0xFFFFu;
                imp = true;
              }
              carry = __shfl_sync(0xffffffffu, v, 31);
              cbkt = __shfl_sync(0xffffffffu, bkt, 31);
            }
            if (lane == 0) {
              s_misc[2] = bst;
              s_misc[3] = (int)ks;
              s_misc[4] = (int)is;
              s_misc[5] = imp ? 1 : 0;
            }
          }
          team_sync<NW>();
        } else {
          // more than RS2_CAP events share one top byte: visit them in (key, id)
          // order by repeated team-wide minimum extraction
          const int bkt = s_cl[g0];
          const uint32_t bm[8] = {(bkt & 0x80) ? ~0u : 0u, (bkt & 0x40) ? ~0u : 0u,
                                  (bkt & 0x20) ? ~0u : 0u, (bkt & 0x10) ? ~0u : 0u,
                                  (bkt & 0x08) ? ~0u : 0u, (bkt & 0x04) ? ~0u : 0u,
                                  (bkt & 0x02) ? ~0u : 0u, (bkt & 0x01) ? ~0u : 0u};
          int run = s_cb[bkt], bst = best;
          uint32_t pk = 0, pid = 0;
          bool first = true, imp = false;
          uint32_t ks = kstar, is = idstar;
          for (int it = 0; it < m; it++) {
            unsigned long long mn = ~0ull;
            int md = 0;
#pragma unroll
            for (int j = 0; j < RB; j++) {
              const uint4 e = s_ev[j * NT + tid];
              uint32_t any = e.x | e.y | e.z | e.w;
              if (!any) continue;
              const uint4 pa = s_planes[(j * NT + tid) * 2], pb = s_planes[(j * NT + tid) * 2 + 1];
              any &= ~(pa.x ^ bm[0]) & ~(pa.y ^ bm[1]) & ~(pa.z ^ bm[2]) & ~(pa.w ^ bm[3]) &
                     ~(pb.x ^ bm[4]) & ~(pb.y ^ bm[5]) & ~(pb.z ^ bm[6]) & ~(pb.w ^ bm[7]);
              const int r = row_of(j);
              const uint32_t wi = (uint32_t)(r * WPR + c);
              while (any) {
                const int b = __ffs(any) - 1;
                any &= any - 1;
                const uint32_t key = ((uint32_t)bkt << 24) | rs2_low24(wi, (uint32_t)t, 2u, b, k0, k1);
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
                s_mm[warp] = mn;
                s_md[warp] = md;
              }
              __syncthreads();
              mn = ~0ull;
              for (int i = 0; i < NW; i++)
                if (s_mm[i] < mn) {
                  mn = s_mm[i];
                  md = s_md[i];
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
            s_misc[2] = bst;
            s_misc[3] = (int)ks;
            s_misc[4] = (int)is;
            s_misc[5] = imp ? 1 : 0;
          }
          team_sync<NW>();
        }
        if (s_misc[5] > 0) {
          best = s_misc[2];
          kstar = (uint32_t)s_misc[3];
          idstar = (uint32_t)s_misc[4];
          improved = true;
        }
        g0 += gs;
        gs = ncand - g0;
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
          const uint32_t f = F[j];
          uint32_t inc = 0;
          if (f) {
            const uint4 pa = s_planes[(j * NT + tid) * 2], pb = s_planes[(j * NT + tid) * 2 + 1];
            const uint32_t P[8] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
            uint32_t lt, tie;
            cmp8(P, kb, lt, tie);
            inc = lt & f;
            uint32_t eqm = tie & f;
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
          s_bs[j * NT + tid] = S[j] ^ f ^ inc;
        }
      }
      RS2_TICK(4);
    }

    if (slice + 1 < a.nslice) {
      // ---- park the trial for its next slice
      uint32_t *st = a.sl_state + (size_t)trial * swords;
      if (tid == 0) {
        st[0] = (uint32_t)cur;
        st[1] = (uint32_t)best;
        st[2] = (uint32_t)executed;
      }
#pragma unroll
      for (int j = 0; j < RB; j++)
        if (act && j < nr) {
          const int wi = (start + j) * WPR + c;
          *reinterpret_cast<uint2 *>(st + 4 + 2 * wi) = make_uint2(S[j], s_bs[j * NT + tid]);
        }
      __threadfence();
      team_sync<NW>();
      if (tid == 0) st_release_u32(a.sl_flag + trial, (uint32_t)(slice + 1));
      item = next_item(item);
      continue;
    }

    // ---- integrity guard (solvers.py:132-133) and outputs
    uint32_t B[RB];
#pragma unroll
    for (int j = 0; j < RB; j++) B[j] = s_bs[j * NT + tid];
    team_sync<NW>();  // the union region is free (no tie queue / bucket pass in flight)
    for (int i = tid; i < a.nstream; i += NT) s_stream[i] = 0u;
    s_xtop[par * NT + tid] = make_uint2(B[0], 0u);
    team_sync<NW>();
    {
      int cb = cut_of(B, s_xtop[par * NT + tid_below].x), z1 = 0, z2 = 0, z3 = 0;
      team_sum4<NW>(s_red, par, lane, warp, cb, z1, z2, z3);
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
        atomicOr(&s_stream[W], x >> sh);
        if (sh && W + 1 < a.nstream) atomicOr(&s_stream[W + 1], x << (32 - sh));
      }
    }
    team_sync<NW>();
    uint8_t *out = a.best_bits + (size_t)trial * a.nbytes;
    for (int i = tid; i < a.nbytes; i += NT)
      out[i] = (uint8_t)(s_stream[i >> 2] >> (24 - 8 * (i & 3)));
    team_sync<NW>();
    item = next_item(item);
  }
  if (a.stats) {
    st_rounds = tid == 0 ? st_rounds : 0;
    st_gated = tid == 0 ? st_gated : 0;
    st_cand = tid == 0 ? st_cand : 0;
    if (st_rounds) atomicAdd(&a.stats[0], st_rounds);
    if (st_gated) atomicAdd(&a.stats[1], st_gated);
    if (st_cand) atomicAdd(&a.stats[2], st_cand);
    if (st_ties) atomicAdd(&a.stats[3], st_ties);
#ifdef GSB_RS2_PROF
    if (tid == 0)
      for (int i = 0; i < 6; i++) atomicAdd(&a.stats[4 + i], (unsigned long long)pf[i]);
#endif
  }
#undef RS2_TICK
}

// kernel entry of an instantiation (nullptr if the shape is not built)
const void *rs2_kernel_nw1(int rb, bool sa);
const void *rs2_kernel_nw2(int rb, bool sa);
const void *rs2_kernel_nw4(int rb, bool sa);
const void *rs2_kernel_nw7(int rb, bool sa);
const void *rs2_kernel_nw8(int rb, bool sa);
const void *rs2_kernel_nw9(int rb, bool sa);
const void *rs2_kernel_nw13(int rb, bool sa);

#define RS2_DEFINE_TABLE(NWV)                                                   \
  const void *rs2_kernel_nw##NWV(int rb, bool sa) {                             \
    switch (rb) {                                                               \
      case 1:                                                                   \
        return sa ? (const void *)rscan2_kernel<NWV, 1, true>                   \
                  : (const void *)rscan2_kernel<NWV, 1, false>;                 \
      case 2:                                                                   \
        return sa ? (const void *)rscan2_kernel<NWV, 2, true>                   \
                  : (const void *)rscan2_kernel<NWV, 2, false>;                 \
      case 3:                                                                   \
        return sa ? (const void *)rscan2_kernel<NWV, 3, true>                   \
                  : (const void *)rscan2_kernel<NWV, 3, false>;                 \
      case 4:                                                                   \
        return sa ? (const void *)rscan2_kernel<NWV, 4, true>                   \
                  : (const void *)rscan2_kernel<NWV, 4, false>;                 \
      case 5:                                                                   \
        return sa ? (const void *)rscan2_kernel<NWV, 5, true>                   \
                  : (const void *)rscan2_kernel<NWV, 5, false>;                 \
      case 7:                                                                   \
        return sa ? (const void *)rscan2_kernel<NWV, 7, true>                   \
                  : (const void *)rscan2_kernel<NWV, 7, false>;                 \
      default:                                                                  \
        return nullptr;                                                         \
    }                                                                           \
  }

// teams beyond 8 warps exist for two rows per lane only (more rows per lane
// would not fit the register file at these team sizes; one row per lane
// measured slower than 7 x 2 on config 2: 13 x 1 2.87e11 vs 3.36e11)
#define RS2_DEFINE_TABLE_WIDE(NWV)                                              \
  const void *rs2_kernel_nw##NWV(int rb, bool sa) {                             \
    switch (rb) {                                                               \
      case 2:                                                                   \
        return sa ? (const void *)rscan2_kernel<NWV, 2, true>                   \
                  : (const void *)rscan2_kernel<NWV, 2, false>;                 \
      default:                                                                  \
        return nullptr;                                                         \
    }                                                                           \
  }

}  // namespace gsb
