// rscan_big.cu -- random-scan engine (kinds *_random_scan) for tori beyond the
// register-resident teams of rscan2 (BASELINE config 5: 2000 x 2000).
//
// Same contract, same results as rscan2_kernel (DESIGN.md "Random-scan
// contract v2"; executable form oracle/gsb_oracle.c:trial_rscan), different
// placement: the planes of up to 8 trials live in global memory (L2-resident
// at config 5: ~12 MB of planes per trial) and ONE persistent cooperative
// kernel walks all (trial, word) pairs phase by phase, with a grid barrier
// between phases; a barrier serves every trial of the batch.  Per sweep:
//   A  priority planes (2 Philox blocks per word), acceptance planes A2 / A4
//      (2 blocks, ties by the low 24 bits decided in place), U = all, S0 = S;
//   B  precedence planes Pr / Pd by 8-plane compares with the right / down
//      word (ties in place: low 24 bits, then ids);  C  Pl / Pu from the
//      neighbours' Pr / Pd;
//   rounds: (S, U) of a word is one 64-bit word updated in place; a word
//      reads its four neighbours' words without waiting (a stale value only
//      shows a neighbour as unvisited: the site waits a round; a site seen as
//      visited has its final spin in the same 64-bit word).  Finished words
//      cost one load.  One grid barrier and one flag per trial and round;
//   D  Delta of every flip at its visit from the end-of-sweep spins, sums;
//   E  (only if cur0 + positive sum can beat best) exact best-so-far in
//      (priority, id) order: 256 top-byte buckets (sum, positive sum), the
//      largest bucket-end value E, candidates = buckets whose start + positive
//      sum reaches max(best + 1, E); their events are gathered with full keys
//      and one CTA per trial finds the first maximum by radix descent (next
//      key byte: sub-bucket sums, the same pruning) down to segments it sorts
//      in shared memory; the snapshot is S0 ^ (flips with key <= argmax key).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cstdio>

#include "rscan2_kernel.cuh"

namespace cg = cooperative_groups;

namespace gsb {

#ifndef RBG_NTV
#define RBG_NTV 256
#endif
constexpr int RBG_NT = RBG_NTV;
constexpr int RBG_MAXT = 8;     // trials per cooperative launch
constexpr int RBG_SORT = 2048;  // events one CTA sorts at once (16 KB of shared memory)
#ifndef RBG_RPB
#define RBG_RPB 4  // passes of the rounds per grid barrier (1: -14 %, 2: -5 %, 6-8: +1 %)
#endif
#ifndef RBG_MINB
#define RBG_MINB 3  // resident CTAs per SM (85 registers): 3 measured best (2: -8 %, 4: -3 %)
#endif

struct RbgArgs {
  int rows, cols, n, WPR, nw, lastvalid;
  const int8_t *w;
  const uint64_t *table;
  int sweeps;
  const uint64_t *seeds;
  int T, sa;
  uint4 *geo;                             // [nw] right, left, up, down word
  uint32_t *Nr, *Nl, *Nd, *Nu;            // [nw] coupling < 0 planes
  uint32_t *P;                            // [T][8][nw] priority planes
  unsigned long long *SU;                 // [T][nw] S | U << 32
  uint32_t *S0, *Pr, *Pl, *Pd, *Pu, *A2, *A4, *BS;  // [T][nw]
  uint4 *EV;                              // [T][nw] flips by Delta: +4, +2, -2, -4
  int *acc;                               // [3][T][4] per-sweep sums: dsum, positive sum, any flip
  int *flags;                             // [3][T] unvisited sites left after the round
  int *res;                               // [T][8] step E results: ncand, E, best, key, id, improved, count
  unsigned long long *hist;               // [T][256] (positive sum << 32) + sum
  int *cb;                                // [T][256] running cut at each bucket start
  int *hcnt, *loff, *lfill;               // [T][256] events per bucket, list offset, fill count
  int *resb;                              // [T][256][4] per candidate bucket: first maximum, key, id
  uint32_t *cmask;                        // [T][8] candidate buckets
  unsigned long long *list;               // [T][n] events of the candidate buckets
  uint32_t *stream;                       // [T][nstream] output staging
  long long *cutacc;                      // [T] cut recomputation
  int64_t *best_cut;
  int32_t *sweeps_exec;
  uint8_t *best_bits;
  int nbytes, nstream;
  int *err;
};

struct RbgShared {
  uint64_t seed[RBG_MAXT];
  int cur[RBG_MAXT], best[RBG_MAXT], active[RBG_MAXT], executed[RBG_MAXT], gated[RBG_MAXT];
  int improved[RBG_MAXT], flipped[RBG_MAXT];
  uint32_t kstar[RBG_MAXT], idstar[RBG_MAXT];
  uint32_t u1q[RBG_MAXT][4], vq[RBG_MAXT][4];
  int part[RBG_MAXT][4];
  uint32_t cm[RBG_MAXT][8];  // candidate bucket masks (step E3)
  union {
    struct {  // step E4, one CTA per trial
      int hsum[4][256], hpos[4][256], hstart[4][256], hnum[4][256];
      unsigned long long sortbuf[RBG_SORT];
    };
    int priv[3][RBG_MAXT][256];  // step E1: this CTA's bucket sums, positive sums, counts
  };
  int cnt, e_best, e_improved;
  uint32_t e_key, e_id;
  int scan_carry;
};

__device__ __forceinline__ unsigned long long ld64(const unsigned long long *p) {
  return __ldcg(p);
}
__device__ __forceinline__ uint32_t ld32(const uint32_t *p) { return __ldcg(p); }

struct RbgGeo {
  int right, left, up, down, cpos, ppos;
  uint32_t V;
};

__device__ __forceinline__ RbgGeo rbg_geo(const RbgArgs &a, int w) {
  const uint4 g = a.geo[w];
  RbgGeo o;
  o.right = (int)g.x;
  o.left = (int)g.y;
  o.up = (int)g.z;
  o.down = (int)g.w;
  // the word's column is its offset from its left neighbour's ... derive from indices:
  // right == w + 1 unless w is the row's last word; left == w - 1 unless it is the first
  const bool lastcol = o.right != w + 1, firstcol = o.left != w - 1;
  const int vb = lastcol ? a.lastvalid : 32;
  o.cpos = vb - 1;
  o.ppos = (firstcol ? a.lastvalid : 32) - 1;
  o.V = vb == 32 ? 0xFFFFFFFFu : (1u << vb) - 1u;
  return o;
}

// bitonic sort of sh.sortbuf[0..m) ascending (m <= RBG_SORT), whole CTA
__device__ void rbg_sort(RbgShared &sh, int m) {
  int np2 = 1;
  while (np2 < m) np2 <<= 1;
  for (int i = threadIdx.x; i < np2; i += RBG_NT)
    if (i >= m) sh.sortbuf[i] = ~0ull;
  __syncthreads();
  for (int k = 2; k <= np2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < np2; i += RBG_NT) {
        const int l = i ^ j;
        if (l > i) {
          const unsigned long long x = sh.sortbuf[i], y = sh.sortbuf[l];
          const bool up = (i & k) == 0;
          if ((x > y) == up) {
            sh.sortbuf[i] = y;
            sh.sortbuf[l] = x;
          }
        }
      }
      __syncthreads();
    }
}

// One segment of the (priority, id) order: the entries of `list` whose key's top
// `pb` bits equal those of `pv`, with the running cut `base` before them.
// Updates sh.e_best / e_key / e_id / e_improved with the FIRST position whose
// running cut exceeds e_best (strictly), scanning in order.  `floor` = a value
// the running cut is known to reach elsewhere (pruning; >= keeps first attainment).
// `cnt` = how many entries match (known from the parent's sub-bucket counts).
__device__ void rbg_segment(RbgShared &sh, const unsigned long long *list, int m, int pb,
                            uint32_t pv, int base, int floorv, int level, int cnt, int *err) {
  const int tid = threadIdx.x;
  const int sh_bits = 32 - pb;
  auto match = [&](unsigned long long e) -> bool {
    return pb == 0 || ((uint32_t)(e >> 32) >> sh_bits) == (pv >> sh_bits);
  };
  // walk the list with four loads in flight (the passes are bound by L2 latency)
  auto walk = [&](auto &&fn) {
    int i = tid;
    for (; i + 3 * RBG_NT < m; i += 4 * RBG_NT) {
      const unsigned long long e0 = ld64(list + i), e1 = ld64(list + i + RBG_NT);
      const unsigned long long e2 = ld64(list + i + 2 * RBG_NT), e3 = ld64(list + i + 3 * RBG_NT);
      fn(e0);
      fn(e1);
      fn(e2);
      fn(e3);
    }
    for (; i < m; i += RBG_NT) fn(ld64(list + i));
  };
  if (cnt == 0) return;
  if (cnt <= RBG_SORT || pb >= 32) {
    if (cnt > RBG_SORT) {  // > 2048 events with equal 32-bit priorities: not supported
      if (tid == 0) atomicExch(err, GSB_EUNSUPPORTED);
      return;
    }
    if (tid == 0) sh.cnt = 0;
    __syncthreads();
    walk([&](unsigned long long e) {
      if (match(e)) sh.sortbuf[atomicAdd(&sh.cnt, 1)] = e;
    });
    __syncthreads();
    rbg_sort(sh, cnt);
    if (tid < 32) {  // in-order scan by one warp
      int carry = base, bst = sh.e_best;
      uint32_t ks = sh.e_key, is = sh.e_id;
      bool imp = false;
      for (int b0 = 0; b0 < cnt; b0 += 32) {
        const int i = b0 + tid;
        const bool valid = i < cnt;
        const unsigned long long e = valid ? sh.sortbuf[i] : 0ull;
        const uint32_t code = (uint32_t)e & 3u;
        int v = valid ? (code == 0 ? -4 : code == 1 ? -2 : code == 2 ? 2 : 4) : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, v, o);
          if (tid >= o) v += y;
        }
        const int val = valid ? carry + v : INT_MIN;
        const int mv = __reduce_max_sync(0xffffffffu, val);
        if (mv > bst) {
          const uint32_t hit = __ballot_sync(0xffffffffu, val == mv);
          const int src = __ffs(hit) - 1;
          bst = mv;
          ks = (uint32_t)(__shfl_sync(0xffffffffu, e, src) >> 32);
          is = ((uint32_t)__shfl_sync(0xffffffffu, e, src) >> 2) & 0x3FFFFFFFu;
          imp = true;
        }
        carry += __shfl_sync(0xffffffffu, v, 31);
      }
      if (tid == 0 && imp) {
        sh.e_best = bst;
        sh.e_key = ks;
        sh.e_id = is;
        sh.e_improved = 1;
      }
    }
    __syncthreads();
    return;
  }
  // descend one key byte
  int *hsum = sh.hsum[level], *hpos = sh.hpos[level], *hstart = sh.hstart[level];
  int *hnum = sh.hnum[level];
  for (int i = tid; i < 256; i += RBG_NT) hsum[i] = hpos[i] = hnum[i] = 0;
  __syncthreads();
  const int bsh = sh_bits - 8;
  walk([&](unsigned long long e) {
    if (!match(e)) return;
    const uint32_t code = (uint32_t)e & 3u;
    const int d = code == 0 ? -4 : code == 1 ? -2 : code == 2 ? 2 : 4;
    const int sb = (int)(((uint32_t)(e >> 32) >> bsh) & 255u);
    atomicAdd(&hsum[sb], d);
    if (d > 0) atomicAdd(&hpos[sb], d);
    atomicAdd(&hnum[sb], 1);
  });
  __syncthreads();
  if (tid < 32) {  // sub-bucket starts: 8 per lane, warp scan; candidates as a bit mask
    int sb8[8], tot = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
      sb8[i] = hsum[tid * 8 + i];
      tot += sb8[i];
    }
    int incl = tot;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, off);
      if (tid >= off) incl += y;
    }
    int run = base + incl - tot, emax = INT_MIN;
#pragma unroll
    for (int i = 0; i < 8; i++) {
      hstart[tid * 8 + i] = run;
      run += sb8[i];
      if (hnum[tid * 8 + i]) emax = max(emax, run);
    }
    emax = __reduce_max_sync(0xffffffffu, emax);
    if (tid == 0) sh.scan_carry = emax;
  }
  __syncthreads();
  const int fl = max(floorv, sh.scan_carry);
  for (int sb = 0; sb < 256; sb++) {
    if (!hnum[sb]) continue;
    if (hstart[sb] + hpos[sb] < max(sh.e_best + 1, fl)) continue;
    rbg_segment(sh, list, m, pb + 8, pv | ((uint32_t)sb << bsh), hstart[sb], fl, level + 1,
                hnum[sb], err);
  }
}

template <bool SA>
__global__ void __launch_bounds__(RBG_NT, RBG_MINB) rscan_big_kernel(RbgArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ RbgShared sh;
  const int tid = threadIdx.x, lane = tid & 31;
  const int G = gridDim.x, nw = a.nw, T = a.T, cols = a.cols, WPR = a.WPR;
  const long long items = (long long)T * nw;
  const long long gtid = (long long)blockIdx.x * RBG_NT + tid, gstride = (long long)G * RBG_NT;
  // CTA c walks the contiguous items [fbeg, fend) of the (trial, word) space: a band of
  // rows of (mostly) one trial, so neighbours and bucket sums stay local to the CTA
  const long long fbeg = items * blockIdx.x / G, fend = items * (blockIdx.x + 1) / G;

  if (tid < T) {
    sh.seed[tid] = a.seeds[tid];
    sh.active[tid] = 1;
    sh.executed[tid] = 0;
  }
  __syncthreads();

  // ---- instance tables: neighbour words and coupling planes
  for (long long w = gtid; w < nw; w += gstride) {
    const int r = (int)(w / WPR), k = (int)(w - (long long)r * WPR);
    const int ru = r == 0 ? a.rows - 1 : r - 1, rd = r + 1 == a.rows ? 0 : r + 1;
    a.geo[w] = make_uint4((uint32_t)(r * WPR + (k + 1 == WPR ? 0 : k + 1)),
                          (uint32_t)(r * WPR + (k == 0 ? WPR - 1 : k - 1)),
                          (uint32_t)(ru * WPR + k), (uint32_t)(rd * WPR + k));
    const int vb = k == WPR - 1 ? a.lastvalid : 32;
    uint32_t nr = 0, nl = 0, nd = 0, nu = 0;
    for (int b = 0; b < vb; b++) {
      const int col = 32 * k + b, v = r * cols + col;
      const int vl = r * cols + (col == 0 ? cols - 1 : col - 1), vu = ru * cols + col;
      nr |= (uint32_t)(a.w[2 * v] < 0) << b;
      nd |= (uint32_t)(a.w[2 * v + 1] < 0) << b;
      nl |= (uint32_t)(a.w[2 * vl] < 0) << b;
      nu |= (uint32_t)(a.w[2 * vu + 1] < 0) << b;
    }
    a.Nr[w] = nr;
    a.Nl[w] = nl;
    a.Nd[w] = nd;
    a.Nu[w] = nu;
  }
  // zero the accumulators of sweep 0 and the cut accumulators
  if (blockIdx.x == 0) {
    for (int i = tid; i < 3 * T * 4; i += RBG_NT) a.acc[i] = 0;
    for (int i = tid; i < 3 * T; i += RBG_NT) a.flags[i] = 0;
    for (int i = tid; i < T; i += RBG_NT) a.cutacc[i] = 0;
    for (int i = tid; i < T * 8; i += RBG_NT) a.res[i] = 0;
  }
  grid.sync();

  // ---- initial spins: bit b of word 0 of Philox(key, (wi, 0, 31, TAG))
  for (long long f = fbeg + tid; f < fend; f += RBG_NT) {
    const int tr = (int)(f / nw), w = (int)(f - (long long)tr * nw);
    const uint64_t seed = sh.seed[tr];
    const RbgGeo g = rbg_geo(a, w);
    const P4 o = philox10(P4{(uint32_t)w, 0u, 31u, RS2_TAG}, (uint32_t)seed, (uint32_t)(seed >> 32));
    const uint32_t s = o.x & g.V;
    a.SU[f] = (unsigned long long)s;
    a.BS[f] = s;
  }
  grid.sync();

  // cut of the spins in `src` (low words of SU when su, else BS) into cutacc
  auto cut_pass = [&](bool su) {
    if (tid < T) sh.part[tid][0] = 0;
    __syncthreads();
    for (long long f = fbeg + tid; f < fend; f += RBG_NT) {
      const int tr = (int)(f / nw), w = (int)(f - (long long)tr * nw);
      const RbgGeo g = rbg_geo(a, w);
      const size_t o = (size_t)tr * nw;
      auto get = [&](int ww) -> uint32_t {
        return su ? (uint32_t)ld64(a.SU + o + ww) : ld32(a.BS + o + ww);
      };
      const uint32_t x = get(w), xr0 = get(g.right), xd = get(g.down);
      const uint32_t R = (x >> 1) | ((xr0 & 1u) << g.cpos);
      const uint32_t er = (x ^ R) & g.V, ed = (x ^ xd) & g.V;
      const uint32_t nr = a.Nr[w], nd = a.Nd[w];
      const int c = __popc(er & ~nr) - __popc(er & nr) + __popc(ed & ~nd) - __popc(ed & nd);
      if (c) atomicAdd(&sh.part[tr][0], c);
    }
    __syncthreads();
    if (tid < T && sh.part[tid][0]) atomicAdd((unsigned long long *)&a.cutacc[tid],
                                              (unsigned long long)(long long)sh.part[tid][0]);
  };
  cut_pass(true);
  grid.sync();
  if (tid < T) {
    sh.cur[tid] = sh.best[tid] = (int)__ldcg(&a.cutacc[tid]);
  }
  __syncthreads();

#ifdef RBG_PROF
  long long pf[12] = {0}, pf_t = clock64();
  long long pf_rounds = 0, pf_gated = 0, pf_cand = 0;
#define RBG_TICK(i)                   \
  do {                                \
    const long long now_ = clock64(); \
    pf[i] += now_ - pf_t;             \
    pf_t = now_;                      \
  } while (0)
#else
#define RBG_TICK(i)
#endif
  for (int t = 0; t < a.sweeps; t++) {
    // every CTA holds the same per-trial state; stop when no trial is active
    int anyact = 0;
    for (int tr = 0; tr < T; tr++) anyact |= sh.active[tr];
    if (!anyact) break;
    int *acc = a.acc + (t % 3) * T * 4;
    uint64_t K2f = 0, K4f = 0;
    if (SA) {
      K2f = a.table[(size_t)t * 4 + 1];
      K4f = a.table[(size_t)t * 4 + 3];
    }
    const uint32_t all2 = K2f > 0xFFFFFFFFull ? ~0u : 0u, all4 = K4f > 0xFFFFFFFFull ? ~0u : 0u;
    if (tid < T * 4) {
      const int tr = tid >> 2, i = tid & 3;
      const uint32_t qs[4] = {0u, 1u, 10u, 11u};
      const uint64_t seed = sh.seed[tr];
      philox_uni((uint32_t)t, qs[i], (uint32_t)seed, (uint32_t)(seed >> 32), sh.u1q[tr][i],
                 sh.vq[tr][i]);
    }
    // housekeeping for later phases / the next sweep (nobody reads these now)
    if (blockIdx.x == 0) {
      int *nacc = a.acc + ((t + 1) % 3) * T * 4;
      for (int i = tid; i < T * 4; i += RBG_NT) nacc[i] = 0;
      for (int i = tid; i < T; i += RBG_NT) a.flags[i] = 0;  // round 0's flags
    }
    if (blockIdx.x < T)
      for (int i = tid; i < 256; i += RBG_NT) {
        a.hist[(size_t)blockIdx.x * 256 + i] = 0ull;
        a.hcnt[blockIdx.x * 256 + i] = 0;
      }
    __syncthreads();

    // ---- A. priority planes, acceptance planes, U = all, S0 = S
    for (long long f = fbeg + tid; f < fend; f += RBG_NT) {
      const int tr = (int)(f / nw), w = (int)(f - (long long)tr * nw);
      if (!sh.active[tr]) continue;
      const uint64_t seed = sh.seed[tr];
      const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
      const RbgGeo g = rbg_geo(a, w);
      uint32_t h1z;
      const PhiloxWord pw = philox_word_tag((uint32_t)w, RS2_TAG, k0, k1, h1z);
      const P4 p0 = philox_block(pw, h1z, 0u, sh.u1q[tr][0], sh.vq[tr][0], k0, k1);
      const P4 p1 = philox_block(pw, h1z, 1u, sh.u1q[tr][1], sh.vq[tr][1], k0, k1);
      uint32_t *P = a.P + (size_t)tr * 8 * nw + w;
      P[0] = p0.x;
      P[(size_t)nw] = p0.y;
      P[(size_t)2 * nw] = p0.z;
      P[(size_t)3 * nw] = p0.w;
      P[(size_t)4 * nw] = p1.x;
      P[(size_t)5 * nw] = p1.y;
      P[(size_t)6 * nw] = p1.z;
      P[(size_t)7 * nw] = p1.w;
      if (SA) {
        const P4 q0 = philox_block(pw, h1z, 10u, sh.u1q[tr][2], sh.vq[tr][2], k0, k1);
        const P4 q1 = philox_block(pw, h1z, 11u, sh.u1q[tr][3], sh.vq[tr][3], k0, k1);
        const uint32_t up8[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
        uint32_t lt2 = 0, ne2 = 0, lt4 = 0, ne4 = 0;
#pragma unroll
        for (int i = 7; i >= 0; i--) {
          cmp_step(up8[i], (uint32_t)((int32_t)((uint32_t)K2f << i) >> 31), lt2, ne2);
          cmp_step(up8[i], (uint32_t)((int32_t)((uint32_t)K4f << i) >> 31), lt4, ne4);
        }
        const uint32_t t2 = ~ne2 & g.V & ~all2, t4 = ~ne4 & g.V & ~all4;
        uint32_t a2 = lt2 | all2, a4 = lt4 | all4;
        uint32_t tie = t2 | t4;
        while (tie) {  // top byte equal to K's: the low 24 bits decide
          const int b = __ffs(tie) - 1;
          tie &= tie - 1;
          const uint32_t lo = rs2_low24((uint32_t)w, (uint32_t)t, 12u, b, k0, k1);
          a2 |= (uint32_t)(((t2 >> b) & 1u) && lo < ((uint32_t)K2f & 0xFFFFFFu)) << b;
          a4 |= (uint32_t)(((t4 >> b) & 1u) && lo < ((uint32_t)K4f & 0xFFFFFFu)) << b;
        }
        a.A2[f] = a2;
        a.A4[f] = a4;
      }
      const uint32_t s = (uint32_t)ld64(a.SU + f);
      a.S0[f] = s;
      a.SU[f] = (unsigned long long)s | ((unsigned long long)g.V << 32);
    }
    grid.sync();
    RBG_TICK(0);

    // ---- B. precedence planes Pr, Pd
    // (step E's results of the previous sweep have been read by every CTA: the
    // barrier after phase A is behind them)
    if (blockIdx.x == 0)
      for (int i = tid; i < T * 8; i += RBG_NT) a.res[i] = 0;
    for (long long f = fbeg + tid; f < fend; f += RBG_NT) {
      const int tr = (int)(f / nw), w = (int)(f - (long long)tr * nw);
      if (!sh.active[tr]) continue;
      const uint64_t seed = sh.seed[tr];
      const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
      const RbgGeo g = rbg_geo(a, w);
      const uint32_t *Pb = a.P + (size_t)tr * 8 * nw;
      uint32_t P[8], R[8], D[8];
      const uint32_t Mr = 1u << g.cpos;
#pragma unroll
      for (int i = 0; i < 8; i++) {
        P[i] = ld32(Pb + (size_t)i * nw + w);
        const uint32_t x = ld32(Pb + (size_t)i * nw + g.right);
        D[i] = ld32(Pb + (size_t)i * nw + g.down);
        R[i] = ((P[i] >> 1) & ~Mr) | ((x & 1u) << g.cpos);
      }
      uint32_t ltR, tieR, ltD, tieD;
      cmp8(R, P, ltR, tieR);
      cmp8(D, P, ltD, tieD);
      tieR &= g.V;
      tieD &= g.V;
      uint32_t pr = ltR & ~tieR, pd = ltD & ~tieD;
      uint32_t tt = tieR | tieD;
      if (tt) {  // equal top bytes: low 24 bits, then ids
        const int r = w / WPR, k = w - r * WPR;
        const int rd = r + 1 == a.rows ? 0 : r + 1;
        while (tt) {
          const int b = __ffs(tt) - 1;
          tt &= tt - 1;
          const uint32_t me = rs2_low24((uint32_t)w, (uint32_t)t, 2u, b, k0, k1);
          const int id = r * cols + 32 * k + b;
          if ((tieR >> b) & 1u) {
            const bool wrapc = b == g.cpos;
            const uint32_t o = rs2_low24((uint32_t)(wrapc ? g.right : w), (uint32_t)t, 2u,
                                         wrapc ? 0 : b + 1, k0, k1);
            const int idn = r * cols + (32 * k + b + 1 == cols ? 0 : 32 * k + b + 1);
            pr |= (uint32_t)(o < me || (o == me && idn < id)) << b;
          }
          if ((tieD >> b) & 1u) {
            const uint32_t o = rs2_low24((uint32_t)g.down, (uint32_t)t, 2u, b, k0, k1);
            const int idn = rd * cols + 32 * k + b;
            pd |= (uint32_t)(o < me || (o == me && idn < id)) << b;
          }
        }
      }
      a.Pr[f] = pr;
      a.Pd[f] = pd;
    }
    grid.sync();
    RBG_TICK(1);

    // ---- C. Pl(v) = !Pr(left(v)), Pu(v) = !Pd(up(v))
    for (long long f = fbeg + tid; f < fend; f += RBG_NT) {
      const int tr = (int)(f / nw), w = (int)(f - (long long)tr * nw);
      if (!sh.active[tr]) continue;
      const RbgGeo g = rbg_geo(a, w);
      const size_t o = (size_t)tr * nw;
      const uint32_t pr = ld32(a.Pr + o + w), prl = ld32(a.Pr + o + g.left);
      a.Pl[f] = ~((pr << 1) | ((prl >> g.ppos) & 1u));
      a.Pu[f] = ~ld32(a.Pd + o + g.up);
    }
    grid.sync();
    RBG_TICK(2);

    // ---- rounds
    for (int rr = 0;; rr++) {
      if (rr >= 1 << 20) {
        if (gtid == 0) atomicExch(a.err, GSB_EUNSUPPORTED);
        break;
      }
#ifdef RBG_PROF
      pf_rounds++;
#endif
      int *flag = a.flags + (rr % 3) * T;
      if (blockIdx.x == 0 && tid < T) a.flags[((rr + 1) % 3) * T + tid] = 0;
      uint32_t leftmask = 0;
      // RBG_RPB passes over the band per grid barrier: the in-place (S, U) words
      // tolerate stale reads, so passes need no barrier between them -- the
      // barrier only serves the end-of-sweep test, and passes over finished
      // words are cheap
      for (int pass = 0; pass < RBG_RPB; pass++) {
      leftmask = 0;
      // four words' (S, U) loaded ahead: most words are finished in the late rounds
      // and cost only this load, so the loads must not queue behind each other
      for (long long f0 = fbeg + tid; f0 < fend; f0 += 4 * RBG_NT) {
        unsigned long long su4[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const long long fq = f0 + (long long)q * RBG_NT;
          su4[q] = fq < fend ? ld64(a.SU + fq) : 0ull;
        }
#pragma unroll
        for (int q = 0; q < 4; q++) {
        const long long f = f0 + (long long)q * RBG_NT;
        const unsigned long long su = su4[q];
        uint32_t s = (uint32_t)su, u = (uint32_t)(su >> 32);
        if (!u) continue;
        const int tr = (int)(f / nw), w = (int)(f - (long long)tr * nw);
        if (!sh.active[tr]) continue;
        const RbgGeo g = rbg_geo(a, w);
        const size_t o = (size_t)tr * nw;
        const unsigned long long sr = ld64(a.SU + o + g.right), sl = ld64(a.SU + o + g.left);
        const unsigned long long sup = ld64(a.SU + o + g.up), sdn = ld64(a.SU + o + g.down);
        const uint32_t RS = (s >> 1) | (((uint32_t)sr & 1u) << g.cpos);
        const uint32_t RU = (u >> 1) | (((uint32_t)(sr >> 32) & 1u) << g.cpos);
        const uint32_t LS = (s << 1) | (((uint32_t)sl >> g.ppos) & 1u);
        const uint32_t LU = (u << 1) | (((uint32_t)(sl >> 32) >> g.ppos) & 1u);
        const uint32_t upS = (uint32_t)sup, upU = (uint32_t)(sup >> 32);
        const uint32_t dnS = (uint32_t)sdn, dnU = (uint32_t)(sdn >> 32);
        const uint32_t pr = a.Pr[f], pl = a.Pl[f], pd = a.Pd[f], pu = a.Pu[f];
        const uint32_t blk = (pr & RU) | (pl & LU) | (pd & dnU) | (pu & upU);
        const uint32_t ready = u & ~blk;
        if (ready) {
          const uint32_t ta = lop3<0x69>(s, RS, a.Nr[w]);
          const uint32_t tb = lop3<0x69>(s, LS, a.Nl[w]);
          const uint32_t tc = lop3<0x69>(s, upS, a.Nu[w]);
          const uint32_t td = lop3<0x69>(s, dnS, a.Nd[w]);
          const uint32_t s1 = lop3<0x96>(ta, tb, tc), c1 = lop3<0xE8>(ta, tb, tc);
          uint32_t flip;
          if (SA) {
            const uint32_t ge2 = lop3<0xF8>(c1, s1, td);
            const uint32_t mux = lop3<0xCA>(s1 ^ td, a.A2[f], a.A4[f]);
            flip = lop3<0xE0>(ready, ge2, mux);
          } else {
            flip = ready & lop3<0xE0>(c1, s1, td);
          }
          s ^= flip;
          u ^= ready;
          __stcg(a.SU + f, (unsigned long long)s | ((unsigned long long)u << 32));
        }
        if (u) leftmask |= 1u << tr;
        }
      }
      }
      leftmask = __reduce_or_sync(0xffffffffu, leftmask);
      if (lane == 0)
        for (int tr = 0; tr < T; tr++)
          if ((leftmask >> tr) & 1u) atomicOr(&flag[tr], 1);
      grid.sync();
      int any = 0;
      for (int tr = 0; tr < T; tr++) any |= __ldcg(&flag[tr]);
      if (!any) break;
    }

    RBG_TICK(3);
    // ---- D. Delta of every flip at its visit, sums
    if (tid < T) sh.part[tid][0] = sh.part[tid][1] = sh.part[tid][2] = 0;
    __syncthreads();
    for (long long f = fbeg + tid; f < fend; f += RBG_NT) {
      const int tr = (int)(f / nw), w = (int)(f - (long long)tr * nw);
      if (!sh.active[tr]) continue;
      const size_t o = (size_t)tr * nw;
      const uint32_t s = (uint32_t)ld64(a.SU + f), fl = ld32(a.S0 + f) ^ s;
      uint4 ev = make_uint4(0u, 0u, 0u, 0u);
      if (fl) {
        const RbgGeo g = rbg_geo(a, w);
        auto sf = [&](int ww, uint32_t &ss, uint32_t &ff) {
          ss = (uint32_t)ld64(a.SU + o + ww);
          ff = ld32(a.S0 + o + ww) ^ ss;
        };
        uint32_t rS, rF, lS, lF, upS, upF, dnS, dnF;
        sf(g.right, rS, rF);
        sf(g.left, lS, lF);
        sf(g.up, upS, upF);
        sf(g.down, dnS, dnF);
        const uint32_t RS = (s >> 1) | ((rS & 1u) << g.cpos), RF = (fl >> 1) | ((rF & 1u) << g.cpos);
        const uint32_t LS = (s << 1) | ((lS >> g.ppos) & 1u), LF = (fl << 1) | ((lF >> g.ppos) & 1u);
        // neighbour spin at the visit: final if it precedes, else initial
        const uint32_t xr = lop3<0xB4>(RS, RF, a.Pr[f]);
        const uint32_t xl = lop3<0xB4>(LS, LF, a.Pl[f]);
        const uint32_t xdn = lop3<0xB4>(dnS, dnF, a.Pd[f]);
        const uint32_t xup = lop3<0xB4>(upS, upF, a.Pu[f]);
        const uint32_t s0 = s ^ fl;
        const uint32_t ta = lop3<0x69>(s0, xr, a.Nr[w]);
        const uint32_t tb = lop3<0x69>(s0, xl, a.Nl[w]);
        const uint32_t tc = lop3<0x69>(s0, xup, a.Nu[w]);
        const uint32_t td = lop3<0x69>(s0, xdn, a.Nd[w]);
        const uint32_t s1 = lop3<0x96>(ta, tb, tc), c1 = lop3<0xE8>(ta, tb, tc);
        ev.x = lop3<0x80>(c1, s1, td) & fl;
        ev.y = lop3<0x60>(c1, s1, td) & fl;
        ev.z = lop3<0x06>(c1, s1, td) & fl;
        ev.w = lop3<0x01>(c1, s1, td) & fl;
        const int pp = 4 * __popc(ev.x) + 2 * __popc(ev.y);
        const int ds = pp - 2 * __popc(ev.z) - 4 * __popc(ev.w);
        if (ds) atomicAdd(&sh.part[tr][0], ds);
        if (pp) atomicAdd(&sh.part[tr][1], pp);
        atomicOr(&sh.part[tr][2], 1);
      }
      if (SA) a.EV[f] = ev;
    }
    __syncthreads();
    if (tid < T) {
      if (sh.part[tid][0]) atomicAdd(&acc[tid * 4], sh.part[tid][0]);
      if (sh.part[tid][1]) atomicAdd(&acc[tid * 4 + 1], sh.part[tid][1]);
      if (sh.part[tid][2]) atomicOr(&acc[tid * 4 + 2], 1);
    }
    grid.sync();
    int anygated = 0;
    if (tid < T) {
      const int tr = tid;
      sh.gated[tr] = 0;
      sh.improved[tr] = 0;
      sh.flipped[tr] = 0;
      if (sh.active[tr]) {
        const int ds = __ldcg(&acc[tr * 4]), pp = __ldcg(&acc[tr * 4 + 1]);
        const int fl = __ldcg(&acc[tr * 4 + 2]);
        const int cur0 = sh.cur[tr];
        sh.cur[tr] = cur0 + ds;
        sh.executed[tr] = t + 1;
        sh.flipped[tr] = fl;
        if (SA) {
          sh.gated[tr] = cur0 + pp > sh.best[tr];
          sh.part[tr][3] = cur0;
        } else if (!fl) {
          sh.active[tr] = 0;
        } else {
          sh.best[tr] = sh.cur[tr];
        }
      }
    }
    __syncthreads();
    for (int tr = 0; tr < T; tr++) anygated |= sh.gated[tr];
    RBG_TICK(4);

    if (!SA) {
      // greedy: Delta > 0 flips only, the best is the end-of-sweep state
      for (long long f = fbeg + tid; f < fend; f += RBG_NT) {
        const int tr = (int)(f / nw);
        if (sh.flipped[tr]) a.BS[f] = (uint32_t)ld64(a.SU + f);
      }
      continue;
    }
    if (!anygated) continue;

    // ---- E1. bucket sums by priority top byte: per CTA in shared memory, then
    // one global atomic per touched (trial, bucket)
    for (int i = tid; i < 3 * RBG_MAXT * 256; i += RBG_NT) (&sh.priv[0][0][0])[i] = 0;
    __syncthreads();
    for (long long f = fbeg + tid; f < fend; f += RBG_NT) {
      const int tr = (int)(f / nw), w = (int)(f - (long long)tr * nw);
      if (!sh.gated[tr]) continue;
      const uint4 e = a.EV[f];
      uint32_t any = e.x | e.y | e.z | e.w;
      if (!any) continue;
      const uint32_t *Pb = a.P + (size_t)tr * 8 * nw + w;
      const uint4 pa = make_uint4(Pb[0], Pb[(size_t)nw], Pb[(size_t)2 * nw], Pb[(size_t)3 * nw]);
      const uint4 pb = make_uint4(Pb[(size_t)4 * nw], Pb[(size_t)5 * nw], Pb[(size_t)6 * nw],
                                  Pb[(size_t)7 * nw]);
      const uint32_t PM = e.x | e.y, M4 = e.x | e.w;
      while (any) {
        const int b = __ffs(any) - 1;
        any &= any - 1;
        const uint32_t key8 = gather8(pa, pb, b);
        const int mag = 2 + 2 * (int)((M4 >> b) & 1u);
        const bool pos = (PM >> b) & 1u;
        atomicAdd(&sh.priv[0][tr][key8], pos ? mag : -mag);
        if (pos) atomicAdd(&sh.priv[1][tr][key8], mag);
        atomicAdd(&sh.priv[2][tr][key8], 1);
      }
    }
    __syncthreads();
    for (int i = tid; i < T * 256; i += RBG_NT) {
      const int tr = i >> 8, bk = i & 255;
      const int cntv = sh.priv[2][tr][bk];
      if (cntv) {
        const long long v = ((long long)sh.priv[1][tr][bk] << 32) + (long long)sh.priv[0][tr][bk];
        atomicAdd(&a.hist[(size_t)tr * 256 + bk], (unsigned long long)v);
        atomicAdd(&a.hcnt[tr * 256 + bk], cntv);
      }
    }
    grid.sync();
    RBG_TICK(5);

    // ---- E2. bucket starts, E, candidates (CTA tr, warp 0)
    if (blockIdx.x < T && sh.gated[blockIdx.x] && tid < 32) {
      const int tr = blockIdx.x;
      const int cur0 = sh.part[tr][3], best = sh.best[tr];
      int sb[8], pbk[8], tot = 0;
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const unsigned long long x = __ldcg(&a.hist[(size_t)tr * 256 + lane * 8 + i]);
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
      int run = cur0 + incl - tot, emax = INT_MIN, cbase[8];
#pragma unroll
      for (int i = 0; i < 8; i++) {
        cbase[i] = run;
        a.cb[tr * 256 + lane * 8 + i] = run;
        run += sb[i];
        emax = max(emax, run);
      }
      const int E = __reduce_max_sync(0xffffffffu, emax);
      const int thr = max(best + 1, E);
      uint32_t cm = 0;
#pragma unroll
      for (int i = 0; i < 8; i++)
        if (pbk[i] | sb[i]) cm |= (uint32_t)(cbase[i] + pbk[i] >= thr) << i;
      // 8 buckets per lane -> bit (lane * 8 + i) of the 256-bit mask
      const uint32_t part = cm << ((lane & 3) * 8);
      uint32_t word = part;
      word |= __shfl_xor_sync(0xffffffffu, word, 1);
      word |= __shfl_xor_sync(0xffffffffu, word, 2);
      if ((lane & 3) == 0) a.cmask[tr * 8 + (lane >> 2)] = word;
      const int nc = (int)__reduce_add_sync(0xffffffffu, (unsigned)__popc(cm));
      // the candidates' events go to consecutive segments of the list, in bucket order
      int cn[8], mine = 0;
#pragma unroll
      for (int i = 0; i < 8; i++) {
        cn[i] = ((cm >> i) & 1u) ? __ldcg(&a.hcnt[tr * 256 + lane * 8 + i]) : 0;
        mine += cn[i];
      }
      int inc2 = mine;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc2, off);
        if (lane >= off) inc2 += y;
      }
      int o2 = inc2 - mine;
#pragma unroll
      for (int i = 0; i < 8; i++) {
        a.loff[tr * 256 + lane * 8 + i] = o2;
        a.lfill[tr * 256 + lane * 8 + i] = 0;
        o2 += cn[i];
      }
      if (lane == 0) {
        a.res[tr * 8] = nc;
        a.res[tr * 8 + 1] = E;
      }
    }
    grid.sync();
    RBG_TICK(6);

    // ---- E3. events of the candidate buckets with their full keys
    if (tid < T * 8) sh.cm[tid >> 3][tid & 7] = __ldcg(&a.cmask[tid]);
    if (tid < T) sh.part[tid][2] = __ldcg(&a.res[tid * 8]);
    __syncthreads();
    for (long long f = fbeg + tid; f < fend; f += RBG_NT) {
      const int tr = (int)(f / nw), w = (int)(f - (long long)tr * nw);
      if (!sh.gated[tr] || sh.part[tr][2] == 0) continue;
      const uint4 e = a.EV[f];
      uint32_t any = e.x | e.y | e.z | e.w;
      if (!any) continue;
      const uint64_t seed = sh.seed[tr];
      const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
      const uint32_t *Pb = a.P + (size_t)tr * 8 * nw + w;
      const uint4 pa = make_uint4(Pb[0], Pb[(size_t)nw], Pb[(size_t)2 * nw], Pb[(size_t)3 * nw]);
      const uint4 pb = make_uint4(Pb[(size_t)4 * nw], Pb[(size_t)5 * nw], Pb[(size_t)6 * nw],
                                  Pb[(size_t)7 * nw]);
      const uint32_t PM = e.x | e.y, M4 = e.x | e.w;
      const int r = w / WPR, k = w - r * WPR;
      while (any) {
        const int b = __ffs(any) - 1;
        any &= any - 1;
        const uint32_t key8 = gather8(pa, pb, b);
        if (!((sh.cm[tr][key8 >> 5] >> (key8 & 31u)) & 1u)) continue;
        const uint32_t key = (key8 << 24) | rs2_low24((uint32_t)w, (uint32_t)t, 2u, b, k0, k1);
        const uint32_t code = ((PM >> b) & 1u) * 2u + (((PM ^ ~M4) >> b) & 1u);
        const int slot = __ldcg(&a.loff[tr * 256 + key8]) + atomicAdd(&a.lfill[tr * 256 + key8], 1);
        a.list[(size_t)tr * a.n + slot] = ((unsigned long long)key << 32) |
                                          ((unsigned long long)(uint32_t)(r * cols + 32 * k + b) << 2) |
                                          code;
      }
    }
    grid.sync();
    RBG_TICK(7);

    // ---- E4. the first maximum of the running cut.  Every candidate bucket is an
    // independent task (its start value is known): task k goes to CTA k mod G,
    // which finds the bucket's own first maximum above the best before this
    // sweep; the buckets' results are then combined in bucket order (strict
    // improvement), which is the sequential scan's first attainment.
    {
      int k = 0;
      for (int tr = 0; tr < T; tr++) {
        if (!sh.gated[tr] || __ldcg(&a.res[tr * 8]) == 0) continue;
        const int E = __ldcg(&a.res[tr * 8 + 1]);
        const unsigned long long *L = a.list + (size_t)tr * a.n;
        for (int q = 0; q < 8; q++) {
          uint32_t mw = __ldcg(&a.cmask[tr * 8 + q]);
          while (mw) {
            const int bkt = 32 * q + __ffs(mw) - 1;
            mw &= mw - 1;
            if (k++ % G != (int)blockIdx.x) continue;
            if (tid == 0) {
              sh.e_best = sh.best[tr];
              sh.e_improved = 0;
              sh.e_key = sh.e_id = 0u;
            }
            __syncthreads();
            const int mb = __ldcg(&a.hcnt[tr * 256 + bkt]);
            rbg_segment(sh, L + __ldcg(&a.loff[tr * 256 + bkt]), mb, 8, (uint32_t)bkt << 24,
                        __ldcg(&a.cb[tr * 256 + bkt]), E, 0, mb, a.err);
            __syncthreads();
            if (tid == 0) {
              int *rb = a.resb + (tr * 256 + bkt) * 4;
              rb[0] = sh.e_improved ? sh.e_best : INT_MIN;
              rb[1] = (int)sh.e_key;
              rb[2] = (int)sh.e_id;
            }
            __syncthreads();
          }
        }
      }
    }
    grid.sync();
    RBG_TICK(8);

    // ---- E5. snapshot: S0 ^ (flips with (priority, id) <= (key*, id*))
    if (tid < T && sh.gated[tid] && __ldcg(&a.res[tid * 8]) > 0) {
      const int tr = tid;
      int bst = sh.best[tr];
      for (int q = 0; q < 8; q++) {
        uint32_t mw = __ldcg(&a.cmask[tr * 8 + q]);
        while (mw) {
          const int bkt = 32 * q + __ffs(mw) - 1;
          mw &= mw - 1;
          const int *rb = a.resb + (tr * 256 + bkt) * 4;
          const int mval = __ldcg(rb);
          if (mval > bst) {
            bst = mval;
            sh.kstar[tr] = (uint32_t)__ldcg(rb + 1);
            sh.idstar[tr] = (uint32_t)__ldcg(rb + 2);
            sh.improved[tr] = 1;
          }
        }
      }
      sh.best[tr] = bst;
    }
    __syncthreads();
    for (long long f = fbeg + tid; f < fend; f += RBG_NT) {
      const int tr = (int)(f / nw), w = (int)(f - (long long)tr * nw);
      if (!sh.improved[tr]) continue;
      const uint32_t s = (uint32_t)ld64(a.SU + f), fl = ld32(a.S0 + f) ^ s;
      uint32_t inc = 0;
      if (fl) {
        const uint32_t kstar = sh.kstar[tr], idstar = sh.idstar[tr];
        const uint32_t k8 = kstar >> 24, klo = kstar & 0xFFFFFFu;
        const uint32_t *Pb = a.P + (size_t)tr * 8 * nw + w;
        uint32_t P[8], kb[8];
#pragma unroll
        for (int i = 0; i < 8; i++) {
          P[i] = Pb[(size_t)i * nw];
          kb[i] = ((k8 >> (7 - i)) & 1u) ? ~0u : 0u;
        }
        uint32_t lt, tie;
        cmp8(P, kb, lt, tie);
        inc = lt & fl;
        uint32_t eqm = tie & fl;
        if (eqm) {
          const uint64_t seed = sh.seed[tr];
          const int r = w / WPR, k = w - r * WPR;
          while (eqm) {
            const int b = __ffs(eqm) - 1;
            eqm &= eqm - 1;
            const uint32_t lo = rs2_low24((uint32_t)w, (uint32_t)t, 2u, b, (uint32_t)seed,
                                          (uint32_t)(seed >> 32));
            const uint32_t id = (uint32_t)(r * cols + 32 * k + b);
            if (lo < klo || (lo == klo && id <= idstar)) inc |= 1u << b;
          }
        }
      }
      a.BS[f] = s ^ fl ^ inc;
    }
    // (the next sweep's phase A does not touch BS; its first barrier orders the rest)
    RBG_TICK(9);
  }
#ifdef RBG_PROF
  if (blockIdx.x == 0 && tid == 0) {
    long long tot = 0;
    for (int i = 0; i < 12; i++) tot += pf[i];
    printf("rbg prof (cycles %%): A %.1f B %.1f C %.1f rounds %.1f D %.1f E1 %.1f E2 %.1f E3 %.1f E4 %.1f "
           "E5 %.1f | total %lld cycles, rounds %lld\n",
           100.0 * pf[0] / tot, 100.0 * pf[1] / tot, 100.0 * pf[2] / tot, 100.0 * pf[3] / tot,
           100.0 * pf[4] / tot, 100.0 * pf[5] / tot, 100.0 * pf[6] / tot, 100.0 * pf[7] / tot,
           100.0 * pf[8] / tot, 100.0 * pf[9] / tot, tot, pf_rounds);
  }
#endif

  // ---- integrity guard (solvers.py:132-133) and outputs
  grid.sync();
  if (blockIdx.x == 0 && tid < T) a.cutacc[tid] = 0;
  for (long long i = gtid; i < (long long)T * a.nstream; i += gstride) a.stream[i] = 0u;
  grid.sync();
  cut_pass(false);
  for (long long f = fbeg + tid; f < fend; f += RBG_NT) {
    const int tr = (int)(f / nw), w = (int)(f - (long long)tr * nw);
    const RbgGeo g = rbg_geo(a, w);
    const uint32_t x = __brev(ld32(a.BS + f) & g.V);
    if (x) {
      const int r = w / WPR, k = w - r * WPR;
      const long long v0 = (long long)r * cols + 32 * k;
      const long long W = v0 >> 5;
      const int shf = (int)(v0 & 31);
      uint32_t *st = a.stream + (size_t)tr * a.nstream;
      atomicOr(&st[W], x >> shf);
      if (shf && W + 1 < a.nstream) atomicOr(&st[W + 1], x << (32 - shf));
    }
  }
  grid.sync();
  if (blockIdx.x == 0 && tid < T) {
    a.best_cut[tid] = sh.best[tid];
    a.sweeps_exec[tid] = sh.executed[tid];
    if ((long long)__ldcg((const unsigned long long *)&a.cutacc[tid]) != (long long)sh.best[tid])
      atomicExch(a.err, GSB_EINTEGRITY);
  }
  for (long long i = gtid; i < (long long)T * a.nbytes; i += gstride) {
    const int tr = (int)(i / a.nbytes);
    const int j = (int)(i - (long long)tr * a.nbytes);
    a.best_bits[i] = (uint8_t)(__ldcg(&a.stream[(size_t)tr * a.nstream + (j >> 2)]) >> (24 - 8 * (j & 3)));
  }
}

// ------------------------------------------------------------------ host
bool rscan_big_fits(int rows, int cols) {
  return rows >= 3 && cols >= 3 && (long long)rows * cols < (1LL << 28);
}

static size_t rbg_layout(int rows, int cols, int T, RbgArgs *a, char *base) {
  const int WPR = (cols + 31) / 32;
  const size_t nw = (size_t)rows * WPR, n = (size_t)rows * cols;
  const int TB = T < RBG_MAXT ? T : RBG_MAXT;
  const size_t nstream = (n + 31) / 32;
  size_t off = 0;
  auto take = [&](size_t bytes) -> char * {
    char *p = base ? base + off : nullptr;
    off += align_up(bytes, 256);
    return p;
  };
  char *geo = take(nw * 16);
  char *Nr = take(nw * 4), *Nl = take(nw * 4), *Nd = take(nw * 4), *Nu = take(nw * 4);
  char *P = take((size_t)TB * 8 * nw * 4);
  char *SU = take((size_t)TB * nw * 8);
  char *S0 = take((size_t)TB * nw * 4), *Pr = take((size_t)TB * nw * 4), *Pl = take((size_t)TB * nw * 4);
  char *Pd = take((size_t)TB * nw * 4), *Pu = take((size_t)TB * nw * 4), *A2 = take((size_t)TB * nw * 4);
  char *A4 = take((size_t)TB * nw * 4), *BS = take((size_t)TB * nw * 4);
  char *EV = take((size_t)TB * nw * 16);
  char *acc = take((size_t)3 * TB * 4 * 4), *flags = take((size_t)3 * TB * 4), *res = take((size_t)TB * 8 * 4);
  char *hist = take((size_t)TB * 256 * 8), *cb = take((size_t)TB * 256 * 4), *cmask = take((size_t)TB * 8 * 4);
  char *hcnt = take((size_t)TB * 256 * 4), *loff = take((size_t)TB * 256 * 4), *lfill = take((size_t)TB * 256 * 4);
  char *resb = take((size_t)TB * 256 * 4 * 4);
  char *list = take((size_t)TB * n * 8);
  char *stream = take((size_t)TB * nstream * 4);
  char *cutacc = take((size_t)TB * 8);
  if (a) {
    a->geo = (uint4 *)geo;
    a->Nr = (uint32_t *)Nr;
    a->Nl = (uint32_t *)Nl;
    a->Nd = (uint32_t *)Nd;
    a->Nu = (uint32_t *)Nu;
    a->P = (uint32_t *)P;
    a->SU = (unsigned long long *)SU;
    a->S0 = (uint32_t *)S0;
    a->Pr = (uint32_t *)Pr;
    a->Pl = (uint32_t *)Pl;
    a->Pd = (uint32_t *)Pd;
    a->Pu = (uint32_t *)Pu;
    a->A2 = (uint32_t *)A2;
    a->A4 = (uint32_t *)A4;
    a->BS = (uint32_t *)BS;
    a->EV = (uint4 *)EV;
    a->acc = (int *)acc;
    a->flags = (int *)flags;
    a->res = (int *)res;
    a->hist = (unsigned long long *)hist;
    a->cb = (int *)cb;
    a->hcnt = (int *)hcnt;
    a->loff = (int *)loff;
    a->lfill = (int *)lfill;
    a->resb = (int *)resb;
    a->cmask = (uint32_t *)cmask;
    a->list = (unsigned long long *)list;
    a->stream = (uint32_t *)stream;
    a->cutacc = (long long *)cutacc;
  }
  return off;
}

size_t rscan_big_workspace_bytes(int rows, int cols, int T) {
  return rbg_layout(rows, cols, T, nullptr, nullptr);
}

int rscan_big_run(int rows, int cols, const int8_t *w_dev, int kind, int sweeps,
                  const uint64_t *table, const uint64_t *seeds, int T, int64_t *best_cut,
                  int32_t *sweeps_exec, uint8_t *best_bits, void *ws, int *err_ws,
                  cudaStream_t stream) {
  if (!rscan_big_fits(rows, cols))
    return set_error(GSB_EUNSUPPORTED, "torus too large for the random-scan engines");
  const int nsm = num_sms();
  if (nsm < 1) return set_error(GSB_ECUDA, "no CUDA device");
  const bool sa = kind == GSB_ANNEALING;
  auto kern = sa ? rscan_big_kernel<true> : rscan_big_kernel<false>;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, RBG_NT, 0) != cudaSuccess || occ < 1)
    return set_error(GSB_ECUDA, "random-scan (large torus) kernel does not fit on an SM");
  if (occ > 4) occ = 4;
  const int G = nsm * occ;
  RbgArgs a;
  rbg_layout(rows, cols, T, &a, (char *)ws);
  a.rows = rows;
  a.cols = cols;
  a.n = rows * cols;
  a.WPR = (cols + 31) / 32;
  a.nw = rows * a.WPR;
  a.lastvalid = cols - 32 * (a.WPR - 1);
  a.w = w_dev;
  a.table = table;
  a.sweeps = sweeps;
  a.sa = sa;
  a.nbytes = (a.n + 7) / 8;
  a.nstream = (a.n + 31) / 32;
  a.err = err_ws;
  for (int t0 = 0; t0 < T; t0 += RBG_MAXT) {
    a.seeds = seeds + t0;
    a.T = T - t0 < RBG_MAXT ? T - t0 : RBG_MAXT;
    a.best_cut = best_cut + t0;
    a.sweeps_exec = sweeps_exec + t0;
    a.best_bits = best_bits + (size_t)t0 * a.nbytes;
    void *args[] = {&a};
    const cudaError_t e = cudaLaunchCooperativeKernel((void *)kern, G, RBG_NT, args, 0, stream);
    if (e != cudaSuccess) return set_error(GSB_ECUDA, cudaGetErrorString(e));
  }
  return GSB_OK;
}

}  // namespace gsb
