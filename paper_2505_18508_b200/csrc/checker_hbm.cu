// checker_hbm.cu -- checkerboard (Philox) sweep engine for tori whose state
// does not fit in one SM's shared memory (BASELINE config 5: 2000x2000).
//
// Same trial semantics, bit layout and RNG contract as checker.cu;
// only the placement changes.  One persistent cooperative kernel runs a batch
// of up to HBM_MAX_T trials in lockstep:
//   * CTA c owns the contiguous word tile [w0, w1) of both colours for EVERY
//     trial of the batch; the tile's couplings and geometry live in its shared
//     memory for the whole launch, so one coupling load serves all trials;
//   * spins live in global memory, [trial][colour][nw] u32 (L2-resident for
//     the config-5 batch: 8 trials x 1 MB), read coalesced word-by-word;
//   * a half-sweep is one pass over the tile's (trial, word) items followed by
//     a grid barrier (the next half-sweep reads the other colour);
//   * per-trial cut bookkeeping: per-CTA partial sums (double buffered by
//     phase parity) reduced after the barrier by every CTA; when the bound
//     cur + sum(positive Delta) can beat best, per-word prefixes in id order
//     (CTA prefix + in-tile scan) find candidate words, the exact first
//     maximum is agreed with a global atomicMax, and owners write the
//     snapshot (two extra barriers, only on those half-sweeps).
#include <cooperative_groups.h>

#include <climits>
#include <cstdint>

#include "checker_common.cuh"
#include "gsb_device.cuh"
#include "gsb_internal.h"

namespace cg = cooperative_groups;

namespace gsb {

constexpr int HBM_MAX_T = 16;
constexpr int HBM_NT = 256;

struct HbmArgs {
  int rows, cols, WPR, nw;
  const uint4 *masks;  // [2][nw]
  const uint4 *geo;    // [nw]
  const uint64_t *table;
  int sweeps;
  const uint64_t *seeds;  // [T]
  int T;
  int greedy;
  uint32_t *state;  // [T][2][nw]
  uint32_t *best;   // [T][2][nw]
  uint32_t *flips;  // [T][nw] accepted mask of the current half-sweep
  int *part;        // [2][T][G] per-CTA Delta sums (tile prefixes)
  int *acc;         // [3][T][2] per-trial (Delta sum, positive-Delta sum) accumulators
  int *cutp;        // [2][T][G] per-CTA cut partials (init / guard)
  long long *keys;  // [2][T]
  int64_t *best_cut;
  int32_t *sweeps_exec;
  uint8_t *best_bits;
  int nbytes;
  int *err;
  unsigned long long *blocks;
};

struct HbmShared {
  int cur[HBM_MAX_T], bestv[HBM_MAX_T], active[HBM_MAX_T], executed[HBM_MAX_T];
  int flipped[HBM_MAX_T];
  int sd[HBM_MAX_T], sp[HBM_MAX_T];  // this CTA's partials of the current phase
  int scan_need[HBM_MAX_T];
  uint64_t seeds[HBM_MAX_T];
};

__device__ __forceinline__ uint32_t ldcg(const uint32_t *p) { return __ldcg(p); }

template <bool SA>
__global__ void __launch_bounds__(HBM_NT) checker_hbm_kernel(HbmArgs a) {
  cg::grid_group grid = cg::this_grid();
  constexpr int NWARP = HBM_NT / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ HbmShared sh;
  __shared__ uint32_t teq[NWARP][32], tc2[NWARP][32], tlt[NWARP][32], tq[NWARP][32];
  __shared__ uint32_t town[NWARP][32];
  __shared__ int wctr[NWARP];
  __shared__ long long kred[NWARP];

  const int G = gridDim.x, c = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = a.nw, T = a.T;
  const int w0 = (int)((long long)nw * c / G), w1 = (int)((long long)nw * (c + 1) / G);
  const int tw = w1 - w0;
  uint4 *mk = (uint4 *)smem_raw;  // [2][tw]
  uint4 *gg = mk + 2 * tw;        // [tw]
  int *wsc = (int *)(gg + tw);    // [tw] per-word scratch for the exact search
  int *isum = wsc + tw;           // [T][tw] (Delta sum << 16) | positive-Delta sum, this phase

  for (int i = tid; i < tw; i += HBM_NT) {
    mk[i] = a.masks[w0 + i];
    mk[tw + i] = a.masks[nw + w0 + i];
    gg[i] = a.geo[w0 + i];
  }
  if (tid < T) {
    sh.seeds[tid] = a.seeds[tid];
    sh.active[tid] = 1;
    sh.executed[tid] = 0;
  }
  if (tid < NWARP) wctr[tid] = 0;
  for (int i = tid; i < NWARP * 32; i += HBM_NT) (&tlt[0][0])[i] = 0;
  __syncthreads();

  // ---- initial spins
  for (int f = tid; f < T * tw; f += HBM_NT) {
    const int tr = f / tw, w = w0 + f % tw;
    const uint64_t seed = sh.seeds[tr];
    const uint32_t V = gg[w - w0].w;
#pragma unroll
    for (int p = 0; p < 2; p++) {
      const P4 o = philox10(P4{(uint32_t)w, 0u, (uint32_t)p, 0u}, (uint32_t)seed,
                            (uint32_t)(seed >> 32));
      const size_t idx = ((size_t)tr * 2 + p) * nw + w;
      a.state[idx] = o.x & V;
      a.best[idx] = o.x & V;
    }
  }
  if (tid == 0 && c == 0)
    for (int tr = 0; tr < T; tr++) {
      a.keys[tr] = a.keys[T + tr] = LLONG_MIN;
      for (int buf = 0; buf < 3; buf++) a.acc[(buf * T + tr) * 2] = a.acc[(buf * T + tr) * 2 + 1] = 0;
    }
  grid.sync();

  // ---- initial cut: colour-0 words, partials per CTA
  if (tid < T) sh.sd[tid] = 0;
  __syncthreads();
  for (int f = tid; f < T * tw; f += HBM_NT) {
    const int tr = f / tw, wl = f % tw, w = w0 + wl;
    const uint32_t *o = a.state + ((size_t)tr * 2 + 1) * nw;
    const uint4 g = gg[wl];
    const uint32_t same = ldcg(o + w);
    const uint32_t shv = shifted_nb(o, same, g.y & 0xFFFFu, g.z & 0xFFFFu);
    const int cc = word_cut(ldcg(a.state + (size_t)tr * 2 * nw + w), same, shv,
                            ldcg(o + (g.x & 0xFFFFu)), ldcg(o + (g.x >> 16)), mk[wl], g.w);
    atomicAdd(&sh.sd[tr], cc);
  }
  __syncthreads();
  if (tid < T) a.cutp[(size_t)tid * G + c] = sh.sd[tid];
  grid.sync();
  if (tid < T) {
    int s = 0;
    for (int i = 0; i < G; i++) s += __ldcg(a.cutp + (size_t)tid * G + i);
    sh.cur[tid] = s;
    sh.bestv[tid] = s;
  }
  __syncthreads();

  unsigned long long tail_blocks = 0;
  int phase = 0, hs = 0;  // phase parity, half-sweep counter
  for (int t = 0; t < a.sweeps; t++) {
    uint32_t K2 = 0, K4 = 0;
    bool all2 = false, all4 = false;
    if (SA) {
      const uint64_t t2 = a.table[(size_t)t * 4 + 1], t4 = a.table[(size_t)t * 4 + 3];
      all2 = t2 > 0xFFFFFFFFull;
      all4 = t4 > 0xFFFFFFFFull;
      K2 = (uint32_t)t2;
      K4 = (uint32_t)t4;
    }
    uint32_t ma[8], mb[8];
#pragma unroll
    for (int q = 0; q < 8; q++) {
      ma[q] = (uint32_t)((int32_t)(K2 << q) >> 31);
      mb[q] = (uint32_t)((int32_t)(K4 << q) >> 31);
    }
    const uint32_t K2lo = K2 & 0xFFFFFFu, K4lo = K4 & 0xFFFFFFu;
    if (tid < T) sh.flipped[tid] = 0;
#pragma unroll 1
    for (int p = 0; p < 2; p++, phase ^= 1, hs++) {
      if (tid < T) {
        sh.sd[tid] = 0;
        sh.sp[tid] = 0;
      }
      __syncthreads();
      // ---- pass over this tile's (trial, word) items; the loop bound is
      // uniform across the block so the warp-cooperative tail stays converged
      const int nitems = T * tw;
      for (int base = 0; base < nitems; base += HBM_NT) {
        const int f = base + tid;
        const bool have = f < nitems;
        const int tr = have ? f / tw : 0;
        const int wl = have ? f % tw : 0;
        const int w = w0 + wl;
        const bool act = have && sh.active[tr];
        uint32_t A = 0, c2 = 0, eq = 0, lt = 0, Sw = 0;
        int wpos = 0, wsum = 0;
        const uint64_t seed = sh.seeds[tr];
        const uint32_t key0 = (uint32_t)seed, key1 = (uint32_t)(seed >> 32);
        if (act) {
          const uint32_t *cw = a.state + ((size_t)tr * 2 + p) * nw;
          const uint32_t *o = a.state + ((size_t)tr * 2 + (p ^ 1)) * nw;
          const uint4 g = gg[wl];
          Sw = ldcg(cw + w);
          const uint32_t same = ldcg(o + w);
          const uint32_t shv = shifted_nb(o, same, p ? (g.y >> 16) : (g.y & 0xFFFFu),
                                          p ? (g.z >> 16) : (g.z & 0xFFFFu));
          const Classes cl = classes(Sw, same, shv, ldcg(o + (g.x & 0xFFFFu)),
                                     ldcg(o + (g.x >> 16)), mk[p * tw + wl], g.w);
          wpos = 2 * __popc(cl.k3) + 4 * __popc(cl.k4);
          if (SA) {
            uint32_t b = cl.ge2;
            int neg = 0;
            if (all2) {
              b |= cl.km2;
              neg += 2 * __popc(cl.km2);
            }
            if (all4) {
              b |= cl.km4;
              neg += 4 * __popc(cl.km4);
            }
            A = b;
            wsum = wpos - neg;
            const uint32_t e2 = (all2 || K2 == 0) ? 0u : cl.km2;
            const uint32_t e4 = (all4 || K4 == 0) ? 0u : cl.km4;
            c2 = e2;
            const uint32_t pend = e2 | e4;
            uint32_t q = pend, l = 0;
            const P4 r0 = philox10(P4{(uint32_t)w, (uint32_t)t, (uint32_t)(2 * p), 1u}, key0, key1);
            const P4 r1 =
                philox10(P4{(uint32_t)w, (uint32_t)t, (uint32_t)(2 * p + 1), 1u}, key0, key1);
            cmp_plane_lsb(r1.w, e2, ma[7], mb[7], q, l);
            cmp_plane_lsb(r1.z, e2, ma[6], mb[6], q, l);
            cmp_plane_lsb(r1.y, e2, ma[5], mb[5], q, l);
            cmp_plane_lsb(r1.x, e2, ma[4], mb[4], q, l);
            cmp_plane_lsb(r0.w, e2, ma[3], mb[3], q, l);
            cmp_plane_lsb(r0.z, e2, ma[2], mb[2], q, l);
            cmp_plane_lsb(r0.y, e2, ma[1], mb[1], q, l);
            cmp_plane_lsb(r0.x, e2, ma[0], mb[0], q, l);
            eq = q;
            lt = l & pend;
            tail_blocks += 2;
          } else {
            A = cl.k3 | cl.k4;
            wsum = wpos;
          }
        }
        if (SA) {
          // warp-cooperative tail (see checker.cu); items are (lane, group)
          uint32_t itm = nibmask8(eq);
          if (eq) {
            teq[warp][lane] = eq;
            tc2[warp][lane] = c2;
            town[warp][lane] = ((uint32_t)tr << 24) | (uint32_t)w;
          }
          bool any_tail = false;
#pragma unroll 1
          while (true) {
            const int cnt = __popc(itm);
            const int sbase = cnt ? atomicAdd(&wctr[warp], cnt) : 0;
            __syncwarp();
            const int total = wctr[warp];
            if (total == 0) break;
            any_tail = true;
            tail_blocks += (lane == 0) ? (unsigned)min(total, 32) : 0u;
            int slot = sbase;
            while (itm && slot < 32) {
              const int gi = __ffs(itm) - 1;
              itm &= itm - 1;
              tq[warp][slot++] = ((uint32_t)lane << 8) | (uint32_t)gi;
            }
            __syncwarp();
            if (lane < total) {
              const uint32_t it = tq[warp][lane];
              const int ol = (int)(it >> 8), gi = (int)(it & 7u);
              const uint32_t own = town[warp][ol];
              const uint64_t sd = sh.seeds[own >> 24];
              const uint32_t wi = own & 0xFFFFFFu;
              const P4 r = philox10(P4{wi, (uint32_t)t, (uint32_t)(4 + 8 * p + gi), 1u},
                                    (uint32_t)sd, (uint32_t)(sd >> 32));
              const uint32_t en = (teq[warp][ol] >> (4 * gi)) & 0xFu;
              const uint32_t cn = (tc2[warp][ol] >> (4 * gi)) & 0xFu;
              const uint32_t tw4[4] = {r.x, r.y, r.z, r.w};
              uint32_t ln = 0;
#pragma unroll
              for (int qq = 0; qq < 4; qq++) {
                const uint32_t klo = ((cn >> qq) & 1u) ? K2lo : K4lo;
                if (((en >> qq) & 1u) && (tw4[qq] >> 8) < klo) ln |= 1u << qq;
              }
              if (ln) atomicOr(&tlt[warp][ol], ln << (4 * gi));
            }
            __syncwarp();
            if (lane == 0) wctr[warp] = 0;
            __syncwarp();
          }
          if (any_tail && eq) {
            lt |= tlt[warp][lane];
            tlt[warp][lane] = 0;
          }
          wsum -= 2 * __popc(lt & c2) + 4 * __popc(lt & ~c2);
          A |= lt;
        }
        if (act) {
          __stcg(a.state + ((size_t)tr * 2 + p) * nw + w, Sw ^ A);
          __stcg(a.flips + (size_t)tr * nw + w, A);
          isum[tr * tw + wl] = (int)((unsigned)wsum << 16) | (wpos & 0xFFFF);
          atomicAdd(&sh.sd[tr], wsum);
          atomicAdd(&sh.sp[tr], wpos);
        }
      }
      __syncthreads();
      // per-trial totals through global accumulators, triple-buffered by
      // half-sweep: buffer hs%3 is added to before the barrier, read after it,
      // and reset one half-sweep later (when every CTA has read it)
      int *pp = a.part + (size_t)phase * T * G;  // per-CTA Delta sums (prefixes)
      int *acc = a.acc + (size_t)(hs % 3) * T * 2;
      if (tid < T) {
        pp[(size_t)tid * G + c] = sh.sd[tid];
        atomicAdd(&acc[2 * tid], sh.sd[tid]);
        atomicAdd(&acc[2 * tid + 1], sh.sp[tid]);
      }
      grid.sync();
      if (tid < T) {
        const int D = __ldcg(&acc[2 * tid]), Pt = __ldcg(&acc[2 * tid + 1]);
        sh.sd[tid] = D;
        sh.sp[tid] = 0;
        if (Pt > 0) sh.flipped[tid] = 1;
        sh.scan_need[tid] = sh.active[tid] && (sh.cur[tid] + Pt > sh.bestv[tid]);
        if (c == 0) {
          // the key slot of the other parity and the previous accumulators
          // have no readers left (all CTAs are past this barrier)
          a.keys[(phase ^ 1) * T + tid] = LLONG_MIN;
          int *prev = a.acc + (size_t)((hs + 2) % 3) * T * 2;
          prev[2 * tid] = 0;
          prev[2 * tid + 1] = 0;
        }
      }
      __syncthreads();
      int need = 0;
      for (int tr = 0; tr < T; tr++) need |= sh.scan_need[tr];
      if (need) {
        // exclusive prefix of this CTA's tile in id order, per trial that needs it
        for (int tr = 0; tr < T; tr++) {
          if (!sh.scan_need[tr]) continue;
          int s = 0;
          for (int i = tid; i < c; i += HBM_NT) s += __ldcg(pp + (size_t)tr * G + i);
          s = (int)__reduce_add_sync(0xffffffffu, (unsigned)s);
          if (lane == 0 && s) atomicAdd(&sh.sp[tr], s);
        }
        __syncthreads();
        // ---- exact new-best search for the trials that need it
        for (int tr = 0; tr < T; tr++) {
          if (!sh.scan_need[tr]) continue;
          const uint32_t *cw = a.state + ((size_t)tr * 2 + p) * nw;
          const uint32_t *o = a.state + ((size_t)tr * 2 + (p ^ 1)) * nw;
          // per-word Delta sums of this half-sweep, recorded by the main pass
          for (int wl = tid; wl < tw; wl += HBM_NT) wsc[wl] = isum[tr * tw + wl] >> 16;
          __syncthreads();
          // exclusive scan of wsc over the tile (warp 0, chunked)
          if (warp == 0) {
            const int per = (tw + 31) / 32;
            const int lo = lane * per, hi = min(lo + per, tw);
            int s = 0;
            for (int i = lo; i < hi; i++) s += wsc[i];
            int incl = s;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
              const int y = __shfl_up_sync(0xffffffffu, incl, off);
              if (lane >= off) incl += y;
            }
            int run = incl - s;
            for (int i = lo; i < hi; i++) {
              const int v = wsc[i];
              wsc[i] = run;
              run += v;
            }
          }
          __syncthreads();
          long long key = LLONG_MIN;
          const int base = sh.cur[tr] + sh.sp[tr];
          for (int wl = tid; wl < tw; wl += HBM_NT) {
            const int w = w0 + wl;
            // only words whose positive-Delta bound can beat best are candidates
            const int pos_bound0 = isum[tr * tw + wl] & 0xFFFF;
            if (pos_bound0 == 0 || base + wsc[wl] + pos_bound0 <= sh.bestv[tr]) continue;
            const uint4 g = gg[wl];
            const uint32_t A = __ldcg(a.flips + (size_t)tr * nw + w);
            if (!A) continue;
            const uint32_t same = ldcg(o + w);
            const uint32_t shv = shifted_nb(o, same, p ? (g.y >> 16) : (g.y & 0xFFFFu),
                                            p ? (g.z >> 16) : (g.z & 0xFFFFu));
            const Classes cl = classes(ldcg(cw + w) ^ A, same, shv, ldcg(o + (g.x & 0xFFFFu)),
                                       ldcg(o + (g.x >> 16)), mk[p * tw + wl], g.w);
            const uint32_t P2 = A & cl.k3, P4m = A & cl.k4, N2 = A & cl.km2, N4 = A & cl.km4;
            const int pos_bound = 2 * __popc(P2) + 4 * __popc(P4m);
            int v = base + wsc[wl];
            if (pos_bound == 0 || v + pos_bound <= sh.bestv[tr]) continue;
            int mx = INT_MIN, mp = -1;
            uint32_t nz = P2 | P4m | N2 | N4;
            while (nz) {
              const int b = __ffs(nz) - 1;
              nz &= nz - 1;
              const uint32_t bm = 1u << b;
              const int d = (P2 & bm) ? 2 : (P4m & bm) ? 4 : (N2 & bm) ? -2 : -4;
              v += d;
              if (d > 0 && v > mx) {
                mx = v;
                mp = b;
              }
            }
            const long long pos = (long long)w * 32 + mp;
            const long long kk = (long long)((unsigned long long)(long long)mx << 32) |
                                 (long long)(0xFFFFFFFFu - (uint32_t)pos);
            key = kk > key ? kk : key;
          }
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            const long long y = __shfl_xor_sync(0xffffffffu, key, off);
            key = y > key ? y : key;
          }
          if (lane == 0) kred[warp] = key;
          __syncthreads();
          if (tid == 0) {
            long long k = LLONG_MIN;
            for (int i = 0; i < NWARP; i++) k = kred[i] > k ? kred[i] : k;
            if (k != LLONG_MIN) atomicMax((long long *)&a.keys[phase * T + tr], k);
          }
          __syncthreads();
        }
        grid.sync();
        // ---- snapshot of every trial whose best improved
        for (int tr = 0; tr < T; tr++) {
          if (!sh.scan_need[tr]) continue;
          const long long key = __ldcg((const long long *)&a.keys[phase * T + tr]);
          const int mval = (int)(key >> 32);
          if (key == LLONG_MIN || mval <= sh.bestv[tr]) continue;
          const long long pos = 0xFFFFFFFFll - (key & 0xFFFFFFFFll);
          const int wstar = (int)(pos >> 5), bstar = (int)(pos & 31);
          for (int wl = tid; wl < tw; wl += HBM_NT) {
            const int w = w0 + wl;
            const uint32_t now = ldcg(a.state + ((size_t)tr * 2 + p) * nw + w);
            const uint32_t A = __ldcg(a.flips + (size_t)tr * nw + w);
            const uint32_t old = now ^ A;
            const uint32_t snap =
                w < wstar ? now : w == wstar ? old ^ (A & ((2u << bstar) - 1u)) : old;
            __stcg(a.best + ((size_t)tr * 2 + p) * nw + w, snap);
            __stcg(a.best + ((size_t)tr * 2 + (p ^ 1)) * nw + w,
                   ldcg(a.state + ((size_t)tr * 2 + (p ^ 1)) * nw + w));
          }
          __syncthreads();
          if (tid == 0) sh.bestv[tr] = mval;
          __syncthreads();
        }
        grid.sync();
      }
      if (tid < T && sh.active[tid]) sh.cur[tid] += sh.sd[tid];
      __syncthreads();
    }
    if (tid < T && sh.active[tid]) {
      sh.executed[tid] = t + 1;
      if (!SA && !sh.flipped[tid]) sh.active[tid] = 0;
    }
    __syncthreads();
    int any_active = 0;
    for (int tr = 0; tr < T; tr++) any_active |= sh.active[tr];
    if (!any_active) break;  // uniform across the grid (same data in every CTA)
  }

  // ---- integrity guard and outputs
  grid.sync();
  if (tid < T) sh.sd[tid] = 0;
  __syncthreads();
  for (int f = tid; f < T * tw; f += HBM_NT) {
    const int tr = f / tw, wl = f % tw, w = w0 + wl;
    const uint32_t *o = a.best + ((size_t)tr * 2 + 1) * nw;
    const uint4 g = gg[wl];
    const uint32_t same = ldcg(o + w);
    const uint32_t shv = shifted_nb(o, same, g.y & 0xFFFFu, g.z & 0xFFFFu);
    const int cc = word_cut(ldcg(a.best + (size_t)tr * 2 * nw + w), same, shv,
                            ldcg(o + (g.x & 0xFFFFu)), ldcg(o + (g.x >> 16)), mk[wl], g.w);
    atomicAdd(&sh.sd[tr], cc);
  }
  __syncthreads();
  if (tid < T) a.cutp[(size_t)(T + tid) * G + c] = sh.sd[tid];
  {
    unsigned long long nb = __reduce_add_sync(0xffffffffu, (unsigned)tail_blocks);
    if (lane == 0 && nb) atomicAdd(a.blocks, nb);
  }
  grid.sync();
  if (c == 0 && tid < T) {
    int s = 0;
    for (int i = 0; i < G; i++) s += __ldcg(a.cutp + (size_t)(T + tid) * G + i);
    a.best_cut[tid] = sh.bestv[tid];
    a.sweeps_exec[tid] = sh.executed[tid];
    if (s != sh.bestv[tid]) atomicExch(a.err, GSB_EINTEGRITY);
    atomicAdd(a.blocks, 2ull * nw);
  }
  // pack best spins MSB-first by site id (grid-stride over all trials' bytes)
  const int n = a.rows * a.cols;
  for (long long byte = (long long)c * HBM_NT + tid; byte < (long long)T * a.nbytes;
       byte += (long long)G * HBM_NT) {
    const int tr = (int)(byte / a.nbytes), bb = (int)(byte % a.nbytes);
    uint32_t v = 0;
    for (int q = 0; q < 8; q++) {
      const int x = bb * 8 + q;
      uint32_t bit = 0;
      if (x < n) {
        const int r = x / a.cols, cc = x - r * a.cols;
        const int p = (r + cc) & 1, k = cc >> 1;
        bit = (ldcg(a.best + ((size_t)tr * 2 + p) * nw + r * a.WPR + (k >> 5)) >> (k & 31)) & 1u;
      }
      v |= bit << (7 - q);
    }
    a.best_bits[(size_t)tr * a.nbytes + bb] = (uint8_t)v;
  }
}

size_t checker_hbm_workspace_bytes(int rows, int cols, int T, int nsm) {
  int WPR, nw;
  checker_words(rows, cols, &WPR, &nw);
  const int TB = T < HBM_MAX_T ? T : HBM_MAX_T;
  const size_t G = (size_t)nsm * 4;
  size_t b = align_up((size_t)2 * nw * 16, 256) + align_up((size_t)nw * 16, 256);  // masks, geo
  b += 2 * align_up((size_t)TB * 2 * nw * 4, 256);                                 // state, best
  b += align_up((size_t)TB * nw * 4, 256);                                         // flips
  b += align_up((size_t)2 * TB * G * 2 * 4, 256) + align_up((size_t)2 * TB * G * 4, 256);
  b += align_up((size_t)2 * TB * 8, 256) + align_up((size_t)3 * TB * 2 * 4, 256);  // keys, acc
  return b;
}

bool checker_hbm_fits(int rows, int cols) {
  if ((rows & 1) || (cols & 1) || rows < 4 || cols < 4) return false;
  int WPR, nw;
  checker_words(rows, cols, &WPR, &nw);
  return nw <= 0xFFFF;  // geometry packs word indices in 16 bits
}

int checker_hbm_run(int rows, int cols, const int8_t *w_dev, int kind, int sweeps,
                    const uint64_t *table, const uint64_t *seeds, int T, int64_t *best_cut,
                    int32_t *sweeps_exec, uint8_t *best_bits, void *ws, int *err_ws,
                    cudaStream_t stream) {
  int WPR, nw;
  checker_words(rows, cols, &WPR, &nw);
  const int nsm = num_sms();
  if (nsm <= 0) return set_error(GSB_ECUDA, "no CUDA device");
  char *p = (char *)ws;
  uint4 *masks = (uint4 *)p;
  p += align_up((size_t)2 * nw * 16, 256);
  uint4 *geo = (uint4 *)p;
  p += align_up((size_t)nw * 16, 256);
  const int TB = T < HBM_MAX_T ? T : HBM_MAX_T;
  uint32_t *state = (uint32_t *)p;
  p += align_up((size_t)TB * 2 * nw * 4, 256);
  uint32_t *best = (uint32_t *)p;
  p += align_up((size_t)TB * 2 * nw * 4, 256);
  uint32_t *flips = (uint32_t *)p;
  p += align_up((size_t)TB * nw * 4, 256);
  checker_masks_kernel_launch(rows, cols, WPR, w_dev, masks, geo, stream);

  const bool sa = kind == GSB_ANNEALING;
  auto kern = sa ? checker_hbm_kernel<true> : checker_hbm_kernel<false>;
  // tile size bounds the dynamic shared memory; use 4 CTAs per SM when they fit
  int G = 0;
  size_t smem = 0;
  for (int per = 4; per >= 1; per--) {
    const int g = nsm * per;
    const int tw = (nw + g - 1) / g;
    const size_t s = (size_t)tw * 16 * 3 + (size_t)tw * 4 * (1 + HBM_MAX_T) + 16;
    if (s > 200 * 1024) continue;
    if (allow_dynamic_smem((const void *)kern, s) != cudaSuccess) continue;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, HBM_NT, s) != cudaSuccess)
      continue;
    if (occ >= per) {
      G = g;
      smem = s;
      break;
    }
  }
  if (G == 0) return set_error(GSB_EUNSUPPORTED, "torus too large for the HBM-tiled engine");
  int *part = (int *)p;
  p += align_up((size_t)2 * TB * G * 2 * 4, 256);
  int *cutp = (int *)p;
  p += align_up((size_t)2 * TB * G * 4, 256);
  long long *keys = (long long *)p;
  p += align_up((size_t)2 * TB * 8, 256);
  int *acc = (int *)p;

  for (int t0 = 0; t0 < T; t0 += HBM_MAX_T) {
    HbmArgs a;
    a.rows = rows;
    a.cols = cols;
    a.WPR = WPR;
    a.nw = nw;
    a.masks = masks;
    a.geo = geo;
    a.table = table;
    a.sweeps = sweeps;
    a.seeds = seeds + t0;
    a.T = T - t0 < HBM_MAX_T ? T - t0 : HBM_MAX_T;
    a.greedy = !sa;
    a.state = state;
    a.best = best;
    a.flips = flips;
    a.part = part;
    a.acc = acc;
    a.cutp = cutp;
    a.keys = keys;
    a.best_cut = best_cut + t0;
    a.sweeps_exec = sweeps_exec + t0;
    a.nbytes = (rows * cols + 7) / 8;
    a.best_bits = best_bits + (size_t)t0 * a.nbytes;
    a.err = err_ws;
    a.blocks = (unsigned long long *)((char *)err_ws + 8);
    void *args[] = {&a};
    const cudaError_t e =
        cudaLaunchCooperativeKernel((void *)kern, G, HBM_NT, args, smem, stream);
    if (e != cudaSuccess) return set_error(GSB_ECUDA, cudaGetErrorString(e));
  }
  return GSB_OK;
}

}  // namespace gsb
