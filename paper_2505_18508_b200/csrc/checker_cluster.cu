// checker_cluster.cu -- checkerboard (Philox) sweep engine for tori whose state
// does not fit one SM but fits the shared memory of one thread-block cluster
// (BASELINE config 5: 2000x2000 on a 16-CTA cluster; SURVEY.md §8(f) rank 4,
// single-trial spatial decomposition over DSMEM).
//
// Same trial semantics, bit layout and RNG contract as checker.cu (DESIGN.md,
// oracle/gsb_oracle.c:trial_checker); only the placement changes.  One
// cluster runs one trial at a time (persistent over trials); CTA q of the
// cluster owns the row band [r0, r0 + R) of both colours:
//   * spins of the band live in shared memory, per colour as padded rows
//     [R + 2][WPR] whose rows 0 and R + 1 are the halo rows of the other CTAs
//     (global rows r0 - 1 and r0 + R); the owner of a boundary word stores it
//     into the neighbour CTA's halo row over DSMEM when it commits;
//   * coupling planes of the band {NS, NSH} and ND (NU of a site is ND of the
//     site above, so ND keeps one extra row) stay in shared memory for the
//     whole launch;
//   * a half-sweep ends with one cluster barrier, which publishes the commits,
//     the halo rows and every CTA's (Delta sum, positive-Delta sum) partial
//     (stored into every CTA of the cluster);
//   * best-so-far tracking (solvers.py:125-127) is one half-sweep behind: after
//     the barrier of half-sweep h every CTA knows the cut before h and the
//     partials, searches its words for the first maximum of the running cut
//     (global prefix = cur + partials of the CTAs before it) and broadcasts its
//     key; the keys are reduced after the next barrier, and the owners write
//     the snapshot from the flips of h (kept in shared memory) -- no extra
//     barrier.  The recompute of a boundary word's classes uses the halo
//     values stashed when it was updated (the neighbour CTA may already be
//     overwriting the halo row with the next half-sweep's values).
// Thread t owns the band words wl = j * NT + t (j < WPT) of both colours; with
// WPR | NT / 2 every thread keeps one word column w = t % WPR and rows of one
// parity, so the neighbour geometry is per-thread constant and the up / down /
// carry words are fixed offsets from three per-thread pointers.
#include <cooperative_groups.h>

#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "checker_common.cuh"
#include "gsb_device.cuh"
#include "gsb_internal.h"

namespace cg = cooperative_groups;

namespace gsb {

constexpr int CL_NT = 512;
constexpr int CL_NWARP = CL_NT / 32;
constexpr int CL_MAXC = 16;

struct ClusterArgs {
  int rows, cols, H, WPR, nw, C;
  const uint4 *masks;  // [2][nw] (checker_masks_kernel)
  const uint64_t *table;
  int sweeps;
  const uint64_t *seeds;
  int T;
  int64_t *best_cut;
  int32_t *sweeps_exec;
  uint8_t *best_bits;
  int nbytes;
  int *err;
  unsigned long long *blocks;
};

struct ClShared {
  int part[2][2][CL_MAXC];  // [slot = h & 1][Delta sum, positive sum][CTA]
  int ipart[2][CL_MAXC];    // initial cut / integrity guard partials
  long long keys[2][CL_MAXC];
  int redD[CL_NWARP], redP[CL_NWARP];
  long long kred[CL_NWARP];
  int scan[8 * CL_NWARP];
  unsigned wctr[CL_NWARP];
};

// band of CTA q: rows [rows*q/C, rows*(q+1)/C)
__host__ __device__ __forceinline__ int band_r0(int rows, int C, int q) {
  return (int)((long long)rows * q / C);
}

struct ClLayout {  // dynamic shared memory, identical in every CTA of a cluster
  size_t mS, mD, st, bst, aprev, stash, tail, total;
};

__host__ __device__ inline ClLayout cl_layout(int Rmax, int WPR, int WPT) {
  ClLayout L;
  size_t o = 0;
  L.mS = o;
  o += (size_t)2 * Rmax * WPR * 8;  // uint2 {NS, NSH}
  L.mD = o;
  o += (size_t)2 * (Rmax + 1) * WPR * 4;  // ND with the row above the band
  L.st = o;
  o += (size_t)2 * (Rmax + 2) * WPR * 4;  // padded spin rows
  L.bst = o;
  o += (size_t)2 * Rmax * WPR * 4;  // best snapshot
  L.aprev = o;
  o += (size_t)Rmax * WPR * 4;  // flips of the half-sweep awaiting its best resolution
  L.stash = o;
  o += (size_t)2 * WPR * 4;  // halo values seen by the boundary rows
  L.tail = o;
  o += (size_t)CL_NWARP * (2 * WPT * 32 + 32) * 4;  // tail exchange + queue per warp
  L.total = o;
  return L;
}

// max of a 64-bit key (value << 32 | tie-break) over the warp: two REDUX ops
__device__ __forceinline__ long long warp_max_key(long long key) {
  const int hi = (int)(key >> 32);
  const int mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? (unsigned)key : 0u);
  return (long long)(((unsigned long long)(unsigned)mh << 32) | ml);
}

__device__ __forceinline__ void cl_arrive_wait() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <int WPT, bool SA>
__global__ void __launch_bounds__(CL_NT, 1) checker_cluster_kernel(ClusterArgs a) {
  constexpr int NT = CL_NT, NWARP = CL_NWARP;
  static_assert(WPT <= 8, "tail items pack (lane, word) as lane << 3 | j");
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ ClShared sh;

  const int C = a.C;
  const int q = (int)cl.block_rank();
  const int cid = (int)(blockIdx.x / C), ncl = (int)(gridDim.x / C);
  const int rows = a.rows, WPR = a.WPR, nw = a.nw, H = a.H;
  const int Rmax = (rows + C - 1) / C;
  const int r0 = band_r0(rows, C, q), R = band_r0(rows, C, q + 1) - r0;
  const int qu = (q + C - 1) % C, qd = (q + 1) % C;  // CTAs above / below
  const int Ru = band_r0(rows, C, qu + 1) - band_r0(rows, C, qu);
  const ClLayout L = cl_layout(Rmax, WPR, WPT);
  uint2 *mS = (uint2 *)(smem_raw + L.mS);
  uint32_t *mD = (uint32_t *)(smem_raw + L.mD);
  uint32_t *st = (uint32_t *)(smem_raw + L.st);
  uint32_t *bst = (uint32_t *)(smem_raw + L.bst);
  uint32_t *aprev = (uint32_t *)(smem_raw + L.aprev);
  uint32_t *stash = (uint32_t *)(smem_raw + L.stash);
  const int RW = Rmax * WPR, RD = (Rmax + 1) * WPR, PS = (Rmax + 2) * WPR;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t *tail = (uint32_t *)(smem_raw + L.tail) + warp * (2 * WPT * 32 + 32);
  uint32_t *teq = tail;                 // [WPT][32] pending masks -> tail-accepted bits
  uint32_t *tc2 = tail + WPT * 32;      // [WPT][32] class -2 masks
  uint32_t *myq = tail + 2 * WPT * 32;  // [32] queue
  unsigned *wctr = &sh.wctr[warp];

  const int w = tid % WPR, lr0 = tid / WPR;  // WPR divides NT / 2
  const int gw0 = r0 * WPR;                  // global index of band word 0
  const int lb = (H - 1) & 31;
  const uint32_t V = (w < WPR - 1 || lb == 31) ? 0xFFFFFFFFu : ((2u << lb) - 1u);
  bool own[WPT];
#pragma unroll
  for (int j = 0; j < WPT; j++) own[j] = lr0 + j * (NT / WPR) < R;

  // remote halo rows: our first row -> bottom halo of the CTA above, our last
  // row -> top halo of the CTA below (colour 0; colour 1 adds PS)
  uint32_t *halo_up = cl.map_shared_rank(st, qu) + (Ru + 1) * WPR + w;
  uint32_t *halo_dn = cl.map_shared_rank(st, qd) + w;

  // ---- coupling planes of the band (same for every trial of the launch)
  for (int i = tid; i < R * WPR; i += NT) {
#pragma unroll
    for (int p = 0; p < 2; p++) {
      const uint4 m = a.masks[(size_t)p * nw + gw0 + i];
      mS[p * RW + i] = make_uint2(m.x, m.y);
      mD[p * RD + WPR + i] = m.w;
    }
  }
  for (int i = tid; i < WPR; i += NT) {
    const int ru = (r0 + rows - 1) % rows;
#pragma unroll
    for (int p = 0; p < 2; p++) mD[p * RD + i] = a.masks[(size_t)p * nw + ru * WPR + i].w;
  }
  if (tid < NWARP) sh.wctr[tid] = 0;
  for (int i = tid; i < NWARP * (2 * WPT * 32 + 32); i += NT)
    ((uint32_t *)(smem_raw + L.tail))[i] = 0;
  cl_arrive_wait();  // every CTA of the cluster runs before any DSMEM access

  unsigned tail_blocks = 0;
  for (int trial = cid; trial < a.T; trial += ncl) {
    const uint64_t seed = a.seeds[trial];
    const uint32_t key0 = (uint32_t)seed, key1 = (uint32_t)(seed >> 32);

    // ---- initial spins: bit b of word 0 of Philox(key, (wi, 0, p, 0))
    uint32_t cur_w[WPT], oth_w[WPT];
#pragma unroll
    for (int j = 0; j < WPT; j++) {
      const int wl = j * NT + tid;
      cur_w[j] = oth_w[j] = 0;
      if (own[j]) {
#pragma unroll
        for (int p = 0; p < 2; p++) {
          const P4 o = philox10(P4{(uint32_t)(gw0 + wl), 0u, (uint32_t)p, 0u}, key0, key1);
          const uint32_t s0 = o.x & V;
          if (p == 0) cur_w[j] = s0; else oth_w[j] = s0;
          st[p * PS + WPR + wl] = s0;
          bst[p * RW + wl] = s0;
          if (wl < WPR) halo_up[p * PS] = s0;
          if (wl >= (R - 1) * WPR) halo_dn[p * PS] = s0;
        }
      }
    }
    cl_arrive_wait();

    // ---- initial cut: colour-0 words (every edge has one colour-0 endpoint)
    auto band_cut = [&](const uint32_t *s0p, const uint32_t *s1p, const uint32_t *up_row,
                        const uint32_t *dn_row) {
      // s0p / s1p: colour 0 / 1 words of the band at index wl; up_row / dn_row:
      // colour-1 words of the rows above / below the band (index w)
      const int e = (r0 + lr0) & 1;  // colour 0 sites of this thread's rows
      const int cw = e == 0 ? (w > 0 ? w - 1 : WPR - 1) : (w < WPR - 1 ? w + 1 : 0);
      const uint32_t src = e == 0 ? (w > 0 ? 31u : (uint32_t)lb) : 0u;
      const uint32_t dst = e == 0 ? 0u : (w < WPR - 1 ? 31u : (uint32_t)lb);
      int c0 = 0;
#pragma unroll
      for (int j = 0; j < WPT; j++) {
        if (!own[j]) continue;
        const int wl = j * NT + tid, lr = lr0 + j * (NT / WPR);
        const uint32_t same = s1p[wl];
        const uint32_t x = s1p[lr * WPR + cw];
        const uint32_t carry = ((x >> src) & 1u) << dst;
        const uint32_t shv = e ? ((same >> 1) | carry) : ((same << 1) | carry);
        const uint32_t up = lr == 0 ? up_row[w] : s1p[wl - WPR];
        const uint32_t dn = lr == R - 1 ? dn_row[w] : s1p[wl + WPR];
        const uint2 m = mS[wl];
        // NU of colour 0 = ND of colour 1 one row up (mD[1] row lr of the padded rows)
        c0 += word_cut(s0p[wl], same, shv, up, dn,
                       make_uint4(m.x, m.y, mD[RD + wl], mD[WPR + wl]), V);
      }
      return c0;
    };
    {
      const int c0 = band_cut(st + WPR, st + PS + WPR, st + PS, st + PS + (R + 1) * WPR);
      const int wsum = (int)__reduce_add_sync(0xffffffffu, (unsigned)c0);
      if (lane == 0) sh.redD[warp] = wsum;
      __syncthreads();
      if (warp == 0) {
        int s = lane < NWARP ? sh.redD[lane] : 0;
        s = (int)__reduce_add_sync(0xffffffffu, (unsigned)s);
        if (lane < C) *cl.map_shared_rank(&sh.ipart[0][q], lane) = s;
      }
    }
    cl_arrive_wait();
    int cur = 0;
    for (int i = 0; i < C; i++) cur += sh.ipart[0][i];
    int best = cur;
    int executed = 0;
    bool pend_prev = false;  // half-sweep h-1 broadcast best keys to resolve

    // resolve the keys of the previous half-sweep: winner, then the snapshot
    // (ow/ap: words of that half-sweep's colour after it and its flips;
    //  cw/aq: the other colour now and its flips since)
    auto resolve = [&](int pp, const uint32_t *ow, const uint32_t *cw, const uint32_t *aq,
                       int slot) {
      const long long key = warp_max_key(lane < C ? sh.keys[slot][lane] : LLONG_MIN);
      const int mval = (int)(key >> 32);
      if (key == LLONG_MIN || mval <= best) return;
      best = mval;
      const long long pos = 0xFFFFFFFFll - (key & 0xFFFFFFFFll);
      const int wstar = (int)(pos >> 5), bstar = (int)(pos & 31);
#pragma unroll
      for (int j = 0; j < WPT; j++) {
        if (!own[j]) continue;
        const int wl = j * NT + tid, gwi = gw0 + wl;
        const uint32_t now = ow[j], Ap = aprev[wl], old = now ^ Ap;
        bst[pp * RW + wl] =
            gwi < wstar ? now : gwi == wstar ? old ^ (Ap & ((2u << bstar) - 1u)) : old;
        bst[(pp ^ 1) * RW + wl] = cw[j] ^ aq[j];
      }
    };

    int hs = 0;  // half-sweep counter
    for (int t = 0; t < a.sweeps; t++) {
      uint32_t K2 = 0, K4 = 0, K2lo = 0, K4lo = 0, me2 = 0, me4 = 0;
      if (SA) {
        const uint64_t t2 = a.table[(size_t)t * 4 + 1], t4 = a.table[(size_t)t * 4 + 3];
        K2 = t2 > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)t2;
        K4 = t4 > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)t4;
        K2lo = t2 > 0xFFFFFFFFull ? 0x1000000u : (K2 & 0xFFFFFFu);
        K4lo = t4 > 0xFFFFFFFFull ? 0x1000000u : (K4 & 0xFFFFFFu);
        me2 = t2 ? ~0u : 0u;
        me4 = t4 ? ~0u : 0u;
      }
      uint32_t ma[8], mb[8];
#pragma unroll
      for (int qq = 0; qq < 8; qq++) {
        ma[qq] = (uint32_t)((int32_t)(K2 << qq) >> 31);
        mb[qq] = (uint32_t)((int32_t)(K4 << qq) >> 31);
      }
      bool sweep_flipped = false;
#pragma unroll 1
      for (int p = 0; p < 2; p++, hs++) {
        const int slot = hs & 1;
        // per-thread geometry of colour p (rows of one parity)
        const int e = (r0 + lr0 + p) & 1;
        const int cwc = e == 0 ? (w > 0 ? w - 1 : WPR - 1) : (w < WPR - 1 ? w + 1 : 0);
        const uint32_t src = e == 0 ? (w > 0 ? 31u : (uint32_t)lb) : 0u;
        const uint32_t dst = e == 0 ? 0u : (w < WPR - 1 ? 31u : (uint32_t)lb);
        const uint32_t rot = e == 0 ? 1u : 31u;
        const uint32_t VG = V & ~(e == 0 ? 1u : 0x80000000u);
        const uint32_t ca = 31u - src, cb = 31u - dst;
        const uint32_t *so = st + (p ^ 1) * PS;
        const uint32_t *so_up = so + tid;                    // + j*NT: row above
        const uint32_t *so_dn = so + 2 * WPR + tid;          // row below
        const uint32_t *so_cy = so + (lr0 + 1) * WPR + cwc;  // carry word
        const uint2 *ms = mS + p * RW + tid;
        const uint32_t *mu = mD + (p ^ 1) * RD + tid;  // NU = ND of the row above
        const uint32_t *md = mD + p * RD + WPR + tid;
        uint32_t *sc = st + p * PS + WPR + tid;

        // per word only the flips A and wsp = 65536 * (positive-Delta sum) +
        // (Delta sum of the accepted flips) stay in registers; undecided sites
        // go to the warp's tail slots right away
        uint32_t A[WPT];
        int wsp[WPT];
#define WS(j) ((int)(short)wsp[j])
#define WP(j) ((wsp[j] - WS(j)) >> 16)
        uint32_t wm = 0;  // bit j: word j has undecided sites (tail items)
        // ---- pass 1: classes and the unconditional planes 0-7
#pragma unroll
        for (int j = 0; j < WPT; j++) {
          const int wl = j * NT + tid;
          const uint32_t gwi = (uint32_t)(gw0 + wl);
          A[j] = 0;
          wsp[j] = 0;
          if (j < WPT - 1 || own[j]) {
            const uint32_t same = oth_w[j];
            const uint32_t x = so_cy[j * NT];
            const uint32_t shv = lop3<0xEA>(__funnelshift_l(same, same, rot), VG, (x << ca) >> cb);
            const uint32_t up = so_up[j * NT], dn = so_dn[j * NT];
            if (j == 0 && wl < WPR) stash[w] = up;
            if (wl >= (R - 1) * WPR && wl < R * WPR) stash[WPR + w] = dn;
            const uint2 m2 = ms[j * NT];
            const Classes c =
                classes_pad(cur_w[j], same, shv, up, dn, make_uint4(m2.x, m2.y, mu[j * NT], md[j * NT]));
            const int wpos = 2 * __popc(c.k3) + 4 * __popc(c.k4);
            if (SA) {
              const uint32_t e2 = c.km2 & me2, e4 = c.km4 & me4;
              const uint32_t pendm = e2 | e4;
              uint32_t qv = pendm, l = 0;
              const P4 q0 = philox10(P4{gwi, (uint32_t)t, (uint32_t)(2 * p), 1u}, key0, key1);
              const P4 q1 = philox10(P4{gwi, (uint32_t)t, (uint32_t)(2 * p + 1), 1u}, key0, key1);
              cmp_plane_lsb(q1.w, e2, ma[7], mb[7], qv, l);
              cmp_plane_lsb(q1.z, e2, ma[6], mb[6], qv, l);
              cmp_plane_lsb(q1.y, e2, ma[5], mb[5], qv, l);
              cmp_plane_lsb(q1.x, e2, ma[4], mb[4], qv, l);
              cmp_plane_lsb(q0.w, e2, ma[3], mb[3], qv, l);
              cmp_plane_lsb(q0.z, e2, ma[2], mb[2], qv, l);
              cmp_plane_lsb(q0.y, e2, ma[1], mb[1], qv, l);
              cmp_plane_lsb(q0.x, e2, ma[0], mb[0], qv, l);
              const uint32_t lt = l & pendm;
              A[j] = (c.ge2 & V) | lt;
              wsp[j] = 65537 * wpos - 2 * __popc(lt & e2) - 4 * __popc(lt & e4);
              if (qv) {
                teq[j * 32 + lane] = qv;
                tc2[j * 32 + lane] = e2;
                wm |= 1u << j;
              }
            } else {
              A[j] = c.k3 | c.k4;
              wsp[j] = 65537 * wpos;
            }
          }
        }
        // ---- pass 2 (SA): warp-cooperative tail (as checker.cu); an item's
        // result overwrites its pending mask in teq
        if (SA) {
          if (__any_sync(0xffffffffu, wm != 0u)) {
            const unsigned wbase = *wctr;
            uint32_t rem = wm;
#pragma unroll 1
            for (unsigned done = 0;;) {
              const int cnt = __popc(rem);
              const int total = (int)__reduce_add_sync(0xffffffffu, (unsigned)cnt);
              if (total == 0) break;
              const int sbase = (int)((cnt ? atomicAdd(wctr, (unsigned)cnt) : 0u) - wbase - done);
              int slot2 = sbase;
              while (rem && slot2 < 32) {
                const int jj = __ffs(rem) - 1;
                rem &= rem - 1;
                myq[slot2++] = ((uint32_t)lane << 3) | (uint32_t)jj;
              }
              __syncwarp();
              if (lane < total) {
                const uint32_t it = myq[lane];
                const int ol = (int)(it >> 3), jj = (int)(it & 7u);
                const uint32_t gwi = (uint32_t)(gw0 + jj * NT + warp * 32 + ol);
                uint32_t ev = teq[jj * 32 + ol];
                const uint32_t cwm = tc2[jj * 32 + ol];
                uint32_t acc = 0;
                while (ev) {
                  const int g4 = (__ffs(ev) - 1) & ~3;
                  const P4 r = philox10(P4{gwi, (uint32_t)t, (uint32_t)(4 + 8 * p + (g4 >> 2)), 1u},
                                        key0, key1);
                  tail_blocks++;
                  const uint32_t en = (ev >> g4) & 0xFu, cn = (cwm >> g4) & 0xFu;
                  const uint32_t tw[4] = {r.x, r.y, r.z, r.w};
                  uint32_t ln = 0;
#pragma unroll
                  for (int qq = 0; qq < 4; qq++) {
                    const uint32_t klo = ((cn >> qq) & 1u) ? K2lo : K4lo;
                    if (((en >> qq) & 1u) && (tw[qq] >> 8) < klo) ln |= 1u << qq;
                  }
                  acc |= ln << g4;
                  ev &= ~(0xFu << g4);
                }
                teq[jj * 32 + ol] = acc;
              }
              __syncwarp();
              done += (unsigned)total;
            }
#pragma unroll
            for (int j = 0; j < WPT; j++) {
              if ((wm >> j) & 1u) {
                const uint32_t tl = teq[j * 32 + lane], c2m = tc2[j * 32 + lane];
                A[j] |= tl;
                wsp[j] -= 2 * __popc(tl & c2m) + 4 * __popc(tl & ~c2m);
              }
            }
          }
        }
        // ---- pass 3: commit; boundary words also go to the neighbours' halos
        int dsum = 0, psum = 0;
#pragma unroll
        for (int j = 0; j < WPT; j++) {
          if (own[j]) {
            const int wl = j * NT + tid;
            cur_w[j] ^= A[j];
            sc[j * NT] = cur_w[j];
            if (wl < WPR) halo_up[p * PS] = cur_w[j];
            if (wl >= (R - 1) * WPR) halo_dn[p * PS] = cur_w[j];
            dsum += WS(j);
            psum += WP(j);
          }
        }
        {
          const int wd = (int)__reduce_add_sync(0xffffffffu, (unsigned)dsum);
          const int wp = (int)__reduce_add_sync(0xffffffffu, (unsigned)psum);
          if (lane == 0) {
            sh.redD[warp] = wd;
            sh.redP[warp] = wp;
          }
          __syncthreads();
          if (warp == 0) {
            int d = lane < NWARP ? sh.redD[lane] : 0, pp = lane < NWARP ? sh.redP[lane] : 0;
            d = (int)__reduce_add_sync(0xffffffffu, (unsigned)d);
            pp = (int)__reduce_add_sync(0xffffffffu, (unsigned)pp);
            if (lane < C) {
              *cl.map_shared_rank(&sh.part[slot][0][q], lane) = d;
              *cl.map_shared_rank(&sh.part[slot][1][q], lane) = pp;
            }
          }
        }
        cl_arrive_wait();

        // ---- after the barrier: resolve half-sweep h-1, then this one's sums
        if (pend_prev) resolve(p ^ 1, oth_w, cur_w, A, slot ^ 1);
        int D, Pt, pre;
        {
          const int d = lane < C ? sh.part[slot][0][lane] : 0;
          const int pp = lane < C ? sh.part[slot][1][lane] : 0;
          D = (int)__reduce_add_sync(0xffffffffu, (unsigned)d);
          Pt = (int)__reduce_add_sync(0xffffffffu, (unsigned)pp);
          pre = (int)__reduce_add_sync(0xffffffffu, (unsigned)(lane < q ? d : 0));
        }
        if (Pt > 0) sweep_flipped = true;  // greedy flips are exactly the positive ones
        const bool pend = cur + Pt > best;  // uniform over the cluster
        if (pend) {
          // per-word prefix bounds in visit order (CTA, j, warp, lane)
          int excl[WPT], rtot[WPT];
#pragma unroll
          for (int j = 0; j < WPT; j += 2) {
            const bool two = j + 1 < WPT;
            uint32_t x = (uint32_t)(WS(j) + 128) |
                         (two ? (uint32_t)(WS(two ? j + 1 : j) + 128) << 16 : 0u);
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
              const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
              if (lane >= off) x += y;
            }
            const uint32_t tot = __shfl_sync(0xffffffffu, x, 31);
            const int bias = 128 * (lane + 1);
            excl[j] = (int)(x & 0xFFFFu) - bias - WS(j);
            rtot[j] = (int)(tot & 0xFFFFu) - 4096;
            if (two) {
              excl[j + 1] = (int)(x >> 16) - bias - WS(j + 1);
              rtot[j + 1] = (int)(tot >> 16) - 4096;
            }
          }
          if (lane == 31) {
#pragma unroll
            for (int j = 0; j < WPT; j++) sh.scan[j * NWARP + warp] = rtot[j];
          }
          __syncthreads();
          if (warp == 0) {  // exclusive scan of the (j, warp) row totals, 4 per lane
            int v[4], s4 = 0;
#pragma unroll
            for (int k = 0; k < 4; k++) {
              const int i = 4 * lane + k;
              v[k] = i < WPT * NWARP ? sh.scan[i] : 0;
              s4 += v[k];
            }
            int x = s4;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
              const int y = __shfl_up_sync(0xffffffffu, x, off);
              if (lane >= off) x += y;
            }
            int run = x - s4;
#pragma unroll
            for (int k = 0; k < 4; k++) {
              const int i = 4 * lane + k;
              if (i < WPT * NWARP) sh.scan[i] = run;
              run += v[k];
            }
          }
          __syncthreads();
#pragma unroll
          for (int j = 0; j < WPT; j++)
            excl[j] += cur + pre + sh.scan[j * NWARP + warp];  // running cut before word j
          int lmax = INT_MIN;
#pragma unroll
          for (int j = 0; j < WPT; j++)
            if (own[j]) lmax = max(lmax, excl[j] + WS(j));
          lmax = __reduce_max_sync(0xffffffffu, lmax);
          const int thr = max(best + 1, lmax);
          bool cand = false;
#pragma unroll
          for (int j = 0; j < WPT; j++) {
            if (own[j]) aprev[j * NT + tid] = A[j];
            if (own[j] && WP(j) > 0 && excl[j] + WP(j) >= thr) cand = true;
          }
          long long key = LLONG_MIN;
          if (__syncthreads_or(cand)) {
#pragma unroll
            for (int j = 0; j < WPT; j++) {
              if (!own[j] || WP(j) <= 0 || excl[j] + WP(j) < thr) continue;
              // classes of the pre-phase word (neighbours as during the update)
              const int wl = j * NT + tid, lr = lr0 + j * (NT / WPR);
              const uint32_t Sold = cur_w[j] ^ A[j];
              const uint32_t same = oth_w[j];
              const uint32_t x = so_cy[j * NT];
              const uint32_t shv =
                  lop3<0xEA>(__funnelshift_l(same, same, rot), VG, (x << ca) >> cb);
              const uint32_t up = lr == 0 ? stash[w] : so_up[j * NT];
              const uint32_t dn = lr == R - 1 ? stash[WPR + w] : so_dn[j * NT];
              const uint2 m2 = ms[j * NT];
              const Classes c = classes_pad(Sold, same, shv, up, dn,
                                            make_uint4(m2.x, m2.y, mu[j * NT], md[j * NT]));
              const uint32_t Aj = A[j];
              const uint32_t P2 = Aj & c.k3, P4m = Aj & c.k4, N2 = Aj & c.km2, N4 = Aj & c.km4;
              int v = excl[j], mx = INT_MIN, mp = -1;
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
              const long long pos = (long long)(gw0 + wl) * 32 + mp;
              const long long kk = (long long)((unsigned long long)(long long)mx << 32) |
                                   (long long)(0xFFFFFFFFu - (uint32_t)pos);
              key = kk > key ? kk : key;
            }
            key = warp_max_key(key);
            if (lane == 0) sh.kred[warp] = key;
            __syncthreads();
            key = warp_max_key(lane < NWARP ? sh.kred[lane] : LLONG_MIN);
          }
          if (tid < C) *cl.map_shared_rank(&sh.keys[slot][q], tid) = key;
        }
#undef WS
#undef WP
        pend_prev = pend;
        cur += D;
#pragma unroll
        for (int j = 0; j < WPT; j++) {  // next phase updates the other colour
          const uint32_t tmp = cur_w[j];
          cur_w[j] = oth_w[j];
          oth_w[j] = tmp;
        }
      }
      executed = t + 1;
      if (!SA && !sweep_flipped) break;
    }
    // ---- resolve the last half-sweep (its colour is now oth_w; no flips since)
    cl_arrive_wait();
    if (pend_prev) {
      uint32_t zero[WPT];
#pragma unroll
      for (int j = 0; j < WPT; j++) zero[j] = 0;
      resolve((hs - 1) & 1, oth_w, cur_w, zero, (hs - 1) & 1);
    }
    cl_arrive_wait();  // snapshots visible to the neighbours

    // ---- integrity guard (solvers.py:132-133): recompute the cut of best
    {
      const uint32_t *up_row = cl.map_shared_rank(bst, qu) + RW + (Ru - 1) * WPR;
      const uint32_t *dn_row = cl.map_shared_rank(bst, qd) + RW;
      // band_cut indexes s1p[lr * WPR + cw] and s1p[wl -/+ WPR] inside the band
      const int cb = band_cut(bst, bst + RW, up_row, dn_row);
      const int wsum2 = (int)__reduce_add_sync(0xffffffffu, (unsigned)cb);
      if (lane == 0) sh.redD[warp] = wsum2;
      __syncthreads();
      if (warp == 0) {
        int s = lane < NWARP ? sh.redD[lane] : 0;
        s = (int)__reduce_add_sync(0xffffffffu, (unsigned)s);
        if (lane < C) *cl.map_shared_rank(&sh.ipart[1][q], lane) = s;
      }
    }
    cl_arrive_wait();
    if (q == 0 && tid == 0) {
      int cbest = 0;
      for (int i = 0; i < C; i++) cbest += sh.ipart[1][i];
      a.best_cut[trial] = best;
      a.sweeps_exec[trial] = executed;
      if (cbest != best) atomicExch(a.err, GSB_EINTEGRITY);
      atomicAdd(a.blocks, 2ull * nw + (SA ? 4ull * nw * (unsigned long long)executed : 0ull));
    }
    // ---- pack best spins MSB-first by site id: bytes whose first site is in
    // this band (the last few bits may come from the next CTA's band)
    {
      const long long n = (long long)rows * a.cols;
      const long long x0 = (long long)r0 * a.cols, x1 = (long long)(r0 + R) * a.cols;
      const uint32_t *bnext = cl.map_shared_rank(bst, qd);
      uint8_t *out = a.best_bits + (size_t)trial * a.nbytes;
      for (long long byte = (x0 + 7) / 8 + tid; byte < (x1 + 7) / 8; byte += NT) {
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < 8; b++) {
          const long long x = byte * 8 + b;
          uint32_t bit = 0;
          if (x < n) {
            const int r = (int)(x / a.cols), c = (int)(x - (long long)r * a.cols);
            const int p = (r + c) & 1, k = c >> 1;
            const uint32_t *src = x < x1 ? bst + (r - r0) * WPR : bnext + (r - r0 - R) * WPR;
            bit = (src[p * RW + (k >> 5)] >> (k & 31)) & 1u;
          }
          v |= bit << (7 - b);
        }
        out[byte] = (uint8_t)v;
      }
    }
    cl_arrive_wait();  // the next trial overwrites halos and snapshots
  }
  {
    const unsigned long long nb = __reduce_add_sync(0xffffffffu, tail_blocks);
    if (lane == 0 && nb) atomicAdd(a.blocks, nb);
  }
}

// ------------------------------------------------------------------ host
static bool pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

static int max_smem_optin() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
      v = 0;
  }
  return v;
}

// words per thread for cluster size C (0 if the shape does not fit)
static int cluster_wpt(int rows, int cols, int C) {
  if ((rows & 1) || (cols & 1) || rows < 4 || cols < 8 || rows < C) return 0;
  int WPR, nw;
  checker_words(rows, cols, &WPR, &nw);
  if (!pow2(WPR) || WPR > CL_NT / 2) return 0;
  const int RJ = CL_NT / WPR;
  const int Rmax = (rows + C - 1) / C;
  const int wpt = (Rmax + RJ - 1) / RJ;
  if (wpt > 8) return 0;
  if ((long long)nw * 32 >= 0xFFFFFFFFll) return 0;
  const size_t smem = cl_layout(Rmax, WPR, wpt).total;
  if (smem + sizeof(ClShared) > (size_t)max_smem_optin()) return 0;
  return wpt;
}

bool checker_cluster_fits(int rows, int cols) {
  for (int C = 1; C <= CL_MAXC; C *= 2)
    if (cluster_wpt(rows, cols, C)) return true;
  return false;
}

size_t checker_cluster_workspace_bytes(int rows, int cols) {
  int WPR, nw;
  checker_words(rows, cols, &WPR, &nw);
  return align_up((size_t)2 * nw * 16, 256) + align_up((size_t)nw * 16, 256);
}

template <int WPT, bool SA>
static int cl_configure(int C, size_t smem, int *max_clusters) {
  auto kern = checker_cluster_kernel<WPT, SA>;
  if (allow_dynamic_smem((const void *)kern, smem) != cudaSuccess)
    return set_error(GSB_ECUDA, "cudaFuncSetAttribute(smem) failed");
  if (C > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                   cudaSuccess)
    return set_error(GSB_ECUDA, "non-portable cluster size not allowed");
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(CL_NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, (void *)kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  *max_clusters = n;
  return GSB_OK;
}

template <int WPT, bool SA>
static int cl_launch(const ClusterArgs &a, size_t smem, int nclusters, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = a.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(nclusters * a.C, 1, 1);
  cfg.blockDim = dim3(CL_NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, checker_cluster_kernel<WPT, SA>, a);
  if (e != cudaSuccess) return set_error(GSB_ECUDA, cudaGetErrorString(e));
  return GSB_OK;
}

template <int WPT>
static int cl_dispatch(ClusterArgs a, bool sa, int T, cudaStream_t stream, bool query_only,
                       int *max_clusters) {
  const int Rmax = (a.rows + a.C - 1) / a.C;
  const size_t smem = cl_layout(Rmax, a.WPR, WPT).total;
  int rc = sa ? cl_configure<WPT, true>(a.C, smem, max_clusters)
              : cl_configure<WPT, false>(a.C, smem, max_clusters);
  if (rc != GSB_OK || query_only) return rc;
  if (*max_clusters < 1) return set_error(GSB_EUNSUPPORTED, "cluster does not fit on the GPU");
  const int ncl = T < *max_clusters ? T : *max_clusters;
  return sa ? cl_launch<WPT, true>(a, smem, ncl, stream) : cl_launch<WPT, false>(a, smem, ncl, stream);
}

static int cl_run_wpt(int wpt, const ClusterArgs &a, bool sa, int T, cudaStream_t stream,
                      bool query_only, int *max_clusters) {
  switch (wpt) {
    case 1: return cl_dispatch<1>(a, sa, T, stream, query_only, max_clusters);
    case 2: return cl_dispatch<2>(a, sa, T, stream, query_only, max_clusters);
    case 3: return cl_dispatch<3>(a, sa, T, stream, query_only, max_clusters);
    case 4: return cl_dispatch<4>(a, sa, T, stream, query_only, max_clusters);
    case 5: return cl_dispatch<5>(a, sa, T, stream, query_only, max_clusters);
    case 6: return cl_dispatch<6>(a, sa, T, stream, query_only, max_clusters);
    case 7: return cl_dispatch<7>(a, sa, T, stream, query_only, max_clusters);
    default: return cl_dispatch<8>(a, sa, T, stream, query_only, max_clusters);
  }
}

static int g_force_cluster = 0;  // test-only override (gsb_test_cluster_size)

void checker_cluster_force_size(int c) { g_force_cluster = c; }

int checker_cluster_run(int rows, int cols, const int8_t *w_dev, int kind, int sweeps,
                        const uint64_t *table, const uint64_t *seeds, int T, int64_t *best_cut,
                        int32_t *sweeps_exec, uint8_t *best_bits, void *ws, int *err_ws,
                        cudaStream_t stream) {
  int WPR, nw;
  checker_words(rows, cols, &WPR, &nw);
  uint4 *masks = (uint4 *)ws;
  uint4 *geo = (uint4 *)((char *)ws + align_up((size_t)2 * nw * 16, 256));
  checker_masks_kernel_launch(rows, cols, WPR, w_dev, masks, geo, stream);
  ClusterArgs a;
  a.rows = rows;
  a.cols = cols;
  a.H = cols / 2;
  a.WPR = WPR;
  a.nw = nw;
  a.masks = masks;
  a.table = table;
  a.sweeps = sweeps;
  a.seeds = seeds;
  a.T = T;
  a.best_cut = best_cut;
  a.sweeps_exec = sweeps_exec;
  a.best_bits = best_bits;
  a.nbytes = (rows * cols + 7) / 8;
  a.err = err_ws;
  a.blocks = (unsigned long long *)((char *)err_ws + 8);
  const bool sa = kind == GSB_ANNEALING;
  // cluster size: the one that keeps the most SMs busy with these T trials
  // (ties -> the smaller cluster); gsb_test_cluster_size forces one (tests)
  int bestC = 0, bestUsed = -1;
  const int forced = g_force_cluster;
  for (int C = 1; C <= CL_MAXC; C *= 2) {
    if (forced && C != forced) continue;
    const int wpt = cluster_wpt(rows, cols, C);
    if (!wpt) continue;
    a.C = C;
    int mc = 0;
    if (cl_run_wpt(wpt, a, sa, T, stream, true, &mc) != GSB_OK || mc < 1) continue;
    const int used = (T < mc ? T : mc) * C;
    if (used > bestUsed) {
      bestUsed = used;
      bestC = C;
    }
  }
  if (!bestC) return set_error(GSB_EUNSUPPORTED, "torus does not fit the cluster engine");
  a.C = bestC;
  int mc = 0;
  const int rc = cl_run_wpt(cluster_wpt(rows, cols, bestC), a, sa, T, stream, false, &mc);
  if (getenv("GSB_VERBOSE"))
    fprintf(stderr, "gsb cluster engine: %dx%d C=%d WPT=%d clusters=%d smem=%zu\n", rows, cols,
            bestC, cluster_wpt(rows, cols, bestC), mc < T ? mc : T,
            cl_layout((rows + bestC - 1) / bestC, WPR, cluster_wpt(rows, cols, bestC)).total);
  return rc;
}

}  // namespace gsb
