// checker.cu -- checkerboard (Philox) sweep engine for +-1 tori that fit in
// shared memory (BASELINE configs 1-4).
//
// Semantics: gsetbench.solvers.run_trial (solvers.py:91-140) with the two
// changes of the checkerboard contract (executable form
// oracle/gsb_oracle.c:trial_checker): sites are visited colour 0 then colour 1,
// each in increasing id, and every random draw is a counter-based Philox4x32-10
// word keyed by the trial seed.  Same-colour sites share no edge, so one
// half-sweep is computed in parallel and is exactly the sequential visit.
//
// Layout (per trial): spins bit-packed per colour, per row:
//   word (p, wi = r*WPR + w) bit b  <->  site (r, c = 2k + ((r+p)&1)), k = 32w+b,
//   H = cols/2 sites per row per colour, WPR = ceil(H/32), padding bits 0.
// One CTA runs one trial at a time (persistent over trials).  Thread `tid`
// owns words wi = j*NT + tid (j < WPT) of BOTH colours and keeps them in
// registers; shared memory holds the copy its neighbours read and the
// best-so-far snapshot.  The instance tables (coupling sign planes, neighbour
// offsets) are the same for every trial and are read through the L1, which
// all CTAs on an SM share.
//
// Per word and half-sweep: 4 positive-term planes P_j = ~(S^N_j^NEG_j),
// bit-sliced counts -> Delta classes, then for the Delta<0 sites a bit-sliced
// comparison (borrow chain) of the 32-bit uniform with K = ceil(exp(Delta/T)*2^32):
// uniform bits 31..24 are 8 Philox planes (two calls per word, unconditional);
// sites still undecided after them take bits 23..0 from a per-site Philox word
// (contract v2), drawn for the whole warp in one cooperative round.
//
// Best-so-far (solvers.py:125-127) per half-sweep: the running cut in visit
// order is cur + prefix sum of the accepted Deltas; a block reduction gives the
// half-sweep total and the sum of positive Deltas, which bounds every prefix.
// Only if that bound can beat `best` are per-word prefix bounds formed, and
// only candidate words run the exact bit-serial maximum; the first position of
// the maximum defines the snapshot (pre-phase words + accepted flips up to it).
#include <climits>
#include <cstdlib>
#include <cstdint>
#include <type_traits>

#include "checker_common.cuh"
#include "gsb_device.cuh"
#include "gsb_internal.h"

namespace gsb {

// Setup tables (shared by every trial on this instance):
//   masks[2][nw] uint4 {NS, NSH, NU, ND}: bit = coupling weight is -1, for the
//     same-k / shifted / up / down neighbour of each site of word (p, wi);
//   geo[nw] uint4 {up | dn<<16, cidx0 | cidx1<<16, cinfo0 | cinfo1<<16, valid}:
//     neighbour word indices, carry word + bit info of the shifted neighbour
//     per colour, valid-bit mask (same for both colours).
__global__ void checker_masks_kernel(int rows, int cols, int WPR, const int8_t *__restrict__ w,
                                     uint4 *__restrict__ masks, uint4 *__restrict__ geo) {
  const int H = cols >> 1;
  const int nw = rows * WPR;
  const int lb = (H - 1) & 31;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < 2 * nw;
       idx += gridDim.x * blockDim.x) {
    const int p = idx / nw, wi = idx % nw;
    const int r = wi / WPR, ww = wi % WPR;
    const int e = (r + p) & 1;
    uint32_t ns = 0, nsh = 0, nu = 0, nd = 0, v = 0;
    for (int b = 0; b < 32; b++) {
      const int k = ww * 32 + b;
      if (k >= H) break;
      const int c = 2 * k + e;
      const int x = r * cols + c;
      const int cl = (c + cols - 1) % cols;
      const int ru = (r + rows - 1) % rows;
      const int8_t w_right = w[2 * x], w_down = w[2 * x + 1];
      const int8_t w_left = w[2 * (r * cols + cl)];
      const int8_t w_up = w[2 * (ru * cols + c) + 1];
      // e==0: same-k other-colour word is the right neighbour, shifted is left
      // e==1: same-k is the left neighbour, shifted is right
      const int8_t wsame = e == 0 ? w_right : w_left;
      const int8_t wsh = e == 0 ? w_left : w_right;
      v |= 1u << b;
      if (wsame < 0) ns |= 1u << b;
      if (wsh < 0) nsh |= 1u << b;
      if (w_up < 0) nu |= 1u << b;
      if (w_down < 0) nd |= 1u << b;
    }
    // padding bits: NU/ND set, NS/NSH clear -> a padding site (spin and
    // neighbours 0) sees exactly two positive terms (classes_pad)
    masks[idx] = make_uint4(ns, nsh, nu | ~v, nd | ~v);
    if (p == 0) {
      uint32_t cidx[2], cinfo[2];
      for (int q = 0; q < 2; q++) {
        if (((r + q) & 1) == 0) {  // k-1 neighbour: carry from the previous word (or row end)
          cidx[q] = ww > 0 ? wi - 1 : r * WPR + WPR - 1;
          cinfo[q] = (uint32_t)(ww > 0 ? 31 : lb);
        } else {  // k+1 neighbour: carry from the next word (or row start)
          cidx[q] = ww < WPR - 1 ? wi + 1 : r * WPR;
          cinfo[q] = ((uint32_t)(ww < WPR - 1 ? 31 : lb) << 5) | (1u << 10);
        }
      }
      const uint32_t up = (r == 0 ? rows - 1 : r - 1) * WPR + ww;
      const uint32_t dn = (r == rows - 1 ? 0 : r + 1) * WPR + ww;
      geo[wi] = make_uint4(up | (dn << 16), cidx[0] | (cidx[1] << 16), cinfo[0] | (cinfo[1] << 16),
                           v);
    }
  }
}

// Per-colour neighbour table for the sweep kernel, geo2[p][wi] = two uint4:
//   {up, down, carry word: byte offsets into the spin copy of colour p^1
//    (relative to st), V},
//   {VG, r, a, b}: the shifted neighbour is rot(same, r) & VG | (x << a) >> b,
//    x = the carry word; r = 1 (k-1 neighbour) or 31 (k+1, a right rotate),
//    VG = V minus the bit the rotate wraps around, a = 31 - src bit,
//    b = 31 - dst bit (the carry lands on exactly one valid bit).
// Read through the L1 (shared by every CTA on the SM), not staged per CTA.
__global__ void checker_geo2_kernel(int nw, const uint4 *__restrict__ geo, uint4 *__restrict__ geo2) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < 2 * nw;
       idx += gridDim.x * blockDim.x) {
    const int p = idx / nw, wi = idx % nw;
    const uint4 g = geo[wi];
    const uint32_t base = (uint32_t)((p ^ 1) * nw);
    const uint32_t cidx = p ? (g.y >> 16) : (g.y & 0xFFFFu);
    const uint32_t cinfo = p ? (g.z >> 16) : (g.z & 0xFFFFu);
    const uint32_t src = cinfo & 31u, dst = (cinfo >> 5) & 31u, dir = (cinfo >> 10) & 1u;
    geo2[2 * idx] = make_uint4((base + (g.x & 0xFFFFu)) * 4u, (base + (g.x >> 16)) * 4u,
                               (base + cidx) * 4u, g.w);
    geo2[2 * idx + 1] = make_uint4(g.w & ~(dir ? 0x80000000u : 1u), dir ? 31u : 1u, 31u - src,
                                   31u - dst);
  }
}

struct CheckerArgs {
  int rows, cols, H, WPR, nw, lb;
  const uint4 *masks;
  const uint4 *geo;
  const uint4 *geo2;
  const uint64_t *table;  // [S][4]
  int sweeps;
  const uint64_t *seeds;
  int T;
  int64_t *best_cut;
  int32_t *sweeps_exec;
  uint8_t *best_bits;
  int nbytes;
  int *err;
  unsigned long long *blocks;  // Philox blocks drawn (statistics, workspace)
  int zp_max;                  // largest comparator specialisation used (8; dev knob)
};


// MINB = resident CTAs per SM the register budget is cut for: 16 warps per
// SM by default, 8 for one-warp teams whose trials cannot fill more (twice
// the registers per lane for interleaving the word bodies).
template <int NT, int WPT, bool SA, int MINB>
__global__ void __launch_bounds__(NT, MINB) checker_sweep_kernel(CheckerArgs a) {
  constexpr int NWARP = NT / 32;
  static_assert(WPT <= 8, "tail items pack (lane, word) as lane << 3 | j");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nw = a.nw;
  // instance tables (identical for every trial) are read through the L1
  const uint4 *__restrict__ msk = a.masks;        // [2][nw]
  const uint4 *__restrict__ geo = a.geo;          // [nw]
  const uint4 *__restrict__ geo2 = a.geo2;        // [2][nw][2]
  // per-trial Philox precomputation of the plane blocks (philox10_from2):
  // tabP[p][wi] = M0*x2 of (wi, q = 2p) and (wi, q = 2p + 1), tabW[wi] = (c1, c2);
  // each thread reads only the entries of its own words
  uint4 *tabP = (uint4 *)smem_raw;                // [2][nw]
  uint2 *tabW = (uint2 *)(tabP + 2 * nw);         // [nw]
  uint32_t *st = (uint32_t *)(tabW + nw);         // [2][nw] neighbour copy
  uint32_t *bst = st + 2 * nw;                    // [2][nw] best snapshot
  uint32_t *tx = bst + 2 * nw;                    // [NWARP][3][WPT][32] tail exchange
  uint32_t *tq = tx + NWARP * 3 * WPT * 32;       // [NWARP][32] tail queue
  int *red = (int *)(tq + NWARP * 32);            // [2 buffers][2][NWARP]
  int *red2 = red + 4 * NWARP;                    // [2][NWARP]
  int *scan = red2 + 2 * NWARP;                   // [WPT][NWARP]
  long long *kred = (long long *)(scan + ((WPT * NWARP + 1) & ~1));  // [NWARP]
  unsigned *wctrs = (unsigned *)(kred + NWARP);    // [NWARP] tail slot counters

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  uint32_t *teq = tx + warp * 3 * WPT * 32;  // [WPT][32] pending masks
  uint32_t *tc2 = teq + WPT * 32;            // [WPT][32] class -2 masks
  uint32_t *tlt = tc2 + WPT * 32;            // [WPT][32] accepted-by-tail bits
  uint32_t *myq = tq + warp * 32;
  unsigned *wctr = wctrs + warp;

  for (int i = tid; i < NWARP * 3 * WPT * 32; i += NT) tx[i] = 0;
  if (tid < NWARP) wctrs[tid] = 0;
  __syncthreads();

  bool own[WPT];
#pragma unroll
  for (int j = 0; j < WPT; j++) own[j] = j < WPT - 1 || j * NT + tid < nw;  // WPT = ceil(nw/NT)

  unsigned tail_blocks = 0;
  for (int trial = blockIdx.x; trial < a.T; trial += gridDim.x) {
    const uint64_t seed = a.seeds[trial];
    const uint32_t key0 = (uint32_t)seed, key1 = (uint32_t)(seed >> 32);

    // ---- initial spins: bit (k&31) of word 0 of Philox(key, (wi, 0, p, 0))
    uint32_t cur_w[WPT], oth_w[WPT];  // owned words of the colour being updated / the other
#pragma unroll
    for (int j = 0; j < WPT; j++) {
      const int wi = j * NT + tid;
      cur_w[j] = oth_w[j] = 0;
      if (own[j]) {
        const uint32_t V = geo[wi].w;
#pragma unroll
        for (int p = 0; p < 2; p++) {
          const P4 o = philox10(P4{(uint32_t)wi, 0u, (uint32_t)p, 0u}, key0, key1);
          const uint32_t s0 = o.x & V;
          if (p == 0) cur_w[j] = s0; else oth_w[j] = s0;
          st[p * nw + wi] = s0;
          bst[p * nw + wi] = s0;
        }
        if (SA) {
          uint32_t h1z, a0, b0, a1, b1;
          const PhiloxWord pw = philox_word((uint32_t)wi, key0, key1, h1z);
          tabW[wi] = make_uint2(pw.c1, pw.c2);
#pragma unroll
          for (int p = 0; p < 2; p++) {
            philox_pre(h1z, 2u * p, key0, a0, b0);
            philox_pre(h1z, 2u * p + 1u, key0, a1, b1);
            tabP[p * nw + wi] = make_uint4(a0, b0, a1, b1);
          }
        }
      }
    }
    __syncthreads();

    // ---- initial cut (every edge has exactly one colour-0 endpoint)
    int c0 = 0;
#pragma unroll
    for (int j = 0; j < WPT; j++) {
      if (own[j]) {
        const int wi = j * NT + tid;
        const uint4 g = geo[wi];
        const uint32_t *o = st + nw;
        const uint32_t sh = shifted_nb(o, oth_w[j], g.y & 0xFFFFu, g.z & 0xFFFFu);
        c0 += word_cut(cur_w[j], oth_w[j], sh, o[g.x & 0xFFFFu], o[g.x >> 16], msk[wi], g.w);
      }
    }
    c0 = (int)__reduce_add_sync(0xffffffffu, (unsigned)c0);
    if (lane == 0) red2[warp] = c0;
    __syncthreads();
    int cur = 0;
#pragma unroll
    for (int i = 0; i < NWARP; i++) cur += red2[i];
    int best = cur;
    int executed = 0;
    int buf = 0;

    for (int t = 0; t < a.sweeps; t++) {
      // K >= 2^32 (always accept) is emulated exactly by K_hi = 0xFF and a
      // tail threshold of 2^24 (every tie accepts); K = 0 (never) drops the
      // class from the pending sites (me = 0), so it draws nothing.
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
      // comparator specialisation (uniform per sweep), where registers allow
      // the extra code paths (measured, tools/zp_ab.py): 256 registers
      // (config 2) L <= 8, +3.5 %; 128 registers and <= 5 words per lane
      // (configs 1, 3) L <= 4, +2 %; 7 words at 128 registers (config 4):
      // none (the specialised bodies spill, -10 %).
      constexpr int kZp = !SA ? 0 : 65536 / (NT * MINB) >= 200 ? 8 : WPT <= 5 ? 4 : 0;
      const int zp = kZp ? min(min(zero_planes(K2, K4), a.zp_max), kZp) : 0;
      bool sweep_flipped = false;
#pragma unroll 1
      for (int p = 0; p < 2; p++, buf ^= 1) {
        uint32_t A[WPT], c2[WPT], eq[WPT], lt[WPT];
        int wpos[WPT], wsum[WPT];
        // rounds 0-1 of the plane blocks that depend only on (t, q): uniform
        uint32_t u1a = 0, va = 0, u1b = 0, vb = 0;
        if (SA) {
          philox_uni((uint32_t)t, 2u * p, key0, key1, u1a, va);
          philox_uni((uint32_t)t, 2u * p + 1u, key0, key1, u1b, vb);
        }
        // ---- pass 1: classes and the unconditional planes 0-7.  Words j <
        // WPT-1 are owned by every lane (the launch picks WPT = ceil(nw/NT)),
        // so only the last one is guarded and the bodies schedule together.
        auto pass1 = [&](auto Lc) {
          constexpr int L = decltype(Lc)::value;
#pragma unroll
          for (int j = 0; j < WPT; j++) {
            const int wi = j * NT + tid;
            A[j] = c2[j] = eq[j] = lt[j] = 0;
            wpos[j] = wsum[j] = 0;
            if (j < WPT - 1 || own[j]) {
              const uint4 ga = __ldg(&geo2[2 * (p * nw + wi)]);
              const uint4 gb = __ldg(&geo2[2 * (p * nw + wi) + 1]);
              const uint4 m = __ldg(&msk[p * nw + wi]);
              const uint32_t same = oth_w[j];
              const uint32_t sh = shifted_nb2(st, same, ga, gb);
              const Classes c =
                  classes_pad(cur_w[j], same, sh, word_at(st, ga.x), word_at(st, ga.y), m);
              wpos[j] = 2 * __popc(c.k3) + 4 * __popc(c.k4);
              if (SA) {
                A[j] = c.ge2 & ga.w;
                wsum[j] = wpos[j];  // minus the accepted Delta<0 flips at commit
                const uint32_t e2 = c.km2 & me2, e4 = c.km4 & me4;
                c2[j] = e2;
                // Philox(key, (wi, t, 2p + j, 1)), j = 0, 1, from round 2 on
                const uint4 pre = tabP[p * nw + wi];
                const uint2 pwv = tabW[wi];
                const PhiloxWord pw{pwv.x, pwv.y};
                const P4 r0 = philox10_from2(pw, pre.x, pre.y, u1a, va, key0, key1);
                const P4 r1 = philox10_from2(pw, pre.z, pre.w, u1b, vb, key0, key1);
                cmp_planes<L>(r0, r1, e2, e2 | e4, K2, K4, eq[j], lt[j]);
              } else {
                A[j] = c.k3 | c.k4;
                wsum[j] = wpos[j];
              }
            }
          }
        };
        if (kZp >= 8 && zp == 8) pass1(std::integral_constant<int, 8>{});
        else if (kZp >= 4 && zp == 4) pass1(std::integral_constant<int, 4>{});
        else pass1(std::integral_constant<int, 0>{});

        // ---- pass 2 (SA): warp-cooperative tail.  Undecided sites take bits
        // 23..0 of their uniform from a per-site Philox word; the warp shares
        // out the words that hold undecided sites (items), 32 per round, and
        // each item walks its 4-site groups (one Philox block per group).
        if (SA) {
          uint32_t wm = 0;  // bit j: word j has undecided sites
#pragma unroll
          for (int j = 0; j < WPT; j++) wm |= (eq[j] != 0u ? 1u : 0u) << j;
          if (__any_sync(0xffffffffu, wm != 0u)) {
#pragma unroll
            for (int j = 0; j < WPT; j++) {
              if (eq[j]) {
                teq[j * 32 + lane] = eq[j];
                tc2[j * 32 + lane] = c2[j];
              }
            }
            // slots come from a per-warp counter that only grows (wbase = its
            // value when this tail started); the total from one REDUX
            const unsigned wbase = *wctr;
            uint32_t rem = wm;
#pragma unroll 1
            for (unsigned done = 0;;) {
              const int cnt = __popc(rem);
              const int total = (int)__reduce_add_sync(0xffffffffu, (unsigned)cnt);
              if (total == 0) break;
              const int sbase = (int)((cnt ? atomicAdd(wctr, (unsigned)cnt) : 0u) - wbase - done);
              int slot = sbase;
              while (rem && slot < 32) {
                const int jj = __ffs(rem) - 1;
                rem &= rem - 1;
                myq[slot++] = ((uint32_t)lane << 3) | (uint32_t)jj;
              }
              __syncwarp();
              if (lane < total) {
                const uint32_t it = myq[lane];
                const int ol = (int)(it >> 3), jj = (int)(it & 7u);
                const uint32_t wi = (uint32_t)(jj * NT + warp * 32 + ol);
                uint32_t e = teq[jj * 32 + ol];
                const uint32_t cw = tc2[jj * 32 + ol];
                uint32_t acc = 0;
                while (e) {
                  const int g4 = (__ffs(e) - 1) & ~3;  // 4 * group
                  const P4 r = philox10(P4{wi, (uint32_t)t, (uint32_t)(4 + 8 * p + (g4 >> 2)), 1u},
                                        key0, key1);
                  tail_blocks++;
                  const uint32_t en = (e >> g4) & 0xFu, cn = (cw >> g4) & 0xFu;
                  const uint32_t tw[4] = {r.x, r.y, r.z, r.w};
                  uint32_t ln = 0;
#pragma unroll
                  for (int q = 0; q < 4; q++) {
                    const uint32_t klo = ((cn >> q) & 1u) ? K2lo : K4lo;
                    if (((en >> q) & 1u) && (tw[q] >> 8) < klo) ln |= 1u << q;
                  }
                  acc |= ln << g4;
                  e &= ~(0xFu << g4);
                }
                tlt[jj * 32 + ol] = acc;  // one item per (word, lane): plain store
              }
              __syncwarp();
              done += (unsigned)total;
            }
#pragma unroll
            for (int j = 0; j < WPT; j++)
              if (eq[j]) lt[j] |= tlt[j * 32 + lane];
          }
        }
        // ---- pass 3: commit the flips
        int dsum = 0, psum = 0;
#pragma unroll
        for (int j = 0; j < WPT; j++) {
          if (own[j]) {
            const int wi = j * NT + tid;
            if (SA) {
              wsum[j] -= 2 * __popc(lt[j] & c2[j]) + 4 * __popc(lt[j] & ~c2[j]);
              A[j] |= lt[j];
            }
            cur_w[j] ^= A[j];
            st[p * nw + wi] = cur_w[j];
            dsum += wsum[j];
            psum += wpos[j];
          }
        }
        // ---- block reduction of (dsum, psum): REDUX per warp, one barrier
        const int wd = (int)__reduce_add_sync(0xffffffffu, (unsigned)dsum);
        const int wp = (int)__reduce_add_sync(0xffffffffu, (unsigned)psum);
        int D = wd, Pt = wp;
        if (NWARP > 1) {
          int *rb = red + buf * 2 * NWARP;
          if (lane == 0) {
            rb[warp] = wd;
            rb[NWARP + warp] = wp;
          }
          __syncthreads();
          D = 0;
          Pt = 0;
#pragma unroll
          for (int i = 0; i < NWARP; i++) {
            D += rb[i];
            Pt += rb[NWARP + i];
          }
        } else {
          __syncwarp();
        }
        if (Pt > 0) sweep_flipped = true;  // greedy flips are exactly the positive ones
        if (cur + Pt > best) {
          // ---- per-word prefix bounds; word order is (j, warp, lane)
          // Two words per scan: wsum + 128 is in [0, 256], so a 32-lane
          // prefix fits 16 bits (<= 8192) and pairs (j, j+1) share one scan.
          int excl[WPT];
          int rtot[WPT];
#pragma unroll
          for (int j = 0; j < WPT; j += 2) {
            const bool two = j + 1 < WPT;
            uint32_t x = (uint32_t)(wsum[j] + 128) |
                         (two ? (uint32_t)(wsum[two ? j + 1 : j] + 128) << 16 : 0u);
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
              const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
              if (lane >= off) x += y;
            }
            const uint32_t tot = __shfl_sync(0xffffffffu, x, 31);
            const int bias = 128 * (lane + 1);
            excl[j] = (int)(x & 0xFFFFu) - bias - wsum[j];
            rtot[j] = (int)(tot & 0xFFFFu) - 4096;
            if (two) {
              excl[j + 1] = (int)(x >> 16) - bias - wsum[j + 1];
              rtot[j + 1] = (int)(tot >> 16) - 4096;
            }
          }
          if (NWARP > 1 && lane == 31) {
#pragma unroll
            for (int j = 0; j < WPT; j++) scan[j * NWARP + warp] = rtot[j];
          }
          if (NWARP > 1) __syncthreads();
          int basep = 0;
          bool cand = false;
#pragma unroll
          for (int j = 0; j < WPT; j++) {
            int wbase = basep;
            if (NWARP > 1) {
              for (int i = 0; i < NWARP; i++) {
                const int v = scan[j * NWARP + i];
                if (i < warp) wbase += v;
                basep += v;
              }
            } else {
              basep += rtot[j];
            }
            excl[j] += wbase;
          }
          // Every word end is an achieved value, so the maximum M is at least
          // the largest of them (Lmax; warp-local for larger teams), and a word
          // can hold a position of value >= Lmax only if its bound cur + excl +
          // wpos reaches Lmax.  Candidates: bound >= max(best + 1, Lmax).
          int lmax = INT_MIN;
#pragma unroll
          for (int j = 0; j < WPT; j++)
            if (own[j]) lmax = max(lmax, excl[j] + wsum[j]);
          lmax = __reduce_max_sync(0xffffffffu, lmax);
          const int thr = max(best + 1, cur + lmax);
#pragma unroll
          for (int j = 0; j < WPT; j++)
            if (own[j] && wpos[j] > 0 && cur + excl[j] + wpos[j] >= thr) cand = true;
          const bool anyc = NWARP > 1 ? __syncthreads_or(cand) : __any_sync(0xffffffffu, cand);
          if (anyc) {
            long long key = LLONG_MIN;
#pragma unroll
            for (int j = 0; j < WPT; j++) {
              if (!own[j] || wpos[j] <= 0 || cur + excl[j] + wpos[j] < thr) continue;
              // recompute the classes of the pre-phase word (neighbours unchanged)
              const int wi = j * NT + tid;
              const uint4 ga = __ldg(&geo2[2 * (p * nw + wi)]);
              const uint4 gb = __ldg(&geo2[2 * (p * nw + wi) + 1]);
              const uint32_t Sold = cur_w[j] ^ A[j];
              const uint32_t same = oth_w[j];
              const uint32_t sh = shifted_nb2(st, same, ga, gb);
              const Classes c = classes_pad(Sold, same, sh, word_at(st, ga.x), word_at(st, ga.y),
                                            __ldg(&msk[p * nw + wi]));
              const uint32_t Aj = A[j];
              const uint32_t P2 = Aj & c.k3, P4m = Aj & c.k4, N2 = Aj & c.km2, N4 = Aj & c.km4;
              int v = cur + excl[j], mx = INT_MIN, mp = -1;
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
              const long long pos = (long long)wi * 32 + mp;
              const long long kk = (long long)((unsigned long long)(long long)mx << 32) |
                                   (long long)(0xFFFFFFFFu - (uint32_t)pos);
              key = kk > key ? kk : key;
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
              const long long y = __shfl_xor_sync(0xffffffffu, key, off);
              key = y > key ? y : key;
            }
            if (NWARP > 1) {
              if (lane == 0) kred[warp] = key;
              __syncthreads();
              key = LLONG_MIN;
#pragma unroll
              for (int i = 0; i < NWARP; i++) key = kred[i] > key ? kred[i] : key;
            }
            const int mval = (int)(key >> 32);
            if (key != LLONG_MIN && mval > best) {
              best = mval;
              const long long pos = 0xFFFFFFFFll - (key & 0xFFFFFFFFll);
              const int wstar = (int)(pos >> 5), bstar = (int)(pos & 31);
#pragma unroll
              for (int j = 0; j < WPT; j++) {
                if (!own[j]) continue;
                const int wi = j * NT + tid;
                const uint32_t now = cur_w[j], old = now ^ A[j];
                const uint32_t snap = wi < wstar    ? now
                                      : wi == wstar ? old ^ (A[j] & ((2u << bstar) - 1u))
                                                    : old;
                bst[p * nw + wi] = snap;
                bst[(p ^ 1) * nw + wi] = oth_w[j];
              }
            }
          }
        }
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

    // ---- integrity guard (solvers.py:132-133): recompute the cut of best
    __syncthreads();
    int cb = 0;
#pragma unroll
    for (int j = 0; j < WPT; j++) {
      if (own[j]) {
        const int wi = j * NT + tid;
        const uint4 g = geo[wi];
        const uint32_t *o = bst + nw;
        const uint32_t same = o[wi];
        const uint32_t sh = shifted_nb(o, same, g.y & 0xFFFFu, g.z & 0xFFFFu);
        cb += word_cut(bst[wi], same, sh, o[g.x & 0xFFFFu], o[g.x >> 16], msk[wi], g.w);
      }
    }
    cb = (int)__reduce_add_sync(0xffffffffu, (unsigned)cb);
    if (lane == 0) red2[NWARP + warp] = cb;
    __syncthreads();
    int cbest = 0;
#pragma unroll
    for (int i = 0; i < NWARP; i++) cbest += red2[NWARP + i];
    if (tid == 0) {
      a.best_cut[trial] = best;
      a.sweeps_exec[trial] = executed;
      if (cbest != best) atomicExch(a.err, GSB_EINTEGRITY);
    }
    {
      // Philox blocks of this trial: 2 init + 2 plane blocks per word and
      // half-sweep (SA) + the cooperative tail groups
      const unsigned long long nb = __reduce_add_sync(0xffffffffu, tail_blocks);
      if (lane == 0 && nb) atomicAdd(a.blocks, nb);
      if (tid == 0)
        atomicAdd(a.blocks, 2ull * nw + (SA ? 4ull * nw * (unsigned long long)executed : 0ull));
      tail_blocks = 0;
    }
    // ---- pack best spins MSB-first by site id
    uint8_t *out = a.best_bits + (size_t)trial * a.nbytes;
    const int n = a.rows * a.cols;
    for (int byte = tid; byte < a.nbytes; byte += NT) {
      uint32_t v = 0;
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const int x = byte * 8 + q;
        uint32_t bit = 0;
        if (x < n) {
          const int r = x / a.cols, c = x - r * a.cols;
          const int p = (r + c) & 1, k = c >> 1;
          bit = (bst[p * nw + r * a.WPR + (k >> 5)] >> (k & 31)) & 1u;
        }
        v |= bit << (7 - q);
      }
      out[byte] = (uint8_t)v;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ launch
static size_t smem_bytes(int nw, int NT, int WPT) {
  const int NWARP = NT / 32;
  size_t b = (size_t)2 * nw * 16 + (size_t)nw * 8;          // tabP, tabW
  b += (size_t)4 * nw * 4;                                  // st, bst
  b += (size_t)NWARP * 3 * WPT * 32 * 4 + (size_t)NWARP * 32 * 4;  // tail exchange + queue
  b += (size_t)(6 * NWARP) * 4;
  b += (size_t)((WPT * NWARP + 1) & ~1) * 4;
  b += (size_t)NWARP * 8 + (size_t)NWARP * 4;
  return b;
}

template <int NT, int WPT, int MINB = 512 / NT>
static int launch_nt(const CheckerArgs &a, bool sa, int nsm, cudaStream_t stream) {
  const size_t smem = smem_bytes(a.nw, NT, WPT);
  auto kern = sa ? checker_sweep_kernel<NT, WPT, true, MINB>
                 : checker_sweep_kernel<NT, WPT, false, MINB>;
  if (allow_dynamic_smem((const void *)kern, smem) != cudaSuccess)
    return set_error(GSB_ECUDA, "cudaFuncSetAttribute failed");
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem) != cudaSuccess ||
      per_sm < 1)
    return set_error(GSB_ECUDA, "checker kernel does not fit on an SM");
  int grid = nsm * per_sm;
  if (grid > a.T) grid = a.T;
  kern<<<grid, NT, smem, stream>>>(a);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(GSB_ECUDA, cudaGetErrorString(e));
  return GSB_OK;
}

int checker_words(int rows, int cols, int *WPR, int *nw) {
  const int H = cols / 2;
  *WPR = (H + 31) / 32;
  *nw = rows * *WPR;
  return 0;
}

bool checker_fits(int rows, int cols) {
  if ((rows & 1) || (cols & 1) || rows < 4 || cols < 4) return false;
  int WPR, nw;
  checker_words(rows, cols, &WPR, &nw);
  return nw <= 2048;
}

size_t checker_workspace_bytes(int rows, int cols) {
  int WPR, nw;
  checker_words(rows, cols, &WPR, &nw);
  return align_up((size_t)2 * nw * 16, 256) + align_up((size_t)nw * 16, 256) +
         align_up((size_t)2 * nw * 32, 256);
}

// test-only overrides (gsb_test_checker_shape): warps per trial (0 = automatic)
// and the one-warp variant (0 = automatic, 1 = 128-register, 2 = 8-per-SM 246-register)
static int g_force_warps = 0, g_force_variant = 0;

void checker_force_shape(int warps, int variant) {
  g_force_warps = warps;
  g_force_variant = variant;
}

template <int WPT>
static int launch_wpt(const CheckerArgs &a, bool sa, int nsm, int W, cudaStream_t stream) {
  switch (W) {
    case 1:
      if (g_force_variant ? g_force_variant == 2 : a.T <= 8 * nsm)
        return launch_nt<32, WPT, 8>(a, sa, nsm, stream);
      return launch_nt<32, WPT>(a, sa, nsm, stream);
    case 2: return launch_nt<64, WPT>(a, sa, nsm, stream);
    case 4: return launch_nt<128, WPT>(a, sa, nsm, stream);
    case 8: return launch_nt<256, WPT>(a, sa, nsm, stream);
    default: return launch_nt<512, WPT>(a, sa, nsm, stream);
  }
}

int checker_run(int rows, int cols, const int8_t *w_dev, int kind, int sweeps,
                const uint64_t *table, const uint64_t *seeds, int T, int64_t *best_cut,
                int32_t *sweeps_exec, uint8_t *best_bits, void *ws, int *err_ws,
                cudaStream_t stream) {
  int WPR, nw;
  checker_words(rows, cols, &WPR, &nw);
  const int nsm = num_sms();
  if (nsm <= 0) return set_error(GSB_ECUDA, "no CUDA device");
  uint4 *masks = (uint4 *)ws;
  uint4 *geo = (uint4 *)((char *)ws + align_up((size_t)2 * nw * 16, 256));
  uint4 *geo2 = (uint4 *)((char *)geo + align_up((size_t)nw * 16, 256));
  checker_masks_kernel<<<(2 * nw + 255) / 256, 256, 0, stream>>>(rows, cols, WPR, w_dev, masks,
                                                                 geo);
  CheckerArgs a;
  a.rows = rows;
  a.cols = cols;
  a.H = cols / 2;
  a.WPR = WPR;
  a.nw = nw;
  a.lb = (a.H - 1) & 31;
  checker_geo2_kernel<<<(2 * nw + 255) / 256, 256, 0, stream>>>(nw, geo, geo2);
  a.masks = masks;
  a.geo = geo;
  a.geo2 = geo2;
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
  a.zp_max = 8;
  const bool sa = kind == GSB_ANNEALING;
  // Team shape: W warps per trial (power of two), WPT <= 8 words per lane.
  // As few warps per trial as possible (a one-warp team needs no CTA barriers
  // at all; fewer, longer lanes have more ILP); grow the team only while the
  // words do not fit or the trials cannot give every SM at least two warps.
  int W = 1;
  while (W < 16 && 32 * W < nw &&
         ((long long)T * W < 2LL * nsm || (nw + 32 * W - 1) / (32 * W) > 8))
    W *= 2;
  if (g_force_warps) {
    const int w = g_force_warps;
    if (!((w == 1 || w == 2 || w == 4 || w == 8 || w == 16) && (nw + 32 * w - 1) / (32 * w) <= 8))
      return set_error(GSB_EUNSUPPORTED, "forced checkerboard team shape cannot hold the torus");
    W = w;
  }
  const int wpt = (nw + 32 * W - 1) / (32 * W);
  if (wpt > 8) return set_error(GSB_EUNSUPPORTED, "checkerboard team shape out of range");
  // the kernel relies on WPT == ceil(nw / NT) exactly (all but the last word owned)
  switch (wpt) {
    case 1: return launch_wpt<1>(a, sa, nsm, W, stream);
    case 2: return launch_wpt<2>(a, sa, nsm, W, stream);
    case 3: return launch_wpt<3>(a, sa, nsm, W, stream);
    case 4: return launch_wpt<4>(a, sa, nsm, W, stream);
    case 5: return launch_wpt<5>(a, sa, nsm, W, stream);
    case 6: return launch_wpt<6>(a, sa, nsm, W, stream);
    case 7: return launch_wpt<7>(a, sa, nsm, W, stream);
    default: return launch_wpt<8>(a, sa, nsm, W, stream);
  }
}

}  // namespace gsb

namespace gsb {
void checker_masks_kernel_launch(int rows, int cols, int WPR, const int8_t *w, uint4 *masks,
                                 uint4 *geo, cudaStream_t stream) {
  const int nw = rows * WPR;
  checker_masks_kernel<<<(2 * nw + 255) / 256, 256, 0, stream>>>(rows, cols, WPR, w, masks, geo);
}
}  // namespace gsb
