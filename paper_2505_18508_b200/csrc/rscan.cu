// rscan.cu -- random-scan (Philox) sweep engine for tori that fit one SM.
//
// The reference's sweep visits every site once in a fresh uniformly random
// order (gsetbench.solvers.run_trial, solvers.py:107-127).  This engine keeps
// that dynamics in law and makes it parallel: the order of sweep t is that of
// per-site Philox priorities (ties by site id), and the sweep runs level by
// level -- a site is visited in round r once every neighbour that precedes it
// has been visited in an earlier round.  Sites of one round share no edge, so
// a round is computed in parallel, and since any visit order that keeps every
// site after its preceding neighbours yields the same spins after each visit,
// the states at round boundaries and at the end of the sweep are exactly those
// of the sequential scan in priority order.  Executable form of the contract:
// oracle/gsb_oracle.c:trial_rscan:
//   initial spin of v: top bit of word (v & 3) of Philox(key, (v >> 2, 0, 0, 3));
//   priority of v at sweep t: word (v & 3) of Philox(key, (v >> 2, t, 0, 4));
//   uniform of v at sweep t:  word (v & 3) of Philox(key, (v >> 2, t, 1, 4)),
//   Delta < 0 accepted iff u < K = ceil(exp(Delta / T_t) * 2^32) (host table);
//   visit order (level, id); best-so-far on strict improvement in that order.
//
// Layout: one CTA runs one trial at a time (persistent over trials).  Thread
// `tid` owns the K = 32 * KW consecutive sites [tid * K, tid * K + K); shared
// memory holds the spins (int8), the round in which each site was visited this
// sweep (uint8), the preceding-neighbour mask (4 bits), the accepted Delta of
// the current round (int8), the priorities / uniforms (u32) and the best
// snapshot (bit-packed).  Couplings are read through the L1.
#include <climits>
#include <cstdint>

#include "gsb_device.cuh"
#include "gsb_internal.h"

namespace gsb {

constexpr int RS_MAXNT = 512;
constexpr int RS_NWARP = RS_MAXNT / 32;

struct RsArgs {
  int rows, cols, n, npad;
  uint32_t rdiv;  // ceil(2^32 / cols): v / cols == __umulhi(v, rdiv) for v < 2^17
  const int8_t *w;
  const uint64_t *table;  // [S][4]: K for Delta = -1..-4
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

struct RsShared {
  int red[2][3][RS_NWARP];  // [round parity][D, P, remaining][warp]
  int scan[RS_NWARP];
  long long kred[RS_NWARP];
};

__device__ __forceinline__ long long rs_warp_max_key(long long key) {
  const int hi = (int)(key >> 32);
  const int mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? (unsigned)key : 0u);
  return (long long)(((unsigned long long)(unsigned)mh << 32) | ml);
}

template <int KW, bool SA>
__global__ void __launch_bounds__(RS_MAXNT) rscan_kernel(RsArgs a) {
  constexpr int K = 32 * KW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ RsShared sh;
  const int n = a.n, npad = a.npad, cols = a.cols, rows = a.rows;
  uint32_t *pu = (uint32_t *)smem_raw;           // [npad] priorities, then uniforms
  uint32_t *bst = pu + npad;                     // [npad / 32] best snapshot bits
  uint32_t *cnt = bst + npad / 32;               // [npad / 8] 4-bit counts of unvisited preceding neighbours
  int8_t *s = (int8_t *)(cnt + npad / 8);        // [npad] spins +-1
  uint8_t *em = (uint8_t *)(s + npad);           // [npad] preceding neighbours: up 1 down 2 left 4 right 8
  int8_t *dl = (int8_t *)(em + npad);            // [npad] accepted Delta of the round
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  const int v0 = tid * K;

  auto nbr = [&](int v, int &up, int &dn, int &lf, int &rt) {
    const int r = (int)__umulhi((uint32_t)v, a.rdiv), c = v - r * cols;
    up = (r == 0 ? rows - 1 : r - 1) * cols + c;
    dn = (r == rows - 1 ? 0 : r + 1) * cols + c;
    lf = r * cols + (c == 0 ? cols - 1 : c - 1);
    rt = r * cols + (c == cols - 1 ? 0 : c + 1);
  };
  // block sum of x (all threads get it); uses sh.scan, two barriers
  auto block_sum = [&](int x) {
    x = (int)__reduce_add_sync(0xffffffffu, (unsigned)x);
    if (lane == 0) sh.scan[warp] = x;
    __syncthreads();
    int t = 0;
    for (int i = 0; i < nwarp; i++) t += sh.scan[i];
    __syncthreads();
    return t;
  };
  // cut contribution of own sites' right and down edges, spins from `get`
  auto own_cut = [&](auto get) {
    int c0 = 0;
    for (int i = 0; i < K; i++) {
      const int v = v0 + i;
      if (v >= n) break;
      int up, dn, lf, rt;
      nbr(v, up, dn, lf, rt);
      const int sv = get(v);
      if (sv != get(rt)) c0 += __ldg(&a.w[2 * v]);
      if (sv != get(dn)) c0 += __ldg(&a.w[2 * v + 1]);
    }
    return c0;
  };

  unsigned long long nblocks = 0;
  for (int trial = blockIdx.x; trial < a.T; trial += gridDim.x) {
    const uint64_t seed = a.seeds[trial];
    const uint32_t key0 = (uint32_t)seed, key1 = (uint32_t)(seed >> 32);
    // ---- initial spins: top bit of word (v & 3) of Philox(key, (v >> 2, 0, 0, 3))
#pragma unroll 4
    for (int i = 0; i < K / 4; i++) {
      const int q = (v0 >> 2) + i;
      const P4 o = philox10(P4{(uint32_t)q, 0u, 0u, 3u}, key0, key1);
      nblocks++;
      const uint32_t ow[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
      for (int i = 0; i < 4; i++) s[4 * q + i] = (ow[i] >> 31) ? 1 : -1;
    }
    for (int j = 0; j < KW; j++) {  // snapshot = initial spins (bit = +1)
      uint32_t b = 0;
      for (int i = 0; i < 32; i++) b |= (s[v0 + 32 * j + i] > 0 ? 1u : 0u) << i;
      bst[tid * KW + j] = b;
    }
    __syncthreads();
    int cur = block_sum(own_cut([&](int v) { return (int)s[v]; }));
    int best = cur;
    int executed = 0;

    for (int t = 0; t < a.sweeps; t++) {
      uint64_t Kd2 = 0, Kd4 = 0;
      if (SA) {
        Kd2 = a.table[(size_t)t * 4 + 1];
        Kd4 = a.table[(size_t)t * 4 + 3];
      }
      // ---- priorities of the sweep (K / 4 independent Philox blocks)
#pragma unroll 4
      for (int i = 0; i < K / 4; i++) {
        const int q = (v0 >> 2) + i;
        const P4 o = philox10(P4{(uint32_t)q, (uint32_t)t, 0u, 4u}, key0, key1);
        *(uint4 *)&pu[4 * q] = make_uint4(o.x, o.y, o.z, o.w);
      }
      nblocks += K / 4;
      __syncthreads();
      // ---- preceding neighbours (p(u), u) < (p(v), v) and the wait counts
      // (4 bits per site, 8 sites per word, all words owned by this thread)
      uint32_t todo[KW];
#pragma unroll
      for (int j = 0; j < KW; j++) {
        todo[j] = 0;
#pragma unroll 1
        for (int b8 = 0; b8 < 4; b8++) {
          uint32_t cw = 0;
#pragma unroll
          for (int b = 8 * b8; b < 8 * b8 + 8; b++) {
            const int v = v0 + 32 * j + b;
            if (v < n) {
              int nb[4];
              nbr(v, nb[0], nb[1], nb[2], nb[3]);
              const uint32_t pv = pu[v];
              uint32_t m = 0;
#pragma unroll
              for (int d = 0; d < 4; d++) {
                const uint32_t pn = pu[nb[d]];
                if (pn < pv || (pn == pv && nb[d] < v)) m |= 1u << d;
              }
              em[v] = (uint8_t)m;
              todo[j] |= 1u << b;
              cw |= (uint32_t)__popc(m) << (4 * (b & 7));
            }
          }
          cnt[(v0 >> 3) + 4 * j + b8] = cw;
        }
      }
      __syncthreads();  // every priority read before the slots take the uniforms
      if (SA) {
#pragma unroll 4
        for (int i = 0; i < K / 4; i++) {
          const int q = (v0 >> 2) + i;
          const P4 o = philox10(P4{(uint32_t)q, (uint32_t)t, 1u, 4u}, key0, key1);
          *(uint4 *)&pu[4 * q] = make_uint4(o.x, o.y, o.z, o.w);
        }
        nblocks += K / 4;
      }
      bool sweep_flipped = false;
      // ---- rounds: a site is ready once its wait count is 0.  Each round:
      // the owners take their ready sites (barrier), visit them and decrement
      // the wait counts of the neighbours they precede (fire-and-forget shared
      // atomics), and the round's sums are reduced (barrier).
      for (int r = 1;; r++) {
        if (r > 4096) {  // no progress: cannot happen on a consistent order
          if (tid == 0) atomicExch(a.err, GSB_EUNSUPPORTED);
          break;
        }
        uint32_t rd[KW];
        int left = 0;
#pragma unroll
        for (int j = 0; j < KW; j++) {
          uint32_t z = 0;  // sites whose 4-bit count is 0
#pragma unroll
          for (int b8 = 0; b8 < 4; b8++) {
            const uint32_t x = cnt[(v0 >> 3) + 4 * j + b8];
            uint32_t y = ~(x | (x >> 1) | (x >> 2) | (x >> 3)) & 0x11111111u;
            y = (y | (y >> 3)) & 0x03030303u;  // nibble flags -> 8 bits
            y = (y | (y >> 6)) & 0x000F000Fu;
            y = (y | (y >> 12)) & 0xFFu;
            z |= y << (8 * b8);
          }
          rd[j] = todo[j] & z;
          todo[j] &= ~rd[j];
          left += __popc(todo[j]);
        }
        __syncthreads();  // every owner has its ready set before any count changes
        uint32_t fl[KW];
        int D = 0, P = 0;
#pragma unroll
        for (int j = 0; j < KW; j++) {
          fl[j] = 0;
          uint32_t m = rd[j];
          while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            const int v = v0 + 32 * j + b;
            int nb[4];
            nbr(v, nb[0], nb[1], nb[2], nb[3]);
            const uint32_t e = em[v];
#pragma unroll
            for (int d = 0; d < 4; d++)
              if (!((e >> d) & 1u)) atomicSub(&cnt[nb[d] >> 3], 1u << (4 * (nb[d] & 7)));
            const int sv = s[v];
            const int h = __ldg(&a.w[2 * v]) * s[nb[3]] + __ldg(&a.w[2 * v + 1]) * s[nb[1]] +
                          __ldg(&a.w[2 * nb[2]]) * s[nb[2]] + __ldg(&a.w[2 * nb[0] + 1]) * s[nb[0]];
            const int delta = sv * h;
            bool acc;
            if (SA) {
              acc = delta >= 0;
              if (!acc) acc = (uint64_t)pu[v] < (delta == -2 ? Kd2 : delta == -4 ? Kd4 : 0ull);
            } else {
              acc = delta > 0;
            }
            if (acc) {
              s[v] = (int8_t)-sv;
              dl[v] = (int8_t)delta;
              fl[j] |= 1u << b;
              D += delta;
              if (delta > 0) P += delta;
            }
          }
        }
        // ---- round totals (partials double-buffered by parity)
        int all_left;
        {
          const int pr = r & 1;
          const int wd = (int)__reduce_add_sync(0xffffffffu, (unsigned)D);
          const int wp = (int)__reduce_add_sync(0xffffffffu, (unsigned)P);
          const int wl = (int)__reduce_add_sync(0xffffffffu, (unsigned)left);
          if (lane == 0) {
            sh.red[pr][0][warp] = wd;
            sh.red[pr][1][warp] = wp;
            sh.red[pr][2][warp] = wl;
          }
          __syncthreads();
          D = P = all_left = 0;
          for (int i = 0; i < nwarp; i++) {
            D += sh.red[pr][0][i];
            P += sh.red[pr][1][i];
            all_left += sh.red[pr][2][i];
          }
        }
        if (P > 0) sweep_flipped = true;
        // ---- best-so-far in (round, id) order: only if the positive Deltas
        // of the round can lift the running cut above best
        if (cur + P > best) {
          int ws = 0;
#pragma unroll
          for (int j = 0; j < KW; j++) {
            uint32_t m = fl[j];
            while (m) {
              const int b = __ffs(m) - 1;
              m &= m - 1;
              ws += dl[v0 + 32 * j + b];
            }
          }
          int x = ws;  // inclusive warp scan, then the warps' totals
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, off);
            if (lane >= off) x += y;
          }
          if (lane == 31) sh.scan[warp] = x;
          __syncthreads();
          int run = cur + x - ws;
          for (int i = 0; i < warp; i++) run += sh.scan[i];
          long long key = LLONG_MIN;
#pragma unroll
          for (int j = 0; j < KW; j++) {
            uint32_t m = fl[j];
            while (m) {
              const int b = __ffs(m) - 1;
              m &= m - 1;
              const int v = v0 + 32 * j + b;
              const int d = dl[v];
              run += d;
              if (d > 0) {
                const long long kk = (long long)(((unsigned long long)(unsigned)run << 32) |
                                                 (0xFFFFFFFFu - (uint32_t)v));
                key = kk > key ? kk : key;
              }
            }
          }
          key = rs_warp_max_key(key);
          if (lane == 0) sh.kred[warp] = key;
          __syncthreads();
          key = LLONG_MIN;
          for (int i = 0; i < nwarp; i++) key = sh.kred[i] > key ? sh.kred[i] : key;
          const int mval = (int)(key >> 32);
          if (key != LLONG_MIN && mval > best) {
            best = mval;
            const int vstar = (int)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFll));
#pragma unroll
            for (int j = 0; j < KW; j++) {
              // current spins, minus this round's flips after the maximum
              uint32_t b = 0;
              for (int i = 0; i < 32; i++) {
                const int v = v0 + 32 * j + i;
                const bool undo = ((fl[j] >> i) & 1u) && v > vstar;
                b |= ((s[v] > 0) != undo ? 1u : 0u) << i;
              }
              bst[tid * KW + j] = b;
            }
          }
          __syncthreads();  // sh.scan / sh.kred reused by the next round
        }
        cur += D;
        if (all_left == 0) break;
      }
      executed = t + 1;
      if (!SA && !sweep_flipped) break;
    }

    // ---- integrity guard (solvers.py:132-133): recompute the cut of best
    __syncthreads();
    const int cb = block_sum(own_cut([&](int v) { return (int)((bst[v >> 5] >> (v & 31)) & 1u); }));
    if (tid == 0) {
      a.best_cut[trial] = best;
      a.sweeps_exec[trial] = executed;
      if (cb != best) atomicExch(a.err, GSB_EINTEGRITY);
    }
    // ---- best spins MSB-first by site id
    uint8_t *out = a.best_bits + (size_t)trial * a.nbytes;
    for (int byte = tid; byte < a.nbytes; byte += blockDim.x) {
      uint32_t v = 0;
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const int x = byte * 8 + q;
        const uint32_t bit = x < n ? (bst[x >> 5] >> (x & 31)) & 1u : 0u;
        v |= bit << (7 - q);
      }
      out[byte] = (uint8_t)v;
    }
    __syncthreads();
  }
  const unsigned long long nb = __reduce_add_sync(0xffffffffu, (unsigned)nblocks);
  if (lane == 0 && nb) atomicAdd(a.blocks, nb);
}

// ------------------------------------------------------------------ host
static int rs_kw(int n) {
  for (int kw = 1; kw <= 4; kw *= 2)
    if ((n + 32 * kw - 1) / (32 * kw) <= RS_MAXNT) return kw;
  return 0;
}

static size_t rs_smem(int npad) {  // pu, bst, cnt, s, em, dl
  return (size_t)npad * 4 + (size_t)npad / 8 + (size_t)npad / 2 + (size_t)npad * 3;
}

bool rscan_fits(int rows, int cols) {
  const int n = rows * cols;
  if (rows < 3 || cols < 3 || cols > 16384 || n >= (1 << 17)) return false;  // __umulhi division exact
  const int kw = rs_kw(n);
  if (!kw) return false;
  const int nt = ((n + 32 * kw - 1) / (32 * kw) + 31) / 32 * 32;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return false;
  return rs_smem(nt * 32 * kw) + sizeof(RsShared) <= (size_t)optin;
}

template <int KW>
static int rs_launch(const RsArgs &a, bool sa, int nt, cudaStream_t stream) {
  const size_t smem = rs_smem(a.npad);
  auto kern = sa ? rscan_kernel<KW, true> : rscan_kernel<KW, false>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return set_error(GSB_ECUDA, "cudaFuncSetAttribute failed");
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nt, smem) != cudaSuccess ||
      per_sm < 1)
    return set_error(GSB_ECUDA, "random-scan kernel does not fit on an SM");
  int grid = num_sms() * per_sm;
  if (grid > a.T) grid = a.T;
  kern<<<grid, nt, smem, stream>>>(a);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(GSB_ECUDA, cudaGetErrorString(e));
  return GSB_OK;
}

int rscan_run(int rows, int cols, const int8_t *w_dev, int kind, int sweeps,
              const uint64_t *table, const uint64_t *seeds, int T, int64_t *best_cut,
              int32_t *sweeps_exec, uint8_t *best_bits, int *err_ws, cudaStream_t stream) {
  if (!rscan_fits(rows, cols))
    return set_error(GSB_EUNSUPPORTED, "torus too large for the random-scan engine");
  if (num_sms() <= 0) return set_error(GSB_ECUDA, "no CUDA device");
  const int n = rows * cols, kw = rs_kw(n);
  const int nt = ((n + 32 * kw - 1) / (32 * kw) + 31) / 32 * 32;
  RsArgs a;
  a.rows = rows;
  a.cols = cols;
  a.n = n;
  a.npad = nt * 32 * kw;
  a.rdiv = (uint32_t)((0x100000000ull + (uint64_t)cols - 1) / (uint64_t)cols);
  a.w = w_dev;
  a.table = table;
  a.sweeps = sweeps;
  a.seeds = seeds;
  a.T = T;
  a.best_cut = best_cut;
  a.sweeps_exec = sweeps_exec;
  a.best_bits = best_bits;
  a.nbytes = (n + 7) / 8;
  a.err = err_ws;
  a.blocks = (unsigned long long *)((char *)err_ws + 8);
  const bool sa = kind == GSB_ANNEALING;
  switch (kw) {
    case 1: return rs_launch<1>(a, sa, nt, stream);
    case 2: return rs_launch<2>(a, sa, nt, stream);
    default: return rs_launch<4>(a, sa, nt, stream);
  }
}

}  // namespace gsb
