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

// Per-site meta byte: preceding-neighbour mask (bits 0-3: up, down, left,
// right), right / down coupling is -1 (bits 4 / 5), spin is +1 (bit 6).
constexpr uint32_t RS_WR = 16, RS_WD = 32, RS_SP = 64;

template <int KW, bool SA>
__global__ void __launch_bounds__(RS_MAXNT, 2) rscan_kernel(RsArgs a) {
  constexpr int K = 32 * KW;                 // sites per thread
  constexpr int LK = KW == 1 ? 5 : KW == 2 ? 6 : 7;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ RsShared sh;
  const int n = a.n, npad = a.npad, cols = a.cols, rows = a.rows;
  const int NT = blockDim.x;
  // Shared arrays are transposed: site v (owner v >> LK, offset o = v & (K-1))
  // lives at o * NT + owner, so the lanes of a warp touching the same offset
  // of their own sites hit consecutive addresses (no bank conflicts).
  uint32_t *pu = (uint32_t *)smem_raw;        // [npad] priorities, then uniforms
  uint32_t *bst = pu + npad;                  // [KW][NT] best snapshot bits (bit b of word j: offset 32j+b)
  uint32_t *cnt = bst + npad / 32;            // [K/8][NT] 4-bit wait counts, 8 offsets per word
  uint8_t *meta = (uint8_t *)(cnt + npad / 8);  // [npad]
  int8_t *dl = (int8_t *)(meta + npad);       // [npad] accepted Delta of the round
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = NT >> 5;
  const int v0 = tid * K;

  auto tix = [&](int v) { return (v & (K - 1)) * NT + (v >> LK); };
  auto nbr = [&](int v, int &up, int &dn, int &lf, int &rt) {
    const int r = (int)__umulhi((uint32_t)v, a.rdiv), c = v - r * cols;
    up = (r == 0 ? rows - 1 : r - 1) * cols + c;
    dn = (r == rows - 1 ? 0 : r + 1) * cols + c;
    lf = r * cols + (c == 0 ? cols - 1 : c - 1);
    rt = r * cols + (c == cols - 1 ? 0 : c + 1);
  };
  auto block_sum = [&](int x) {
    x = (int)__reduce_add_sync(0xffffffffu, (unsigned)x);
    if (lane == 0) sh.scan[warp] = x;
    __syncthreads();
    int t = 0;
    for (int i = 0; i < nwarp; i++) t += sh.scan[i];
    __syncthreads();
    return t;
  };
  // cut of own sites' right and down edges; spin(v) in {0, 1} from `get`
  auto own_cut = [&](auto get) {
    int c0 = 0;
    for (int o = 0; o < K; o++) {
      const int v = v0 + o;
      if (v >= n) break;
      int up, dn, lf, rt;
      nbr(v, up, dn, lf, rt);
      const uint32_t m = meta[o * NT + tid];
      const uint32_t sv = get(v);
      if (sv != get(rt)) c0 += (m & RS_WR) ? -1 : 1;
      if (sv != get(dn)) c0 += (m & RS_WD) ? -1 : 1;
    }
    return c0;
  };
  auto bst_bit = [&](int v) -> uint32_t {
    const int o = v & (K - 1);
    return (bst[(o >> 5) * NT + (v >> LK)] >> (o & 31)) & 1u;
  };

  // coupling bits of the own sites (same for every trial)
  for (int o = 0; o < K; o++) {
    const int v = v0 + o;
    uint32_t m = 0;
    if (v < n) {
      if (a.w[2 * v] < 0) m |= RS_WR;
      if (a.w[2 * v + 1] < 0) m |= RS_WD;
    }
    meta[o * NT + tid] = (uint8_t)m;
  }

  unsigned long long nblocks = 0;
  for (int trial = blockIdx.x; trial < a.T; trial += gridDim.x) {
    const uint64_t seed = a.seeds[trial];
    const uint32_t key0 = (uint32_t)seed, key1 = (uint32_t)(seed >> 32);
    // ---- initial spins: top bit of word (v & 3) of Philox(key, (v >> 2, 0, 0, 3))
    uint32_t sb[KW];  // own spins, bit o & 31 of word o >> 5 (1 = +1)
#pragma unroll
    for (int j = 0; j < KW; j++) sb[j] = 0;
#pragma unroll 4
    for (int i = 0; i < K / 4; i++) {
      const P4 o4 = philox10(P4{(uint32_t)((v0 >> 2) + i), 0u, 0u, 3u}, key0, key1);
      const uint32_t nib = (o4.x >> 31) | ((o4.y >> 31) << 1) | ((o4.z >> 31) << 2) | ((o4.w >> 31) << 3);
#pragma unroll
      for (int j = 0; j < KW; j++)
        if ((i >> 3) == j) sb[j] |= nib << (4 * (i & 7));
    }
    nblocks += K / 4;
    for (int o = 0; o < K; o++) {
      const uint32_t bit = (sb[o >> 5] >> (o & 31)) & 1u;
      meta[o * NT + tid] = (uint8_t)((meta[o * NT + tid] & (RS_WR | RS_WD)) | (bit ? RS_SP : 0u));
    }
#pragma unroll
    for (int j = 0; j < KW; j++) bst[j * NT + tid] = sb[j];
    __syncthreads();
    int cur = block_sum(own_cut([&](int v) { return (uint32_t)(meta[tix(v)] >> 6) & 1u; }));
    int best = cur;
    int executed = 0;

    for (int t = 0; t < a.sweeps; t++) {
      uint64_t Kd2 = 0, Kd4 = 0;
      if (SA) {
        Kd2 = a.table[(size_t)t * 4 + 1];
        Kd4 = a.table[(size_t)t * 4 + 3];
      }
      // ---- priorities of the sweep
#pragma unroll 4
      for (int i = 0; i < K / 4; i++) {
        const P4 o4 = philox10(P4{(uint32_t)((v0 >> 2) + i), (uint32_t)t, 0u, 4u}, key0, key1);
        pu[(4 * i) * NT + tid] = o4.x;
        pu[(4 * i + 1) * NT + tid] = o4.y;
        pu[(4 * i + 2) * NT + tid] = o4.z;
        pu[(4 * i + 3) * NT + tid] = o4.w;
      }
      nblocks += K / 4;
      __syncthreads();
      // ---- preceding neighbours (p(u), u) < (p(v), v) and the wait counts
      uint32_t todo[KW];
#pragma unroll
      for (int j = 0; j < KW; j++) todo[j] = 0;
#pragma unroll 1
      for (int o8 = 0; o8 < K / 8; o8++) {
        uint32_t cw = 0;
#pragma unroll 2
        for (int b = 0; b < 8; b++) {
          const int o = 8 * o8 + b, v = v0 + o;
          if (v < n) {
            int nb[4];
            nbr(v, nb[0], nb[1], nb[2], nb[3]);
            const uint32_t pv = pu[o * NT + tid];
            uint32_t m = 0;
#pragma unroll
            for (int d = 0; d < 4; d++) {
              const uint32_t pn = pu[tix(nb[d])];
              if (pn < pv || (pn == pv && nb[d] < v)) m |= 1u << d;
            }
            meta[o * NT + tid] = (uint8_t)((meta[o * NT + tid] & 0xF0u) | m);
            cw |= (uint32_t)__popc(m) << (4 * b);
#pragma unroll
            for (int j = 0; j < KW; j++)
              if ((o >> 5) == j) todo[j] |= 1u << (o & 31);
          }
        }
        cnt[o8 * NT + tid] = cw;
      }
      __syncthreads();  // every priority read before the slots take the uniforms
      if (SA) {
#pragma unroll 4
        for (int i = 0; i < K / 4; i++) {
          const P4 o4 = philox10(P4{(uint32_t)((v0 >> 2) + i), (uint32_t)t, 1u, 4u}, key0, key1);
          pu[(4 * i) * NT + tid] = o4.x;
          pu[(4 * i + 1) * NT + tid] = o4.y;
          pu[(4 * i + 2) * NT + tid] = o4.z;
          pu[(4 * i + 3) * NT + tid] = o4.w;
        }
        nblocks += K / 4;
      }
      bool sweep_flipped = false;
      // ---- rounds: a site is ready once its wait count is 0.  Each round the
      // owners take their ready sites (barrier), visit them and decrement the
      // counts of the neighbours they precede, and the round's sums are
      // reduced (barrier).
      for (int r = 1;; r++) {
        if (r > 4096) {  // no progress: cannot happen on a consistent order
          if (tid == 0) atomicExch(a.err, GSB_EUNSUPPORTED);
          break;
        }
        uint32_t rd[KW];
        int left = 0;
#pragma unroll
        for (int j = 0; j < KW; j++) {
          uint32_t z = 0;  // offsets whose 4-bit count is 0
#pragma unroll
          for (int b8 = 0; b8 < 4; b8++) {
            const uint32_t x = cnt[(4 * j + b8) * NT + tid];
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
            const int o = 32 * j + b, v = v0 + o;
            int nb[4];
            nbr(v, nb[0], nb[1], nb[2], nb[3]);
            const uint32_t mv = meta[o * NT + tid];
            const uint32_t mu = meta[tix(nb[0])], md = meta[tix(nb[1])];
            const uint32_t ml = meta[tix(nb[2])], mr = meta[tix(nb[3])];
#pragma unroll
            for (int d = 0; d < 4; d++)
              if (!((mv >> d) & 1u)) {
                const int u = nb[d], ou = u & (K - 1);
                atomicSub(&cnt[(ou >> 3) * NT + (u >> LK)], 1u << (4 * (ou & 7)));
              }
            // Delta = s_v * sum_j w_vj s_j; a term is -1 iff (w < 0) != (s_j < 0)
            const uint32_t neg = (((mv >> 4) ^ (mr >> 6) ^ 1u) & 1u) |
                                 ((((mv >> 5) ^ (md >> 6) ^ 1u) & 1u) << 1) |
                                 ((((ml >> 4) ^ (ml >> 6) ^ 1u) & 1u) << 2) |
                                 ((((mu >> 5) ^ (mu >> 6) ^ 1u) & 1u) << 3);
            const int h = 4 - 2 * __popc(neg);
            const int delta = (mv & RS_SP) ? h : -h;
            bool acc;
            if (SA) {
              acc = delta >= 0;
              if (!acc) acc = (uint64_t)pu[o * NT + tid] < (delta == -2 ? Kd2 : delta == -4 ? Kd4 : 0ull);
            } else {
              acc = delta > 0;
            }
            if (acc) {
              meta[o * NT + tid] = (uint8_t)(mv ^ RS_SP);
              dl[o * NT + tid] = (int8_t)delta;
              fl[j] |= 1u << b;
              D += delta;
              if (delta > 0) P += delta;
            }
          }
          sb[j] ^= fl[j];
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
              ws += dl[(32 * j + b) * NT + tid];
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
              const int d = dl[(32 * j + b) * NT + tid];
              run += d;
              if (d > 0) {
                const long long kk = (long long)(((unsigned long long)(unsigned)run << 32) |
                                                 (0xFFFFFFFFu - (uint32_t)(v0 + 32 * j + b)));
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
            // own spins now, minus this round's flips after the maximum
#pragma unroll
            for (int j = 0; j < KW; j++) {
              const int first = vstar - (v0 + 32 * j);  // offsets > first are after it
              const uint32_t after = first < 0 ? 0xFFFFFFFFu : first >= 31 ? 0u : (0xFFFFFFFFu << (first + 1));
              bst[j * NT + tid] = sb[j] ^ (fl[j] & after);
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
    const int cb = block_sum(own_cut(bst_bit));
    if (tid == 0) {
      a.best_cut[trial] = best;
      a.sweeps_exec[trial] = executed;
      if (cb != best) atomicExch(a.err, GSB_EINTEGRITY);
    }
    // ---- best spins MSB-first by site id: byte B holds sites 8B..8B+7, all
    // owned by one thread (K is a multiple of 8)
    uint8_t *out = a.best_bits + (size_t)trial * a.nbytes;
    for (int byte = tid; byte < a.nbytes; byte += NT) {
      const int v = 8 * byte;
      const int o = v & (K - 1);
      const uint32_t w8 = (bst[(o >> 5) * NT + (v >> LK)] >> (o & 31)) & 0xFFu;
      uint32_t bits = __brev(w8) >> 24;  // site 8B -> MSB
      if (v + 8 > n) bits &= 0xFFu << (v + 8 - n);  // padding bits 0
      out[byte] = (uint8_t)bits;
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

static size_t rs_smem(int npad) {  // pu, bst, cnt, meta, dl
  return (size_t)npad * 4 + (size_t)npad / 8 + (size_t)npad / 2 + (size_t)npad * 2;
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
