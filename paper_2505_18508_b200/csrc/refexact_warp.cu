// refexact_warp.cu -- warp-cooperative reference-exact engine for +-1 tori.
//
// Bit-for-bit gsetbench.solvers.run_trial (solvers.py:91-140), like
// refexact.cu, but one WARP per trial with the trial's state in shared memory:
//   perm  u16[n]    the sweep's visit order (rng.permutation(n), solvers.py:110)
//   spins u32[n/32] bit-packed, bit x <-> site x (id order)
//   best  u32[n/32] snapshot of the best-so-far state
//   mark  u32[n/32] per-batch scratch: sites flipped in the current batch
//   wneg  u32[2][n/32] coupling sign planes (right, down), per CTA
// and the PCG64 stream state in registers (warp-uniform).  Lane l holds the
// jump-ahead coefficients of output l+1 (A = M^(l+1), C = inc*(M^l+...+1)), so
// the next 32 PCG64 outputs are computed in parallel, one per lane.
//
// Fisher-Yates (numpy shuffle, i = n-1..1, masked rejection on next32 draws):
// a batch of <= 32 draws is resolved at once.  Lane l's draw is accepted for
// certain if (d & mask) <= i - l, rejected for certain if > i, ambiguous
// otherwise; the batch is cut before the first ambiguous lane and before the
// first lane whose swap touches a position touched by an earlier lane of the
// batch (then the committed swaps are disjoint and run in parallel), and is
// limited so the rejection mask cannot change inside it.  The next32 half-word
// buffer (numpy pcg64_next32) is carried across batches, sweeps and the visit
// phase, which draws whole next64 words without touching it.
//
// Visits: 32 consecutive permutation entries per batch.  Delta uses the
// pre-batch spins; a Delta<0 lane (SA) takes the PCG64 output of its rank
// among the batch's Delta<0 lanes.  The batch is committed up to (excluding)
// the first lane that has a flipped neighbour inside the batch -- all earlier
// lanes saw exactly the sequential state -- and the rest is redone.  Best-so-
// far: warp prefix sum of the committed Deltas in visit order; the first lane
// reaching a new maximum above `best` defines the snapshot.
#include <climits>
#include <cstdint>
#include <cstdlib>

#include "gsb_device.cuh"
#include "gsb_internal.h"

namespace gsb {

struct RefWarpArgs {
  int rows, cols, n, nwords;
  const int8_t *w;        // [2n] torus couplings
  const uint64_t *table;  // [S][4] K = ceil(exp(-d/T)*2^53)
  int sweeps, sa;
  uint32_t inv_cols;  // ceil(2^32 / cols)
  const uint64_t *seeds;
  int T;
  const uint64_t *jump;  // [33][4] u64: A_k (lo, hi), S_k (lo, hi), k = 1..32 at index k
  int64_t *best_cut;
  int32_t *sweeps_exec;
  uint8_t *best_bits;
  int nbytes;
  int *err;
};

__device__ __forceinline__ u128 shfl128(u128 v, int src) {
  const uint64_t lo = __shfl_sync(0xffffffffu, (unsigned long long)(uint64_t)v, src);
  const uint64_t hi = __shfl_sync(0xffffffffu, (unsigned long long)(uint64_t)(v >> 64), src);
  return ((u128)hi << 64) | lo;
}

__device__ __forceinline__ int getbit(const uint32_t *a, int x) { return (a[x >> 5] >> (x & 31)) & 1; }

// V2 (default): Fisher-Yates batches of up to 64 draws (all 32 computed
// outputs used; draws lane and lane + 32 per lane, duplicate targets found
// with the `mark` bitmap) and the visit batches' best-so-far scan gated on
// cur + (sum of positive committed Deltas) > best.  V1: 32-draw batches,
// ungated scan (kept for A/B, GSB_REFWARP_V1=1).
template <bool V2>
__global__ void __launch_bounds__(32) ref_warp_kernel(RefWarpArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = a.n, nwd = a.nwords, lane = threadIdx.x;
  uint32_t *spins = (uint32_t *)smem_raw;  // [nwd]
  uint32_t *bestw = spins + nwd;           // [nwd]
  uint32_t *mark = bestw + nwd;            // [nwd]
  uint32_t *wneg = mark + nwd;             // [2][nwd]
  uint16_t *perm = (uint16_t *)(wneg + 2 * nwd);  // [n]
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u;

  for (int i = lane; i < nwd; i += 32) {
    uint32_t r = 0, d = 0;
    for (int b = 0; b < 32; b++) {
      const int x = i * 32 + b;
      if (x < n) {
        r |= (uint32_t)(a.w[2 * x] < 0) << b;
        d |= (uint32_t)(a.w[2 * x + 1] < 0) << b;
      }
    }
    wneg[i] = r;
    wneg[nwd + i] = d;
    mark[i] = 0;
  }
  // jump-ahead coefficients of output lane+1
  const u128 Aj = ((u128)a.jump[(lane + 1) * 4 + 1] << 64) | a.jump[(lane + 1) * 4 + 0];
  const u128 Sj = ((u128)a.jump[(lane + 1) * 4 + 3] << 64) | a.jump[(lane + 1) * 4 + 2];
  const int cols = a.cols, rows = a.rows;
  __syncwarp();

  for (int trial = blockIdx.x; trial < a.T; trial += gridDim.x) {
    u128 s, inc;
    pcg_seed(a.seeds[trial], s, inc);
    const u128 Cj = inc * Sj;  // C_{lane+1}
    int has32 = 0;
    uint32_t buf = 0;

    // ---- initial spins: n next32 draws, spin = bit 31 (solvers.py:96)
    for (int x0 = 0; x0 < n; x0 += 32) {
      // 32 draws: outputs 1..16 (has32 == 0 here: n draws from a fresh stream
      // are consumed in full pairs except possibly the last)
      const u128 sl = Aj * s + Cj;  // state after output lane+1
      const uint64_t o = pcg_out(sl);
      const int src = lane >> 1;
      const uint64_t ov = __shfl_sync(FULL, (unsigned long long)o, src);
      const uint32_t d = (lane & 1) ? (uint32_t)(ov >> 32) : (uint32_t)ov;
      const int x = x0 + lane;
      const unsigned bits = __ballot_sync(FULL, x < n && (d >> 31));
      if (lane == 0) spins[x0 >> 5] = bits;
      const int m = min(32, n - x0);
      const int outs = (m + 1) >> 1;
      s = shfl128(sl, outs - 1);
      if (m & 1) {
        has32 = 1;
        buf = __shfl_sync(FULL, (unsigned)(o >> 32), outs - 1);
      }
    }
    __syncwarp();
    // ---- initial cut (solvers.py:101): each site's right and down edge
    int cutv = 0;
    for (int x = lane; x < n; x += 32) {
      const int r = x / cols, c = x - r * cols;
      const int xr = r * cols + (c + 1 == cols ? 0 : c + 1);
      const int xd = (r + 1 == rows ? 0 : r + 1) * cols + c;
      const int sx = getbit(spins, x);
      if (sx != getbit(spins, xr)) cutv += getbit(wneg, x) ? -1 : 1;
      if (sx != getbit(spins, xd)) cutv += getbit(wneg + nwd, x) ? -1 : 1;
    }
    int cur = (int)__reduce_add_sync(FULL, (unsigned)cutv);
    int best = cur;
    for (int i = lane; i < nwd; i += 32) bestw[i] = spins[i];
    int executed = 0;

    for (int t = 0; t < a.sweeps; t++) {
      // ---- permutation: perm = arange(n), then Fisher-Yates
      for (int i = lane; i < n; i += 32) perm[i] = (uint16_t)i;
      __syncwarp();
      int i = n - 1;
      while (i >= 1) {
        uint32_t mask = (uint32_t)i;
        mask |= mask >> 1;
        mask |= mask >> 2;
        mask |= mask >> 4;
        mask |= mask >> 8;
        mask |= mask >> 16;
        const int half = (int)((mask + 1) >> 1);
        const int h = has32;
        const u128 sl = Aj * s + Cj;
        const uint64_t o = pcg_out(sl);
        if (V2) {
          // draws k = lane (set A) and k = lane + 32 (set B); draw k is the
          // buffered half if k < h, else half (k-h)&1 of output (k-h)>>1
          const int nb = min(64, i - half + 1);  // mask constant for draws < nb
          const uint32_t olo = (uint32_t)o, ohi = (uint32_t)(o >> 32);
          const int qa = lane - h, qb = lane + 32 - h;
          const int sa = qa >= 0 ? (qa >> 1) : 0, sb = qb >> 1;
          const uint32_t alo = __shfl_sync(FULL, olo, sa), ahi = __shfl_sync(FULL, ohi, sa);
          const uint32_t blo = __shfl_sync(FULL, olo, sb), bhi = __shfl_sync(FULL, ohi, sb);
          const int va = (int)((qa < 0 ? buf : ((qa & 1) ? ahi : alo)) & mask);
          const int vb = (int)(((qb & 1) ? bhi : blo) & mask);
          const int kb = lane + 32;
          const bool ina = lane < nb, inb = kb < nb;
          // draw k is accepted for sure if v <= i - k, rejected if v > i
          const bool sacc_a = ina && va <= i - lane, sacc_b = inb && vb <= i - kb;
          const unsigned ambA = __ballot_sync(FULL, ina && !sacc_a && va <= i);
          const unsigned ambB = __ballot_sync(FULL, inb && !sacc_b && vb <= i);
          int L = ambA ? __ffs(ambA) - 1 : ambB ? 31 + __ffs(ambB) : nb;  // draw 0 is never ambiguous
          unsigned mA = __ballot_sync(FULL, sacc_a), mB = __ballot_sync(FULL, sacc_b);
          mA &= L >= 32 ? FULL : (1u << L) - 1u;
          mB &= L >= 64 ? FULL : L <= 32 ? 0u : (1u << (L - 32)) - 1u;
          const int na = __popc(mA), nacc = na + __popc(mB);
          const bool ea = (mA >> lane) & 1u, eb = (mB >> lane) & 1u;
          const int ila = i - __popc(mA & lt_mask), ilb = i - na - __popc(mB & lt_mask);
          // a target inside the batch's position window is the position of
          // the (later) accepted draw of rank i - v
          int cfirst = 64;
          auto window = [&](bool e, int v, int il) {
            if (e && v != il && v > i - nacc) {
              const int r2 = i - v;
              const int k2 = r2 < na ? (int)__fns(mA, 0, r2 + 1) : 32 + (int)__fns(mB, 0, r2 - na + 1);
              cfirst = min(cfirst, k2);
            }
          };
          window(ea, va, ila);
          window(eb, vb, ilb);
          // duplicate targets: the draw that finds its bit already set conflicts
          // (set A before set B; within a set the order is arbitrary, which can
          // only cut earlier than needed)
          if (ea && (atomicOr(&mark[va >> 5], 1u << (va & 31)) >> (va & 31)) & 1u)
            cfirst = min(cfirst, lane);
          __syncwarp();
          if (eb && (atomicOr(&mark[vb >> 5], 1u << (vb & 31)) >> (vb & 31)) & 1u)
            cfirst = min(cfirst, kb);
          __syncwarp();
          if (ea) mark[va >> 5] = 0u;  // only this batch's bits are set
          if (eb) mark[vb >> 5] = 0u;
          cfirst = (int)__reduce_min_sync(FULL, (unsigned)cfirst);
          if (cfirst < L) {
            L = max(cfirst, 1);  // draw 0 alone is always exact
            mA &= L >= 32 ? FULL : (1u << L) - 1u;
            mB &= L <= 32 ? 0u : (1u << (L - 32)) - 1u;
          }
          // execute the committed swaps (disjoint positions)
          const bool doa = (mA >> lane) & 1u, dob = (mB >> lane) & 1u;
          uint16_t pa0 = 0, pa1 = 0, pb0 = 0, pb1 = 0;
          if (doa) {
            pa0 = perm[ila];
            pa1 = perm[va];
          }
          if (dob) {
            pb0 = perm[ilb];
            pb1 = perm[vb];
          }
          __syncwarp();
          if (doa) {
            perm[ila] = pa1;
            perm[va] = pa0;
          }
          if (dob) {
            perm[ilb] = pb1;
            perm[vb] = pb0;
          }
          __syncwarp();
          i -= __popc(mA) + __popc(mB);
          const int fresh = L - h;
          if (fresh <= 0) {
            has32 = 0;
          } else {
            const int outs = (fresh + 1) >> 1;
            s = shfl128(sl, outs - 1);
            if (fresh & 1) {
              has32 = 1;
              buf = __shfl_sync(FULL, ohi, outs - 1);
            } else {
              has32 = 0;
            }
          }
          continue;
        }
        const int nb = min(32, i - half + 1);  // mask constant for lanes < nb
        // draw lane: next32 #lane of the stream
        const int q = lane - h;  // index among fresh halves
        const int src = q >= 0 ? (q >> 1) : 0;
        const uint64_t ov = __shfl_sync(FULL, (unsigned long long)o, src);
        uint32_t d = (q < 0) ? buf : ((q & 1) ? (uint32_t)(ov >> 32) : (uint32_t)ov);
        const int v = (int)(d & mask);
        const bool inb = lane < nb;
        const bool sure_acc = inb && v <= i - lane;
        const bool sure_rej = inb && v > i;
        const bool amb = inb && !sure_acc && !sure_rej;
        const unsigned ambm = __ballot_sync(FULL, amb);
        int L = ambm ? (__ffs(ambm) - 1) : nb;  // lanes [0, L) are resolved
        unsigned accm = __ballot_sync(FULL, sure_acc) & ((L >= 32) ? FULL : ((1u << L) - 1u));
        // position of each accepted lane: i_l = i - rank
        const int rank = __popc(accm & lt_mask);
        const int il = i - rank;
        const bool acc = (accm >> lane) & 1u;
        // conflicts: v inside the batch's position window at another lane's i
        const int nacc = __popc(accm);
        int cfirst = 32;
        if (acc && v != il && v > i - nacc) {
          // v equals i_{l'} for l' = the accepted lane of rank i - v (later lane)
          const int r2 = i - v;
          const int l2 = __fns(accm, 0, r2 + 1);
          if (l2 > lane) cfirst = l2;
        }
        // duplicate targets among accepted lanes: the later one conflicts
        const unsigned same_v = __match_any_sync(FULL, acc ? v : -1 - lane);
        if (acc && (same_v & lt_mask)) cfirst = min(cfirst, lane);
        cfirst = __reduce_min_sync(FULL, (unsigned)cfirst);
        if (cfirst < L) {
          L = cfirst;
          accm &= (1u << L) - 1u;
        }
        // execute the committed swaps (disjoint positions)
        const bool doit = (accm >> lane) & 1u;
        uint16_t pa = 0, pb = 0;
        if (doit) {
          pa = perm[il];
          pb = perm[v];
        }
        __syncwarp();
        if (doit) {
          perm[il] = pb;
          perm[v] = pa;
        }
        __syncwarp();
        i -= __popc(accm);
        // advance the stream by L draws
        const int fresh = L - h;  // halves taken from new outputs
        if (fresh <= 0) {
          has32 = 0;  // L == 1 and the buffered half was used
        } else {
          const int outs = (fresh + 1) >> 1;
          s = shfl128(sl, outs - 1);
          if (fresh & 1) {
            has32 = 1;
            buf = __shfl_sync(FULL, (unsigned)(o >> 32), outs - 1);
          } else {
            has32 = 0;
          }
        }
      }

      // ---- visits in permutation order (solvers.py:110-127)
      uint64_t K2 = 0, K4 = 0;
      if (a.sa) {
        K2 = a.table[(size_t)t * 4 + 1];
        K4 = a.table[(size_t)t * 4 + 3];
      }
      bool flipped = false;
      int k0 = 0;
      while (k0 < n) {
        const int nb = min(32, n - k0);
        const bool inb = lane < nb;
        int x = 0, delta = 0;
        int xr = 0, xd = 0, xl = 0, xu = 0;
        if (inb) {
          x = perm[k0 + lane];
          // x < 2^16: __umulhi with ceil(2^32/cols) is the exact quotient
          const int r = (int)__umulhi((unsigned)x, a.inv_cols), c = x - r * cols;
          xr = r * cols + (c + 1 == cols ? 0 : c + 1);
          xl = r * cols + (c == 0 ? cols - 1 : c - 1);
          xd = (r + 1 == rows ? 0 : r + 1) * cols + c;
          xu = (r == 0 ? rows - 1 : r - 1) * cols + c;
          const int sx = getbit(spins, x);
          // term positive iff (s_x == s_j) == (w == +1)
          int k = 0;
          k += (sx == getbit(spins, xr)) != getbit(wneg, x);
          k += (sx == getbit(spins, xd)) != getbit(wneg + nwd, x);
          k += (sx == getbit(spins, xl)) != getbit(wneg, xl);
          k += (sx == getbit(spins, xu)) != getbit(wneg + nwd, xu);
          delta = 2 * k - 4;
        }
        bool acc;
        unsigned negm = 0;
        u128 sl = 0;
        if (a.sa) {
          negm = __ballot_sync(FULL, inb && delta < 0);
          sl = Aj * s + Cj;
          const uint64_t o = pcg_out(sl);
          const int rk = __popc(negm & lt_mask);
          const uint64_t my = __shfl_sync(FULL, (unsigned long long)o, rk & 31);
          acc = inb && (delta >= 0 || (my >> 11) < (delta == -2 ? K2 : K4));
        } else {
          acc = inb && delta > 0;
        }
        // neighbour conflicts inside the batch
        if (acc) atomicOr(&mark[x >> 5], 1u << (x & 31));
        __syncwarp();
        const bool hit = inb && (getbit(mark, xr) | getbit(mark, xl) | getbit(mark, xd) |
                                 getbit(mark, xu));
        __syncwarp();
        if (acc) atomicAnd(&mark[x >> 5], ~(1u << (x & 31)));
        const unsigned hitm = __ballot_sync(FULL, hit);
        // commit lanes [0, L); lane 0 always saw the exact sequential state
        const int L = hitm ? max(__ffs(hitm) - 1, 1) : nb;
        const bool commit = acc && lane < L;
        const unsigned cm = __ballot_sync(FULL, commit);
        // running cut and the first new maximum (strict >, solvers.py:125);
        // V2 scans only if the positive committed Deltas can lift cur above best
        int pre = commit ? delta : 0;
        if (V2) {
          const int tot = (int)__reduce_add_sync(FULL, (unsigned)pre);
          const int pos = (int)__reduce_add_sync(FULL, (unsigned)(pre > 0 ? pre : 0));
          if (cur + pos <= best) {
            if (commit) atomicXor(&spins[x >> 5], 1u << (x & 31));
            cur += tot;
            if (cm) flipped = true;
            if (a.sa) {
              const int used = __popc(negm & ((L >= 32) ? FULL : ((1u << L) - 1u)));
              if (used) s = shfl128(sl, used - 1);
            }
            __syncwarp();
            k0 += L;
            continue;
          }
        }
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int y = __shfl_up_sync(FULL, pre, off);
          if (lane >= off) pre += y;
        }
        const int run = cur + pre;
        const bool cand = commit && run > best;
        int mx = cand ? run : INT_MIN;
        mx = (int)__reduce_max_sync(FULL, (unsigned)(mx ^ INT_MIN)) ^ INT_MIN;
        const unsigned atmax = __ballot_sync(FULL, cand && run == mx);
        __syncwarp();
        if (atmax) {
          const int js = __ffs(atmax) - 1;
          if (commit && lane <= js) atomicXor(&spins[x >> 5], 1u << (x & 31));
          __syncwarp();
          for (int q = lane; q < nwd; q += 32) bestw[q] = spins[q];
          __syncwarp();
          if (commit && lane > js) atomicXor(&spins[x >> 5], 1u << (x & 31));
          best = mx;
        } else if (commit) {
          atomicXor(&spins[x >> 5], 1u << (x & 31));
        }
        cur = __shfl_sync(FULL, run, 31);
        if (cm) flipped = true;
        if (a.sa) {
          const int used = __popc(negm & ((L >= 32) ? FULL : ((1u << L) - 1u)));
          if (used) s = shfl128(sl, used - 1);
        }
        __syncwarp();
        k0 += L;
      }
      executed = t + 1;
      if (!a.sa && !flipped) break;
    }

    // ---- integrity guard (solvers.py:132-133) and output
    int cb = 0;
    for (int x = lane; x < n; x += 32) {
      const int r = x / cols, c = x - r * cols;
      const int xr = r * cols + (c + 1 == cols ? 0 : c + 1);
      const int xd = (r + 1 == rows ? 0 : r + 1) * cols + c;
      const int sx = getbit(bestw, x);
      if (sx != getbit(bestw, xr)) cb += getbit(wneg, x) ? -1 : 1;
      if (sx != getbit(bestw, xd)) cb += getbit(wneg + nwd, x) ? -1 : 1;
    }
    cb = (int)__reduce_add_sync(FULL, (unsigned)cb);
    if (lane == 0) {
      a.best_cut[trial] = best;
      a.sweeps_exec[trial] = executed;
      if (cb != best) atomicExch(a.err, GSB_EINTEGRITY);
    }
    uint8_t *out = a.best_bits + (size_t)trial * a.nbytes;
    for (int byte = lane; byte < a.nbytes; byte += 32) {
      const uint32_t wv = bestw[byte >> 2];
      const uint32_t b8 = (wv >> ((byte & 3) * 8)) & 0xFFu;
      out[byte] = (uint8_t)(__brev(b8) >> 24);  // site 8*byte+j -> bit 7-j
    }
    __syncwarp();
  }
}

bool ref_warp_fits(int rows, int cols) {
  const int n = rows * cols;
  return n <= 65535 && n >= 2;
}

size_t ref_warp_smem(int n) {
  const int nwd = (n + 31) / 32;
  return (size_t)nwd * 4 * 5 + (size_t)n * 2 + 16;
}

int ref_warp_run(int rows, int cols, const int8_t *w_dev, int kind, int sweeps,
                 const uint64_t *table, const uint64_t *seeds, int T, int64_t *best_cut,
                 int32_t *sweeps_exec, uint8_t *best_bits, void *ws, int *err_ws,
                 cudaStream_t stream) {
  const int n = rows * cols;
  const int nsm = num_sms();
  if (nsm <= 0) return set_error(GSB_ECUDA, "no CUDA device");
  // jump-ahead table (host): A_k = M^k, S_k = 1 + M + ... + M^(k-1)
  uint64_t jt[33 * 4];
  {
    u128 A = 1, S = 0;
    const u128 M = pcg_mult();
    for (int k = 0; k <= 32; k++) {
      jt[k * 4 + 0] = (uint64_t)A;
      jt[k * 4 + 1] = (uint64_t)(A >> 64);
      jt[k * 4 + 2] = (uint64_t)S;
      jt[k * 4 + 3] = (uint64_t)(S >> 64);
      S = S + A;
      A = A * M;
    }
  }
  uint64_t *jump = (uint64_t *)ws;
  if (cudaMemcpyAsync(jump, jt, sizeof(jt), cudaMemcpyHostToDevice, stream) != cudaSuccess)
    return set_error(GSB_ECUDA, "jump table copy failed");
  RefWarpArgs a;
  a.rows = rows;
  a.cols = cols;
  a.n = n;
  a.nwords = (n + 31) / 32;
  a.w = w_dev;
  a.table = table;
  a.sweeps = sweeps;
  a.sa = kind == GSB_ANNEALING;
  a.seeds = seeds;
  a.T = T;
  a.jump = jump;
  a.best_cut = best_cut;
  a.sweeps_exec = sweeps_exec;
  a.best_bits = best_bits;
  a.nbytes = (n + 7) / 8;
  a.inv_cols = (uint32_t)((((uint64_t)1 << 32) + (uint64_t)cols - 1) / (uint64_t)cols);
  a.err = err_ws;
  const size_t smem = ref_warp_smem(n);
  auto kern = ref_warp_kernel<true>;
  if (allow_dynamic_smem((const void *)kern, smem) != cudaSuccess)
    return set_error(GSB_ECUDA, "cudaFuncSetAttribute failed");
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32, smem) !=
          cudaSuccess ||
      per_sm < 1)
    return set_error(GSB_ECUDA, "reference warp kernel does not fit");
  int grid = nsm * per_sm;
  if (grid > T) grid = T;
  kern<<<grid, 32, smem, stream>>>(a);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GSB_OK : set_error(GSB_ECUDA, cudaGetErrorString(e));
}

}  // namespace gsb
