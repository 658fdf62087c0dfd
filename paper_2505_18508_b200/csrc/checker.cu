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
// Layout (per trial, shared memory): spins bit-packed per colour, per row:
//   word (p, r*WPR + w) bit b  <->  site (r, c = 2k + ((r+p)&1)), k = 32w + b,
//   H = cols/2 sites per row per colour, WPR = ceil(H/32), padding bits 0.
// Couplings are 4 sign planes per word (bit = weight is -1), shared by all
// trials, held in registers.  One CTA runs one trial at a time (persistent
// over trials); thread i owns words i, i+NT, ... of both colours.
//
// Per word and half-sweep: 4 positive-term bit planes P_j = ~(S^N_j^NEG_j),
// bit-sliced counts -> Delta classes, then for the Delta<0 sites a bit-sliced,
// MSB-first comparison of the 32-bit uniform against the threshold
// K = ceil(exp(Delta/T)*2^32) that draws Philox planes lazily (4 planes per
// call) and stops as soon as every pending site is decided.
#include <climits>
#include <cstdint>

#include "gsb_device.cuh"
#include "gsb_internal.h"

namespace gsb {

// masks layout: [2][nw][8] uint32: NS, NSH, NU, ND, VALID, pad...
__global__ void checker_masks_kernel(int rows, int cols, int WPR, const int8_t *__restrict__ w,
                                     uint32_t *__restrict__ masks) {
  const int H = cols >> 1;
  const int nw = rows * WPR;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < 2 * nw;
       idx += gridDim.x * blockDim.x) {
    int p = idx / nw, wi = idx % nw;
    int r = wi / WPR, ww = wi % WPR;
    int e = (r + p) & 1;
    uint32_t ns = 0, nsh = 0, nu = 0, nd = 0, valid = 0;
    for (int b = 0; b < 32; b++) {
      int k = ww * 32 + b;
      if (k >= H) break;
      int c = 2 * k + e;
      int x = r * cols + c;
      int cl = (c + cols - 1) % cols;
      int ru = (r + rows - 1) % rows;
      int8_t w_right = w[2 * x], w_down = w[2 * x + 1];
      int8_t w_left = w[2 * (r * cols + cl)];
      int8_t w_up = w[2 * (ru * cols + c) + 1];
      // e==0: same-k other-colour word is the right neighbour, shifted is left
      // e==1: same-k is the left neighbour, shifted is right
      int8_t wsame = e == 0 ? w_right : w_left;
      int8_t wsh = e == 0 ? w_left : w_right;
      valid |= 1u << b;
      if (wsame < 0) ns |= 1u << b;
      if (wsh < 0) nsh |= 1u << b;
      if (w_up < 0) nu |= 1u << b;
      if (w_down < 0) nd |= 1u << b;
    }
    uint32_t *m = masks + (size_t)idx * 8;
    m[0] = ns;
    m[1] = nsh;
    m[2] = nu;
    m[3] = nd;
    m[4] = valid;
    m[5] = m[6] = m[7] = 0;
  }
}

struct WordMasks {
  uint32_t ns, nsh, nu, nd, valid;
};

struct CheckerArgs {
  int rows, cols, H, WPR, nw, lb;
  const uint32_t *masks;
  const uint64_t *table;  // [S][4]
  int sweeps;
  const uint64_t *seeds;
  int T;
  int64_t *best_cut;
  int32_t *sweeps_exec;
  uint8_t *best_bits;
  int nbytes;
  int *err;
};

// neighbour words of word wi (colour p) from the other colour's array `o`
__device__ __forceinline__ void neighbours(const uint32_t *__restrict__ o, int rows, int WPR, int lb,
                                           int r, int ww, int e, uint32_t &same, uint32_t &sh,
                                           uint32_t &up, uint32_t &dn) {
  int base = r * WPR;
  int rup = (r == 0 ? rows - 1 : r - 1) * WPR;
  int rdn = (r == rows - 1 ? 0 : r + 1) * WPR;
  same = o[base + ww];
  up = o[rup + ww];
  dn = o[rdn + ww];
  if (e == 0) {  // k-1 neighbour (left)
    uint32_t carry = ww > 0 ? (o[base + ww - 1] >> 31) : ((o[base + WPR - 1] >> lb) & 1u);
    sh = (same << 1) | carry;
  } else {  // k+1 neighbour (right)
    uint32_t carry = ww < WPR - 1 ? ((o[base + ww + 1] & 1u) << 31) : ((o[base] & 1u) << lb);
    sh = (same >> 1) | carry;
  }
}

// cut contribution of colour-0 word: sum over its 4 edges of w*[differ]
__device__ __forceinline__ int word_cut(uint32_t s, uint32_t same, uint32_t sh, uint32_t up,
                                        uint32_t dn, const WordMasks &m) {
  int c = 0;
  uint32_t x;
  x = (s ^ same) & m.valid;
  c += __popc(x & ~m.ns) - __popc(x & m.ns);
  x = (s ^ sh) & m.valid;
  c += __popc(x & ~m.nsh) - __popc(x & m.nsh);
  x = (s ^ up) & m.valid;
  c += __popc(x & ~m.nu) - __popc(x & m.nu);
  x = (s ^ dn) & m.valid;
  c += __popc(x & ~m.nd) - __popc(x & m.nd);
  return c;
}

template <int NT>
__device__ __forceinline__ int block_sum_int(int v, int *red, int slot) {
  // red: [2][32] ints; all threads return the total
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[slot * 32 + warp] = v;
  __syncthreads();
  int t = 0;
#pragma unroll
  for (int i = 0; i < NT / 32; i++) t += red[slot * 32 + i];
  return t;
}

template <int NT, int WPT, bool SA>
__global__ void __launch_bounds__(NT) checker_sweep_kernel(CheckerArgs a) {
  extern __shared__ uint32_t smem[];
  const int nw = a.nw;
  uint32_t *st = smem;            // [2][nw]
  uint32_t *bst = smem + 2 * nw;  // [2][nw]
  int *red = (int *)(smem + 4 * nw);                    // [2][96] phase reductions
  int *red2 = red + 2 * 96;                             // [2][32] misc block sums
  long long *kred = (long long *)(red2 + 64);           // [32]
  int *wsum = (int *)(kred + 32);                       // [nw] word sums / prefixes

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  // this thread's words and their coupling masks (identical for every trial)
  WordMasks mk[2][WPT];
  int wr[WPT], wcol[WPT];
#pragma unroll
  for (int j = 0; j < WPT; j++) {
    int wi = tid + j * NT;
    wr[j] = wi / a.WPR;
    wcol[j] = wi % a.WPR;
#pragma unroll
    for (int p = 0; p < 2; p++) {
      if (wi < nw) {
        const uint32_t *m = a.masks + ((size_t)p * nw + wi) * 8;
        mk[p][j] = WordMasks{m[0], m[1], m[2], m[3], m[4]};
      } else {
        mk[p][j] = WordMasks{0, 0, 0, 0, 0};
      }
    }
  }

  for (int trial = blockIdx.x; trial < a.T; trial += gridDim.x) {
    const uint64_t seed = a.seeds[trial];
    const uint32_t key0 = (uint32_t)seed, key1 = (uint32_t)(seed >> 32);

    // ---- initial spins: bit (k&31) of word 0 of Philox(key, (wi, 0, p, 0))
#pragma unroll
    for (int j = 0; j < WPT; j++) {
      int wi = tid + j * NT;
      if (wi < nw) {
#pragma unroll
        for (int p = 0; p < 2; p++) {
          P4 o = philox10(P4{(uint32_t)wi, 0u, (uint32_t)p, 0u}, key0, key1);
          uint32_t s = o.x & mk[p][j].valid;
          st[p * nw + wi] = s;
          bst[p * nw + wi] = s;
        }
      }
    }
    __syncthreads();

    // ---- initial cut (every edge has exactly one colour-0 endpoint)
    int c0 = 0;
#pragma unroll
    for (int j = 0; j < WPT; j++) {
      int wi = tid + j * NT;
      if (wi < nw) {
        int e = wr[j] & 1;  // p = 0
        uint32_t same, sh, up, dn;
        neighbours(st + nw, a.rows, a.WPR, a.lb, wr[j], wcol[j], e, same, sh, up, dn);
        c0 += word_cut(st[wi], same, sh, up, dn, mk[0][j]);
      }
    }
    int cur = block_sum_int<NT>(c0, red2, 0);
    int best = cur;
    int executed = 0;
    int phase = 0;

    for (int t = 0; t < a.sweeps; t++) {
      uint32_t K2 = 0, K4 = 0;
      bool all2 = false, all4 = false;
      if (SA) {
        uint64_t t2 = a.table[(size_t)t * 4 + 1], t4 = a.table[(size_t)t * 4 + 3];
        all2 = t2 > 0xFFFFFFFFull;
        all4 = t4 > 0xFFFFFFFFull;
        K2 = (uint32_t)t2;
        K4 = (uint32_t)t4;
      }
      int sweep_flips = 0;
#pragma unroll 1
      for (int p = 0; p < 2; p++, phase ^= 1) {
        const uint32_t *o = st + (p ^ 1) * nw;
        uint32_t Am[WPT], Pos2[WPT], Pos4[WPT], Neg2[WPT], Neg4[WPT];
        int dsum = 0, psum = 0, nflip = 0;
#pragma unroll
        for (int j = 0; j < WPT; j++) {
          int wi = tid + j * NT;
          Am[j] = Pos2[j] = Pos4[j] = Neg2[j] = Neg4[j] = 0;
          if (wi < nw) {
            const WordMasks &m = mk[p][j];
            int e = (wr[j] + p) & 1;
            uint32_t same, sh, up, dn;
            neighbours(o, a.rows, a.WPR, a.lb, wr[j], wcol[j], e, same, sh, up, dn);
            uint32_t S = st[p * nw + wi];
            uint32_t P0 = ~(S ^ same ^ m.ns) & m.valid;
            uint32_t P1 = ~(S ^ sh ^ m.nsh) & m.valid;
            uint32_t P2 = ~(S ^ up ^ m.nu) & m.valid;
            uint32_t P3 = ~(S ^ dn ^ m.nd) & m.valid;
            uint32_t x01 = P0 ^ P1, c01 = P0 & P1, x23 = P2 ^ P3, c23 = P2 & P3;
            uint32_t ones = x01 ^ x23, ad = x01 & x23;
            uint32_t ge2 = c01 | c23 | ad;               // k >= 2  (Delta >= 0)
            uint32_t k4 = c01 & c23;                     // Delta = +4
            uint32_t ge3 = k4 | ((c01 | c23) & ones);    // Delta > 0
            uint32_t k3 = ge3 & ~k4;                     // Delta = +2
            uint32_t any = P0 | P1 | P2 | P3;
            uint32_t km2 = any & ~ge2;                   // Delta = -2
            uint32_t km4 = m.valid & ~any;               // Delta = -4
            uint32_t A;
            if (SA) {
              A = ge2;
              if (all2) A |= km2;
              if (all4) A |= km4;
              uint32_t e2 = all2 ? 0u : km2;
              uint32_t e4 = all4 ? 0u : km4;
              if (K2 == 0) e2 = 0;  // exp underflow: never accepted, no draw needed
              if (K4 == 0) e4 = 0;
              uint32_t eq = e2 | e4, lt = 0;
              // MSB-first bit-sliced compare u < K, planes drawn lazily
#pragma unroll 1
              for (int g = 0; g < 8 && eq; g++) {
                P4 r = philox10(P4{(uint32_t)wi, (uint32_t)t, (uint32_t)(8 * p + g), 1u}, key0, key1);
                uint32_t pl[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
                for (int q = 0; q < 4; q++) {
                  int bit = 31 - (4 * g + q);
                  uint32_t tb = (((K2 >> bit) & 1u) ? e2 : 0u) | (((K4 >> bit) & 1u) ? e4 : 0u);
                  uint32_t R = pl[q];
                  lt |= eq & ~R & tb;
                  eq &= ~(R ^ tb);
                }
              }
              A |= lt;
            } else {
              A = ge3;
            }
            A &= m.valid;
            st[p * nw + wi] = S ^ A;
            Am[j] = A;
            Pos2[j] = A & k3;
            Pos4[j] = A & k4;
            Neg2[j] = A & km2;
            Neg4[j] = A & km4;
            int pp = 2 * __popc(Pos2[j]) + 4 * __popc(Pos4[j]);
            psum += pp;
            dsum += pp - 2 * __popc(Neg2[j]) - 4 * __popc(Neg4[j]);
            nflip += __popc(A);
          }
        }
        // ---- block reduction of (dsum, psum, nflip)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          dsum += __shfl_xor_sync(0xffffffffu, dsum, off);
          psum += __shfl_xor_sync(0xffffffffu, psum, off);
          nflip += __shfl_xor_sync(0xffffffffu, nflip, off);
        }
        int *rb = red + phase * 96;
        if (lane == 0) {
          rb[warp] = dsum;
          rb[32 + warp] = psum;
          rb[64 + warp] = nflip;
        }
        __syncthreads();
        int D = 0, Pt = 0, F = 0;
#pragma unroll
        for (int i = 0; i < NT / 32; i++) {
          D += rb[i];
          Pt += rb[32 + i];
          F += rb[64 + i];
        }
        sweep_flips += F;
        if (cur + Pt > best) {
          // ---- exact best tracking: first position of the half-sweep maximum
          int wmaxv[WPT], wpos[WPT];
#pragma unroll
          for (int j = 0; j < WPT; j++) {
            int wi = tid + j * NT;
            int v = 0, mx = INT32_MIN, mp = -1;
            uint32_t nz = Pos2[j] | Pos4[j] | Neg2[j] | Neg4[j];
            while (nz) {
              int b = __ffs(nz) - 1;
              nz &= nz - 1;
              uint32_t bm = 1u << b;
              int d = (Pos2[j] & bm) ? 2 : (Pos4[j] & bm) ? 4 : (Neg2[j] & bm) ? -2 : -4;
              v += d;
              if (d > 0 && v > mx) {
                mx = v;
                mp = b;
              }
            }
            wmaxv[j] = mx;
            wpos[j] = mp;
            if (wi < nw) wsum[wi] = v;
          }
          __syncthreads();
          // exclusive scan of wsum over word order, by warp 0
          if (warp == 0) {
            int per = (nw + 31) / 32;
            int lo = lane * per, hi = min(lo + per, nw);
            int s = 0;
            for (int i = lo; i < hi; i++) s += wsum[i];
            int incl = s;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
              int y = __shfl_up_sync(0xffffffffu, incl, off);
              if (lane >= off) incl += y;
            }
            int run = incl - s;
            for (int i = lo; i < hi; i++) {
              int v = wsum[i];
              wsum[i] = run;
              run += v;
            }
          }
          __syncthreads();
          long long key = LLONG_MIN;
#pragma unroll
          for (int j = 0; j < WPT; j++) {
            int wi = tid + j * NT;
            if (wi < nw && wpos[j] >= 0) {
              long long val = (long long)cur + wsum[wi] + wmaxv[j];
              long long pos = (long long)wi * 32 + wpos[j];
              long long kk = (long long)((unsigned long long)val << 32) | (long long)(0xFFFFFFFFu - (uint32_t)pos);
              key = kk > key ? kk : key;
            }
          }
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            long long y = __shfl_xor_sync(0xffffffffu, key, off);
            key = y > key ? y : key;
          }
          if (lane == 0) kred[warp] = key;
          __syncthreads();
          key = LLONG_MIN;
#pragma unroll
          for (int i = 0; i < NT / 32; i++) key = kred[i] > key ? kred[i] : key;
          int mval = (int)(key >> 32);
          if (key != LLONG_MIN && mval > best) {
            best = mval;
            long long pos = 0xFFFFFFFFll - (key & 0xFFFFFFFFll);
            int wstar = (int)(pos >> 5), bstar = (int)(pos & 31);
#pragma unroll
            for (int j = 0; j < WPT; j++) {
              int wi = tid + j * NT;
              if (wi < nw) {
                uint32_t now = st[p * nw + wi];
                uint32_t old = now ^ Am[j];
                uint32_t snap = wi < wstar ? now
                                : wi == wstar
                                    ? old ^ (Am[j] & (bstar == 31 ? 0xFFFFFFFFu : ((2u << bstar) - 1u)))
                                    : old;
                bst[p * nw + wi] = snap;
                bst[(p ^ 1) * nw + wi] = st[(p ^ 1) * nw + wi];
              }
            }
          }
          __syncthreads();
        }
        cur += D;
      }
      executed = t + 1;
      if (!SA && sweep_flips == 0) break;
    }

    // ---- integrity guard (solvers.py:132-133): recompute the cut of best
    __syncthreads();
    int cb = 0;
#pragma unroll
    for (int j = 0; j < WPT; j++) {
      int wi = tid + j * NT;
      if (wi < nw) {
        int e = wr[j] & 1;
        uint32_t same, sh, up, dn;
        neighbours(bst + nw, a.rows, a.WPR, a.lb, wr[j], wcol[j], e, same, sh, up, dn);
        cb += word_cut(bst[wi], same, sh, up, dn, mk[0][j]);
      }
    }
    int cbest = block_sum_int<NT>(cb, red2, 1);
    if (tid == 0) {
      a.best_cut[trial] = best;
      a.sweeps_exec[trial] = executed;
      if (cbest != best) atomicExch(a.err, GSB_EINTEGRITY);
    }
    // ---- pack best spins MSB-first by site id
    uint8_t *out = a.best_bits + (size_t)trial * a.nbytes;
    const int n = a.rows * a.cols;
    for (int byte = tid; byte < a.nbytes; byte += NT) {
      uint32_t v = 0;
#pragma unroll
      for (int q = 0; q < 8; q++) {
        int x = byte * 8 + q;
        uint32_t bit = 0;
        if (x < n) {
          int r = x / a.cols, c = x - r * a.cols;
          int p = (r + c) & 1, k = c >> 1;
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
template <int NT, int WPT>
static int launch_nt(const CheckerArgs &a, bool sa, int nsm, cudaStream_t stream) {
  size_t smem = (size_t)4 * a.nw * 4 + (2 * 96 + 64) * 4 + 32 * 8 + (size_t)a.nw * 4;
  auto kern = sa ? checker_sweep_kernel<NT, WPT, true> : checker_sweep_kernel<NT, WPT, false>;
  if (smem > 48 * 1024) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return set_error(GSB_ECUDA, "cudaFuncSetAttribute failed");
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem) != cudaSuccess ||
      per_sm < 1)
    return set_error(GSB_ECUDA, "checker kernel does not fit on an SM");
  int grid = nsm * per_sm;
  if (grid > a.T) grid = a.T;
  kern<<<grid, NT, smem, stream>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(GSB_ECUDA, cudaGetErrorString(e));
  return GSB_OK;
}

int checker_words(int rows, int cols, int *WPR, int *nw) {
  int H = cols / 2;
  *WPR = (H + 31) / 32;
  *nw = rows * *WPR;
  return 0;
}

bool checker_fits(int rows, int cols) {
  if ((rows & 1) || (cols & 1) || rows < 4 || cols < 4) return false;
  int WPR, nw;
  checker_words(rows, cols, &WPR, &nw);
  return nw <= 4 * 1024;
}

int checker_run(int rows, int cols, const int8_t *w_dev, int kind, int sweeps,
                const uint64_t *table, const uint64_t *seeds, int T, int64_t *best_cut,
                int32_t *sweeps_exec, uint8_t *best_bits, uint32_t *masks_ws, int *err_ws,
                cudaStream_t stream) {
  int WPR, nw;
  checker_words(rows, cols, &WPR, &nw);
  int nsm = num_sms();
  if (nsm <= 0) return set_error(GSB_ECUDA, "no CUDA device");
  checker_masks_kernel<<<(2 * nw + 255) / 256, 256, 0, stream>>>(rows, cols, WPR, w_dev, masks_ws);
  CheckerArgs a;
  a.rows = rows;
  a.cols = cols;
  a.H = cols / 2;
  a.WPR = WPR;
  a.nw = nw;
  a.lb = (a.H - 1) & 31;
  a.masks = masks_ws;
  a.table = table;
  a.sweeps = sweeps;
  a.seeds = seeds;
  a.T = T;
  a.best_cut = best_cut;
  a.sweeps_exec = sweeps_exec;
  a.best_bits = best_bits;
  a.nbytes = (rows * cols + 7) / 8;
  a.err = err_ws;
  bool sa = kind == GSB_ANNEALING;
  // one word per thread per colour where possible
  if (nw <= 32) return launch_nt<32, 1>(a, sa, nsm, stream);
  if (nw <= 64) return launch_nt<64, 1>(a, sa, nsm, stream);
  if (nw <= 128) return launch_nt<128, 1>(a, sa, nsm, stream);
  if (nw <= 224) return launch_nt<224, 1>(a, sa, nsm, stream);
  if (nw <= 320) return launch_nt<320, 1>(a, sa, nsm, stream);
  if (nw <= 416) return launch_nt<416, 1>(a, sa, nsm, stream);
  if (nw <= 512) return launch_nt<512, 1>(a, sa, nsm, stream);
  if (nw <= 1024) return launch_nt<512, 2>(a, sa, nsm, stream);
  if (nw <= 2048) return launch_nt<512, 4>(a, sa, nsm, stream);
  if (nw <= 4096) return launch_nt<512, 8>(a, sa, nsm, stream);
  return set_error(GSB_EUNSUPPORTED, "torus too large for the shared-memory checkerboard path");
}

}  // namespace gsb
