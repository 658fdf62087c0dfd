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
// registers; shared memory holds the copy its neighbours read, the couplings
// (4 sign planes per word, uint4) and the best-so-far snapshot.
//
// Per word and half-sweep: 4 positive-term planes P_j = ~(S^N_j^NEG_j),
// bit-sliced counts -> Delta classes, then for the Delta<0 sites an MSB-first
// bit-sliced comparison of the 32-bit uniform with K = ceil(exp(Delta/T)*2^32):
// Philox planes 0-7 are drawn unconditionally (two calls), later planes only
// while a site of the word is still undecided.
//
// Best-so-far (solvers.py:125-127) per half-sweep: the running cut in visit
// order is cur + prefix sum of the accepted Deltas; a block reduction gives the
// half-sweep total and the sum of positive Deltas, which bounds every prefix.
// Only if that bound can beat `best` are per-word prefix bounds formed, and
// only candidate words run the exact bit-serial maximum; the first position of
// the maximum defines the snapshot (pre-phase words + accepted flips up to it).
#include <climits>
#include <cstdint>

#include "gsb_device.cuh"
#include "gsb_internal.h"

namespace gsb {

// masks: [2][nw] uint4 {NS, NSH, NU, ND} (bit = weight -1) and valid[2][nw]
__global__ void checker_masks_kernel(int rows, int cols, int WPR, const int8_t *__restrict__ w,
                                     uint4 *__restrict__ masks, uint32_t *__restrict__ valid) {
  const int H = cols >> 1;
  const int nw = rows * WPR;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < 2 * nw;
       idx += gridDim.x * blockDim.x) {
    int p = idx / nw, wi = idx % nw;
    int r = wi / WPR, ww = wi % WPR;
    int e = (r + p) & 1;
    uint32_t ns = 0, nsh = 0, nu = 0, nd = 0, v = 0;
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
      v |= 1u << b;
      if (wsame < 0) ns |= 1u << b;
      if (wsh < 0) nsh |= 1u << b;
      if (w_up < 0) nu |= 1u << b;
      if (w_down < 0) nd |= 1u << b;
    }
    masks[idx] = make_uint4(ns, nsh, nu, nd);
    valid[idx] = v;
  }
}

struct CheckerArgs {
  int rows, cols, H, WPR, nw, lb;
  const uint4 *masks;
  const uint32_t *valid;
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

// per-thread geometry of one owned word (both colours share up/dn rows)
struct WordGeo {
  int up, dn;         // word index of the row above / below (same ww)
  int cidx[2];        // carry word for colour p (shifted neighbour)
  uint32_t cinfo[2];  // bits 0-4: source bit, 5-9: destination bit, 10: direction (1 = k+1)
};

__device__ __forceinline__ uint32_t shifted_nb(const uint32_t *__restrict__ o, uint32_t same,
                                               int cidx, uint32_t cinfo) {
  const uint32_t src = cinfo & 31u, dst = (cinfo >> 5) & 31u;
  const uint32_t carry = ((o[cidx] >> src) & 1u) << dst;
  return ((cinfo >> 10) & 1u) ? ((same >> 1) | carry) : ((same << 1) | carry);
}

// cut contribution of a colour-0 word: sum over its 4 edges of w*[differ]
__device__ __forceinline__ int word_cut(uint32_t s, uint32_t same, uint32_t sh, uint32_t up,
                                        uint32_t dn, uint4 m, uint32_t v) {
  int c = 0;
  uint32_t x;
  x = (s ^ same) & v;
  c += __popc(x & ~m.x) - __popc(x & m.x);
  x = (s ^ sh) & v;
  c += __popc(x & ~m.y) - __popc(x & m.y);
  x = (s ^ up) & v;
  c += __popc(x & ~m.z) - __popc(x & m.z);
  x = (s ^ dn) & v;
  c += __popc(x & ~m.w) - __popc(x & m.w);
  return c;
}

// MSB-first bit-sliced compare step for the 4 planes of Philox group g
__device__ __forceinline__ void cmp_planes(P4 r, int g, uint32_t K2, uint32_t K4, uint32_t e2,
                                           uint32_t e4, uint32_t &eq, uint32_t &lt) {
  const uint32_t pl[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const int bit = 31 - (4 * g + q);
    const uint32_t m2 = (uint32_t)((int32_t)(K2 << (31 - bit)) >> 31);
    const uint32_t m4 = (uint32_t)((int32_t)(K4 << (31 - bit)) >> 31);
    const uint32_t tb = (e2 & m2) | (e4 & m4);
    const uint32_t R = pl[q];
    lt |= eq & ~R & tb;
    eq &= ~(R ^ tb);
  }
}

template <int NT, int WPT, bool SA>
__global__ void __launch_bounds__(NT) checker_sweep_kernel(CheckerArgs a) {
  constexpr int NWARP = NT / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nw = a.nw;
  uint4 *msk = (uint4 *)smem_raw;             // [2][nw]
  uint32_t *st = (uint32_t *)(msk + 2 * nw);  // [2][nw] neighbour copy
  uint32_t *bst = st + 2 * nw;                // [2][nw] best snapshot
  int *red = (int *)(bst + 2 * nw);           // [2 buffers][2][NWARP]
  int *red2 = red + 4 * NWARP;                // [2][NWARP] misc
  int *scan = red2 + 2 * NWARP;               // [WPT][NWARP]
  long long *kred = (long long *)(scan + ((WPT * NWARP + 1) & ~1));  // [NWARP]

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  // ---- per-kernel setup: couplings to shared memory, per-thread geometry
  for (int i = tid; i < 2 * nw; i += NT) msk[i] = a.masks[i];
  WordGeo geo[WPT];
  uint32_t vmask[2][WPT];
  bool own[WPT];
#pragma unroll
  for (int j = 0; j < WPT; j++) {
    const int wi = j * NT + tid;
    own[j] = wi < nw;
    const int wic = own[j] ? wi : 0;
    const int r = wic / a.WPR, ww = wic - r * a.WPR;
    geo[j].up = (r == 0 ? a.rows - 1 : r - 1) * a.WPR + ww;
    geo[j].dn = (r == a.rows - 1 ? 0 : r + 1) * a.WPR + ww;
#pragma unroll
    for (int p = 0; p < 2; p++) {
      const int e = (r + p) & 1;
      if (e == 0) {  // k-1 neighbour: carry from the previous word (or row end)
        geo[j].cidx[p] = ww > 0 ? wic - 1 : r * a.WPR + a.WPR - 1;
        geo[j].cinfo[p] = (uint32_t)(ww > 0 ? 31 : a.lb);
      } else {  // k+1 neighbour: carry from the next word (or row start)
        geo[j].cidx[p] = ww < a.WPR - 1 ? wic + 1 : r * a.WPR;
        geo[j].cinfo[p] = ((uint32_t)(ww < a.WPR - 1 ? 31 : a.lb) << 5) | (1u << 10);
      }
      vmask[p][j] = own[j] ? a.valid[p * nw + wi] : 0u;
    }
  }
  __syncthreads();

  for (int trial = blockIdx.x; trial < a.T; trial += gridDim.x) {
    const uint64_t seed = a.seeds[trial];
    const uint32_t key0 = (uint32_t)seed, key1 = (uint32_t)(seed >> 32);

    // ---- initial spins: bit (k&31) of word 0 of Philox(key, (wi, 0, p, 0))
    uint32_t S[2][WPT];
#pragma unroll
    for (int j = 0; j < WPT; j++) {
      const int wi = j * NT + tid;
#pragma unroll
      for (int p = 0; p < 2; p++) {
        S[p][j] = 0;
        if (own[j]) {
          P4 o = philox10(P4{(uint32_t)wi, 0u, (uint32_t)p, 0u}, key0, key1);
          S[p][j] = o.x & vmask[p][j];
          st[p * nw + wi] = S[p][j];
          bst[p * nw + wi] = S[p][j];
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
        const uint32_t *o = st + nw;
        const uint32_t same = S[1][j];
        const uint32_t sh = shifted_nb(o, same, geo[j].cidx[0], geo[j].cinfo[0]);
        c0 += word_cut(S[0][j], same, sh, o[geo[j].up], o[geo[j].dn], msk[wi], vmask[0][j]);
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
      uint32_t K2 = 0, K4 = 0;
      bool all2 = false, all4 = false;
      if (SA) {
        const uint64_t t2 = a.table[(size_t)t * 4 + 1], t4 = a.table[(size_t)t * 4 + 3];
        all2 = t2 > 0xFFFFFFFFull;
        all4 = t4 > 0xFFFFFFFFull;
        K2 = (uint32_t)t2;
        K4 = (uint32_t)t4;
      }
      bool sweep_flipped = false;
#pragma unroll
      for (int p = 0; p < 2; p++, buf ^= 1) {
        const uint32_t *o = st + (p ^ 1) * nw;
        uint32_t Am[WPT], Pos2[WPT], Pos4[WPT], Neg2[WPT], Neg4[WPT];
        int dsum = 0, psum = 0;
#pragma unroll
        for (int j = 0; j < WPT; j++) {
          const int wi = j * NT + tid;
          Am[j] = Pos2[j] = Pos4[j] = Neg2[j] = Neg4[j] = 0;
          if (own[j]) {
            const uint4 m = msk[p * nw + wi];
            const uint32_t V = vmask[p][j];
            const uint32_t Sw = S[p][j];
            const uint32_t same = S[p ^ 1][j];
            const uint32_t sh = shifted_nb(o, same, geo[j].cidx[p], geo[j].cinfo[p]);
            const uint32_t up = o[geo[j].up], dn = o[geo[j].dn];
            const uint32_t P0 = ~(Sw ^ same ^ m.x);
            const uint32_t P1 = ~(Sw ^ sh ^ m.y);
            const uint32_t P2 = ~(Sw ^ up ^ m.z);
            const uint32_t P3 = ~(Sw ^ dn ^ m.w);
            const uint32_t x01 = P0 ^ P1, c01 = P0 & P1, x23 = P2 ^ P3, c23 = P2 & P3;
            const uint32_t ones = x01 ^ x23;
            const uint32_t ge2 = c01 | c23 | (x01 & x23);  // Delta >= 0
            const uint32_t k4 = c01 & c23 & V;             // Delta = +4
            const uint32_t k3 = ((c01 | c23) & ones) & V;  // Delta = +2
            const uint32_t any = P0 | P1 | P2 | P3;
            const uint32_t km2 = any & ~ge2 & V;           // Delta = -2
            const uint32_t km4 = ~any & V;                 // Delta = -4
            uint32_t A;
            if (SA) {
              A = ge2 & V;
              if (all2) A |= km2;
              if (all4) A |= km4;
              const uint32_t e2 = (all2 || K2 == 0) ? 0u : km2;
              const uint32_t e4 = (all4 || K4 == 0) ? 0u : km4;
              uint32_t eq = e2 | e4, lt = 0;
              const P4 r0 =
                  philox10(P4{(uint32_t)wi, (uint32_t)t, (uint32_t)(8 * p), 1u}, key0, key1);
              const P4 r1 =
                  philox10(P4{(uint32_t)wi, (uint32_t)t, (uint32_t)(8 * p + 1), 1u}, key0, key1);
              cmp_planes(r0, 0, K2, K4, e2, e4, eq, lt);
              cmp_planes(r1, 1, K2, K4, e2, e4, eq, lt);
#pragma unroll 1
              for (int g = 2; g < 8 && eq; g++) {
                const P4 r =
                    philox10(P4{(uint32_t)wi, (uint32_t)t, (uint32_t)(8 * p + g), 1u}, key0, key1);
                cmp_planes(r, g, K2, K4, e2, e4, eq, lt);
              }
              A |= lt;
            } else {
              A = k4 | k3;
            }
            const uint32_t Sn = Sw ^ A;
            S[p][j] = Sn;
            st[p * nw + wi] = Sn;
            Am[j] = A;
            Pos2[j] = A & k3;
            Pos4[j] = A & k4;
            Neg2[j] = A & km2;
            Neg4[j] = A & km4;
            const int pp = 2 * __popc(Pos2[j]) + 4 * __popc(Pos4[j]);
            psum += pp;
            dsum += pp - 2 * __popc(Neg2[j]) - 4 * __popc(Neg4[j]);
          }
        }
        // ---- block reduction of (dsum, psum): REDUX per warp, one barrier
        const int wd = (int)__reduce_add_sync(0xffffffffu, (unsigned)dsum);
        const int wp = (int)__reduce_add_sync(0xffffffffu, (unsigned)psum);
        int *rb = red + buf * 2 * NWARP;
        if (lane == 0) {
          rb[warp] = wd;
          rb[NWARP + warp] = wp;
        }
        __syncthreads();
        int D = 0, Pt = 0;
#pragma unroll
        for (int i = 0; i < NWARP; i++) {
          D += rb[i];
          Pt += rb[NWARP + i];
        }
        if (Pt > 0) sweep_flipped = true;  // greedy flips are exactly the positive ones
        if (cur + Pt > best) {
          // ---- per-word prefix bounds; word order is (j, tid)
          int wpos[WPT], excl[WPT];
#pragma unroll
          for (int j = 0; j < WPT; j++) {
            wpos[j] = 2 * __popc(Pos2[j]) + 4 * __popc(Pos4[j]);
            const int ws = wpos[j] - 2 * __popc(Neg2[j]) - 4 * __popc(Neg4[j]);
            int incl = ws;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
              const int y = __shfl_up_sync(0xffffffffu, incl, off);
              if (lane >= off) incl += y;
            }
            excl[j] = incl - ws;
            if (lane == 31) scan[j * NWARP + warp] = incl;
          }
          __syncthreads();
          int base = 0;
          bool cand = false;
#pragma unroll
          for (int j = 0; j < WPT; j++) {
            int wbase = base;
            for (int i = 0; i < NWARP; i++) {
              const int v = scan[j * NWARP + i];
              if (i < warp) wbase += v;
              base += v;
            }
            excl[j] += wbase;
            if (own[j] && wpos[j] > 0 && cur + excl[j] + wpos[j] > best) cand = true;
          }
          if (__syncthreads_or(cand)) {
            long long key = LLONG_MIN;
#pragma unroll
            for (int j = 0; j < WPT; j++) {
              if (!own[j] || wpos[j] <= 0 || cur + excl[j] + wpos[j] <= best) continue;
              int v = cur + excl[j], mx = INT_MIN, mp = -1;
              uint32_t nz = Pos2[j] | Pos4[j] | Neg2[j] | Neg4[j];
              while (nz) {
                const int b = __ffs(nz) - 1;
                nz &= nz - 1;
                const uint32_t bm = 1u << b;
                const int d = (Pos2[j] & bm) ? 2 : (Pos4[j] & bm) ? 4 : (Neg2[j] & bm) ? -2 : -4;
                v += d;
                if (d > 0 && v > mx) {
                  mx = v;
                  mp = b;
                }
              }
              const long long pos = (long long)(j * NT + tid) * 32 + mp;
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
            key = LLONG_MIN;
#pragma unroll
            for (int i = 0; i < NWARP; i++) key = kred[i] > key ? kred[i] : key;
            const int mval = (int)(key >> 32);
            if (key != LLONG_MIN && mval > best) {
              best = mval;
              const long long pos = 0xFFFFFFFFll - (key & 0xFFFFFFFFll);
              const int wstar = (int)(pos >> 5), bstar = (int)(pos & 31);
#pragma unroll
              for (int j = 0; j < WPT; j++) {
                if (!own[j]) continue;
                const int wi = j * NT + tid;
                const uint32_t now = S[p][j], old = now ^ Am[j];
                const uint32_t snap = wi < wstar    ? now
                                      : wi == wstar ? old ^ (Am[j] & ((2u << bstar) - 1u))
                                                    : old;
                bst[p * nw + wi] = snap;
                bst[(p ^ 1) * nw + wi] = S[p ^ 1][j];
              }
            }
          }
        }
        cur += D;
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
        const uint32_t *o = bst + nw;
        const uint32_t same = o[wi];
        const uint32_t sh = shifted_nb(o, same, geo[j].cidx[0], geo[j].cinfo[0]);
        cb += word_cut(bst[wi], same, sh, o[geo[j].up], o[geo[j].dn], msk[wi], vmask[0][j]);
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
  size_t b = (size_t)2 * nw * 16 + (size_t)4 * nw * 4;
  b += (size_t)(6 * NWARP) * 4;
  b += (size_t)((WPT * NWARP + 1) & ~1) * 4;
  b += (size_t)NWARP * 8;
  return b;
}

template <int NT, int WPT>
static int launch_nt(const CheckerArgs &a, bool sa, int nsm, cudaStream_t stream) {
  const size_t smem = smem_bytes(a.nw, NT, WPT);
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
  return nw <= 4096;
}

size_t checker_workspace_bytes(int rows, int cols) {
  int WPR, nw;
  checker_words(rows, cols, &WPR, &nw);
  return align_up((size_t)2 * nw * 16, 256) + align_up((size_t)2 * nw * 4, 256);
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
  uint32_t *valid = (uint32_t *)((char *)ws + align_up((size_t)2 * nw * 16, 256));
  checker_masks_kernel<<<(2 * nw + 255) / 256, 256, 0, stream>>>(rows, cols, WPR, w_dev, masks,
                                                                 valid);
  CheckerArgs a;
  a.rows = rows;
  a.cols = cols;
  a.H = cols / 2;
  a.WPR = WPR;
  a.nw = nw;
  a.lb = (a.H - 1) & 31;
  a.masks = masks;
  a.valid = valid;
  a.table = table;
  a.sweeps = sweeps;
  a.seeds = seeds;
  a.T = T;
  a.best_cut = best_cut;
  a.sweeps_exec = sweeps_exec;
  a.best_bits = best_bits;
  a.nbytes = (rows * cols + 7) / 8;
  a.err = err_ws;
  const bool sa = kind == GSB_ANNEALING;
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
