// rscan_bs.cu -- bit-sliced random-scan (Philox) engine.
//
// Same contract and results as rscan.cu (oracle/gsb_oracle.c:trial_rscan,
// DESIGN.md "Random-scan contract"); the rounds run 32 sites per instruction.
// Layout: row-major words of 32 consecutive sites, WPR = ceil(cols / 32)
// words per row, word w = r * WPR + k holds sites (r, 32k + b), padding bits 0.
// Per sweep:
//   1. priorities and uniforms, one Philox block per 4 consecutive sites
//      (lane per quad): priorities to shared memory, uniform top bytes too;
//   2. lane per site, warp per word: the preceding-neighbour planes E[4][w]
//      (ballots of the down and right comparisons; up and left follow from
//      them because "precedes" is a strict total order) and the uniform's top 8 bits as
//      planes PL4[w][2] (ballots; 8 planes per word, 32 B);
//   3. rounds, lane per word: ready = unvisited sites whose preceding
//      neighbours are all visited (bit-sliced over the unvisited planes of the
//      four aligned neighbour words), Delta classes, the 8-plane comparison
//      with the sweep's thresholds (undecided sites draw their block again and
//      compare the low 24 bits), commit, Delta sums, and best-so-far in
//      (round, id) order exactly as the checkerboard engine does per
//      half-sweep.  One barrier per round (the round totals; see below).
#include <climits>
#include <cstdint>

#include "checker_common.cuh"
#include "gsb_device.cuh"
#include "gsb_internal.h"

namespace gsb {

constexpr int RB_NT = 256;
constexpr int RB_NWARP = RB_NT / 32;

struct RbArgs {
  int rows, cols, n, WPR, nw, lb;
  const int8_t *w;
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

struct RbShared {
  int red[2][3][RB_NWARP];
  int scan[8 * RB_NWARP];
  long long kred[RB_NWARP];
};

// ballot of (x & m) != 0: one LOP3 with a predicate result and one VOTE (the
// C++ form compiles to shift, and, compare and predicate spills)
__device__ __forceinline__ uint32_t ballot_bit(uint32_t x, uint32_t m) {
  uint32_t r;
  asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\tand.b32 t, %1, %2;\n\t"
      "setp.ne.u32 p, t, 0;\n\tvote.sync.ballot.b32 %0, p, 0xffffffff;\n\t}"
      : "=r"(r)
      : "r"(x), "r"(m));
  return r;
}

template <int WPT, bool SA>
__global__ void __launch_bounds__(RB_NT) rscan_bs_kernel(RbArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ RbShared sh;
  const int rows = a.rows, cols = a.cols, n = a.n, WPR = a.WPR, nw = a.nw, lb = a.lb;
  const int nq = (n + 3) >> 2;
  uint32_t *prio = (uint32_t *)smem_raw;  // [4 * nq] per site
  uint4 *PL4 = (uint4 *)(prio + 4 * nq);  // [nw][2] uniform bits 31..24 (planes 0-3, 4-7)
  uint32_t *S = (uint32_t *)(PL4 + 2 * nw);  // [nw] spins (1 = +1)
  uint32_t *U = S + nw;                   // [2][nw] unvisited, by round parity
  uint32_t *E = U + 2 * nw;               // [4][nw] preceding neighbour: up, down, left, right
  uint32_t *NC = E + 4 * nw;              // [4][nw] coupling < 0: right, left, up, down neighbour
  uint32_t *BS = NC + 4 * nw;             // [nw] best snapshot
  uint8_t *ub = (uint8_t *)(BS + nw);     // [4 * nq] uniform top bytes
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // geometry of word w: row, column word, valid bits, neighbour words, carries
  auto wgeo = [&](int w, int &r, int &k) {
    r = w / WPR;
    k = w - r * WPR;
  };
  auto vmask = [&](int k) -> uint32_t { return k < WPR - 1 || lb == 31 ? 0xFFFFFFFFu : (2u << lb) - 1u; };
  // X aligned to the left / right neighbours of w's sites (X = a word array)
  auto alignL = [&](const uint32_t *X, int w, int r, int k) -> uint32_t {
    const uint32_t c = k > 0 ? X[w - 1] >> 31 : (X[r * WPR + WPR - 1] >> lb) & 1u;
    return (X[w] << 1) | c;
  };
  auto alignR = [&](const uint32_t *X, int w, int r, int k) -> uint32_t {
    if (k < WPR - 1) return (X[w] >> 1) | ((X[w + 1] & 1u) << 31);
    return (X[w] >> 1) | ((X[r * WPR] & 1u) << lb);
  };
  auto upw = [&](int r, int k) { return (r == 0 ? rows - 1 : r - 1) * WPR + k; };
  auto dnw = [&](int r, int k) { return (r == rows - 1 ? 0 : r + 1) * WPR + k; };

  // ---- static coupling planes (same for every trial)
  for (int w = tid; w < nw; w += RB_NT) {
    int r, k;
    wgeo(w, r, k);
    uint32_t nr = 0, nd = 0;
    for (int b = 0; b < 32; b++) {
      const int c = 32 * k + b;
      if (c >= cols) break;
      const int v = r * cols + c;
      if (a.w[2 * v] < 0) nr |= 1u << b;
      if (a.w[2 * v + 1] < 0) nd |= 1u << b;
    }
    NC[w] = nr;
    NC[3 * nw + w] = nd;
  }
  __syncthreads();
  for (int w = tid; w < nw; w += RB_NT) {
    int r, k;
    wgeo(w, r, k);
    NC[nw + w] = alignL(NC, w, r, k) & vmask(k);  // right coupling of the left neighbour
    NC[2 * nw + w] = NC[3 * nw + upw(r, k)];       // down coupling of the site above
  }
  __syncthreads();

  bool own[WPT];
  int orow[WPT], ocol[WPT];  // (row, column word) of the own words
#pragma unroll
  for (int j = 0; j < WPT; j++) {
    own[j] = j * RB_NT + tid < nw;
    wgeo(own[j] ? j * RB_NT + tid : 0, orow[j], ocol[j]);
  }

  unsigned long long nblocks = 0;
  for (int trial = blockIdx.x; trial < a.T; trial += gridDim.x) {
    const uint64_t seed = a.seeds[trial];
    const uint32_t key0 = (uint32_t)seed, key1 = (uint32_t)(seed >> 32);
    // ---- initial spins (top bit of word v & 3 of Philox(v >> 2, 0, 0, 3)),
    // via the byte array, then packed per word
    for (int q = tid; q < nq; q += RB_NT) {
      const P4 o = philox10(P4{(uint32_t)q, 0u, 0u, 3u}, key0, key1);
      nblocks++;
      ub[4 * q] = (uint8_t)(o.x >> 31);
      ub[4 * q + 1] = (uint8_t)(o.y >> 31);
      ub[4 * q + 2] = (uint8_t)(o.z >> 31);
      ub[4 * q + 3] = (uint8_t)(o.w >> 31);
    }
    __syncthreads();
    for (int w = warp; w < nw; w += RB_NWARP) {
      int r, k;
      wgeo(w, r, k);
      const int c = 32 * k + lane;
      const bool valid = c < cols;
      const uint32_t bit = __ballot_sync(0xffffffffu, valid && ub[r * cols + c]);
      if (lane == 0) {
        S[w] = bit;
        BS[w] = bit;
      }
    }
    __syncthreads();
    // initial cut: right and down edges of own words
    int c0 = 0;
#pragma unroll
    for (int j = 0; j < WPT; j++) {
      if (!own[j]) continue;
      const int w = j * RB_NT + tid;
      const int r = orow[j], k = ocol[j];
      const uint32_t V = vmask(k), s = S[w];
      const uint32_t xr = (s ^ alignR(S, w, r, k)) & V, xd = (s ^ S[dnw(r, k)]) & V;
      c0 += __popc(xr & ~NC[w]) - __popc(xr & NC[w]) + __popc(xd & ~NC[3 * nw + w]) -
            __popc(xd & NC[3 * nw + w]);
    }
    c0 = (int)__reduce_add_sync(0xffffffffu, (unsigned)c0);
    if (lane == 0) sh.scan[warp] = c0;
    __syncthreads();
    int cur = 0;
    for (int i = 0; i < RB_NWARP; i++) cur += sh.scan[i];
    __syncthreads();
    int best = cur, executed = 0;

    for (int t = 0; t < a.sweeps; t++) {
      uint32_t K2 = 0, K4 = 0, K2lo = 0, K4lo = 0, me2 = 0, me4 = 0;
      uint64_t K2f = 0, K4f = 0;
      if (SA) {
        K2f = a.table[(size_t)t * 4 + 1];
        K4f = a.table[(size_t)t * 4 + 3];
        K2 = K2f > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)K2f;
        K4 = K4f > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)K4f;
        K2lo = K2f > 0xFFFFFFFFull ? 0x1000000u : (K2 & 0xFFFFFFu);
        K4lo = K4f > 0xFFFFFFFFull ? 0x1000000u : (K4 & 0xFFFFFFu);
        me2 = K2f ? ~0u : 0u;
        me4 = K4f ? ~0u : 0u;
      }
      // ---- 1. priorities and uniform top bytes (lane per quad)
      for (int q = tid; q < nq; q += RB_NT) {
        nblocks += SA ? 2u : 1u;
        const P4 p = philox10(P4{(uint32_t)q, (uint32_t)t, 0u, 4u}, key0, key1);
        *(uint4 *)&prio[4 * q] = make_uint4(p.x, p.y, p.z, p.w);
        if (SA) {
          const P4 u = philox10(P4{(uint32_t)q, (uint32_t)t, 1u, 4u}, key0, key1);
          *(uint32_t *)&ub[4 * q] =
              (u.x >> 24) | ((u.y >> 24) << 8) | ((u.z >> 24) << 16) | ((u.w >> 24) << 24);
        }
      }
      __syncthreads();
      // ---- 2. preceding-neighbour and uniform planes (warp per word)
      int r2, k2;
      wgeo(warp, r2, k2);
      const int dr = RB_NWARP / WPR, dk = RB_NWARP - dr * WPR;  // word step in (row, column word)
      for (int w = warp; w < nw; w += RB_NWARP) {
        const int r = r2, k = k2;
        k2 += dk;
        r2 += dr;
        if (k2 >= WPR) {
          k2 -= WPR;
          r2++;
        }
        const int c = 32 * k + lane;
        const bool valid = c < cols;
        const int cc = valid ? c : 0;
        const int v = r * cols + cc;
        const int vd = v + (r == rows - 1 ? cols - n : cols);
        const int vr = v + (cc == cols - 1 ? 1 - cols : 1);
        const uint32_t pv = prio[v];
        auto prec = [&](int u) {
          const uint32_t pn = prio[u];
          return (int)valid & ((int)(pn < pv) | ((int)(pn == pv) & (int)(u < v)));
        };
        // only the down and right planes: "precedes" is a strict total order,
        // so up(v) = !down(v - cols) and left(v) = !right(v - 1) (below)
        const uint32_t ed = __ballot_sync(0xffffffffu, prec(vd));
        const uint32_t er = __ballot_sync(0xffffffffu, prec(vr));
        uint32_t pl[8];
        const uint32_t byte = valid ? ub[v] : 0u;
#pragma unroll
        for (int jj = 0; jj < 8; jj++) pl[jj] = ballot_bit(byte, 0x80u >> jj);
        if (lane == 0) {
          E[nw + w] = ed;
          E[3 * nw + w] = er;
          U[nw + w] = vmask(k);  // read by round 1
          if (SA) {
            PL4[2 * w] = make_uint4(pl[0], pl[1], pl[2], pl[3]);
            PL4[2 * w + 1] = make_uint4(pl[4], pl[5], pl[6], pl[7]);
          }
        }
      }
      __syncthreads();
      // up and left planes of the own words from the down / right planes of
      // the neighbours (padding bits stay 0)
#pragma unroll
      for (int j = 0; j < WPT; j++) {
        if (!own[j]) continue;
        const int w = j * RB_NT + tid;
        const int r = orow[j], k = ocol[j];
        const uint32_t V = vmask(k);
        E[w] = ~E[nw + upw(r, k)] & V;
        E[2 * nw + w] = ~alignL(E + 3 * nw, w, r, k) & V;
      }
      __syncthreads();
      bool sweep_flipped = false;
      // ---- 3. rounds
      for (int rr = 1;; rr++) {
        if (rr > 4096) {
          if (tid == 0) atomicExch(a.err, GSB_EUNSUPPORTED);
          break;
        }
        uint32_t rd[WPT];
        int left = 0;
        const uint32_t *Uc = U + (rr & 1) * nw;
        uint32_t *Un = U + ((rr + 1) & 1) * nw;
#pragma unroll
        for (int j = 0; j < WPT; j++) {
          rd[j] = 0;
          if (!own[j]) continue;
          const int w = j * RB_NT + tid;
          const int r = orow[j], k = ocol[j];
          const uint32_t u = Uc[w];
          if (!u) {
            Un[w] = 0u;
            continue;
          }
          const uint32_t block = (E[w] & Uc[upw(r, k)]) | (E[nw + w] & Uc[dnw(r, k)]) |
                                 (E[2 * nw + w] & alignL(Uc, w, r, k)) |
                                 (E[3 * nw + w] & alignR(Uc, w, r, k));
          rd[j] = u & ~block;
          Un[w] = u & block;
          left += __popc(u & block);
        }
        // No barrier before the commits: two sites ready in the same round are
        // never neighbours (one precedes the other), so every bit a ready
        // site's Delta reads is stable during the round, and the unvisited
        // planes are double-buffered (this round reads Uc, writes Un).
        uint32_t A[WPT];
        int wsum[WPT], wpos[WPT];
        int D = 0, P = 0;
#pragma unroll
        for (int j = 0; j < WPT; j++) {
          A[j] = 0;
          wsum[j] = wpos[j] = 0;
          if (!rd[j]) continue;
          const int w = j * RB_NT + tid;
          const int r = orow[j], k = ocol[j];
          const uint32_t V = vmask(k), s = S[w];
          const Classes c = classes(s, alignR(S, w, r, k), alignL(S, w, r, k), S[upw(r, k)],
                                    S[dnw(r, k)],
                                    make_uint4(NC[w], NC[nw + w], NC[2 * nw + w], NC[3 * nw + w]), V);
          const uint32_t ready = rd[j];
          uint32_t acc;
          if (SA) {
            const uint32_t e2 = c.km2 & me2 & ready, e4 = c.km4 & me4 & ready;
            uint32_t eq, lt;
            const uint4 pa = PL4[2 * w], pb = PL4[2 * w + 1];
            const P4 r0{pa.x, pa.y, pa.z, pa.w};
            const P4 r1{pb.x, pb.y, pb.z, pb.w};
            cmp_planes<0>(r0, r1, e2, e2 | e4, K2, K4, eq, lt);
            // undecided sites (top byte equal to K's): the low 24 bits
            while (eq) {
              const int b = __ffs(eq) - 1;
              eq &= eq - 1;
              const int v = r * cols + 32 * k + b;
              const P4 u4 = philox10(P4{(uint32_t)(v >> 2), (uint32_t)t, 1u, 4u}, key0, key1);
              const uint32_t uw = (v & 3) == 0 ? u4.x : (v & 3) == 1 ? u4.y : (v & 3) == 2 ? u4.z : u4.w;
              const uint32_t klo = ((e2 >> b) & 1u) ? K2lo : K4lo;
              if ((uw & 0xFFFFFFu) < klo) lt |= 1u << b;
            }
            acc = (c.ge2 & ready) | lt;
          } else {
            acc = (c.k3 | c.k4) & ready;
          }
          A[j] = acc;
          wpos[j] = 2 * __popc(c.k3 & ready) + 4 * __popc(c.k4 & ready);
          wsum[j] = 2 * __popc(acc & c.k3) + 4 * __popc(acc & c.k4) - 2 * __popc(acc & c.km2) -
                    4 * __popc(acc & c.km4);
          D += wsum[j];
          P += wpos[j];
          S[w] = s ^ acc;
        }
        // ---- round totals
        int all_left;
        {
          const int pr = rr & 1;
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
#pragma unroll
          for (int i = 0; i < RB_NWARP; i++) {
            D += sh.red[pr][0][i];
            P += sh.red[pr][1][i];
            all_left += sh.red[pr][2][i];
          }
        }
        if (P > 0) sweep_flipped = true;
        if (cur + P > best) {
          // prefix of the word sums in word order (j, warp, lane), as checker.cu
          int excl[WPT];
#pragma unroll
          for (int j = 0; j < WPT; j++) {
            int x = wsum[j];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
              const int y = __shfl_up_sync(0xffffffffu, x, off);
              if (lane >= off) x += y;
            }
            excl[j] = x - wsum[j];
            if (lane == 31) sh.scan[j * RB_NWARP + warp] = x;
          }
          __syncthreads();
          int base = 0;
#pragma unroll
          for (int j = 0; j < WPT; j++) {
            int wb = base;
            for (int i = 0; i < RB_NWARP; i++) {
              const int v = sh.scan[j * RB_NWARP + i];
              if (i < warp) wb += v;
              base += v;
            }
            excl[j] += wb + cur;
          }
          long long key = LLONG_MIN;
#pragma unroll
          for (int j = 0; j < WPT; j++) {
            if (!A[j] || wpos[j] <= 0 || excl[j] + wpos[j] <= best) continue;
            const int w = j * RB_NT + tid;
            const int r = orow[j], k = ocol[j];
            const uint32_t V = vmask(k), sold = S[w] ^ A[j];
            const Classes c =
                classes(sold, alignR(S, w, r, k), alignL(S, w, r, k), S[upw(r, k)], S[dnw(r, k)],
                        make_uint4(NC[w], NC[nw + w], NC[2 * nw + w], NC[3 * nw + w]), V);
            const uint32_t Aj = A[j];
            int vrun = excl[j], mx = INT_MIN, mp = -1;
            uint32_t nz = Aj;
            while (nz) {
              const int b = __ffs(nz) - 1;
              nz &= nz - 1;
              const uint32_t bm = 1u << b;
              const int d = (c.k3 & bm) ? 2 : (c.k4 & bm) ? 4 : (c.km2 & bm) ? -2 : (c.km4 & bm) ? -4 : 0;
              vrun += d;
              if (d > 0 && vrun > mx) {
                mx = vrun;
                mp = b;
              }
            }
            if (mp >= 0) {
              const long long pos = (long long)w * 32 + mp;
              const long long kk = (long long)((unsigned long long)(long long)mx << 32) |
                                   (long long)(0xFFFFFFFFu - (uint32_t)pos);
              key = kk > key ? kk : key;
            }
          }
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            const long long y = __shfl_xor_sync(0xffffffffu, key, off);
            key = y > key ? y : key;
          }
          if (lane == 0) sh.kred[warp] = key;
          __syncthreads();
          key = LLONG_MIN;
#pragma unroll
          for (int i = 0; i < RB_NWARP; i++) key = sh.kred[i] > key ? sh.kred[i] : key;
          const int mval = (int)(key >> 32);
          if (key != LLONG_MIN && mval > best) {
            best = mval;
            const long long pos = 0xFFFFFFFFll - (key & 0xFFFFFFFFll);
            const int wstar = (int)(pos >> 5), bstar = (int)(pos & 31);
            for (int w = tid; w < nw; w += RB_NT) {  // all words (other rounds' flips are in S)
              const int j = w / RB_NT;
              uint32_t Aw = 0;
#pragma unroll
              for (int jj = 0; jj < WPT; jj++)
                if (jj == j) Aw = A[jj];
              const uint32_t now = S[w], old = now ^ Aw;
              BS[w] = w < wstar ? now : w == wstar ? old ^ (Aw & ((2u << bstar) - 1u)) : old;
            }
          }
          __syncthreads();
        }
        cur += D;
        if (all_left == 0) break;
      }
      executed = t + 1;
      if (!SA && !sweep_flipped) break;
    }

    // ---- integrity guard (solvers.py:132-133)
    __syncthreads();
    int cb = 0;
#pragma unroll
    for (int j = 0; j < WPT; j++) {
      if (!own[j]) continue;
      const int w = j * RB_NT + tid;
      const int r = orow[j], k = ocol[j];
      const uint32_t V = vmask(k), s = BS[w];
      const uint32_t xr = (s ^ alignR(BS, w, r, k)) & V, xd = (s ^ BS[dnw(r, k)]) & V;
      cb += __popc(xr & ~NC[w]) - __popc(xr & NC[w]) + __popc(xd & ~NC[3 * nw + w]) -
            __popc(xd & NC[3 * nw + w]);
    }
    cb = (int)__reduce_add_sync(0xffffffffu, (unsigned)cb);
    if (lane == 0) sh.scan[warp] = cb;
    __syncthreads();
    if (tid == 0) {
      int cbest = 0;
      for (int i = 0; i < RB_NWARP; i++) cbest += sh.scan[i];
      a.best_cut[trial] = best;
      a.sweeps_exec[trial] = executed;
      if (cbest != best) atomicExch(a.err, GSB_EINTEGRITY);
    }
    // ---- best spins MSB-first by site id
    uint8_t *out = a.best_bits + (size_t)trial * a.nbytes;
    for (int byte = tid; byte < a.nbytes; byte += RB_NT) {
      uint32_t v8 = 0;
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const int x = byte * 8 + q;
        uint32_t bit = 0;
        if (x < n) {
          const int r = x / cols, c = x - r * cols;
          bit = (BS[r * WPR + (c >> 5)] >> (c & 31)) & 1u;
        }
        v8 |= bit << (7 - q);
      }
      out[byte] = (uint8_t)v8;
    }
    __syncthreads();
  }
  const unsigned long long nb = __reduce_add_sync(0xffffffffu, (unsigned)nblocks);
  if (lane == 0 && nb) atomicAdd(a.blocks, nb);
}

// ------------------------------------------------------------------ host
static size_t rb_smem(int n, int nw) {
  const size_t nq = (size_t)(n + 3) / 4;
  return nq * 16 + (size_t)nw * 4 * 20 + nq * 4;
}

static int rb_wpt(int rows, int cols) {
  const int WPR = (cols + 31) / 32;
  const long long nw = (long long)rows * WPR;
  const long long wpt = (nw + RB_NT - 1) / RB_NT;
  return wpt <= 8 ? (int)wpt : 0;
}

bool rscan_bs_fits(int rows, int cols) {
  if (rows < 3 || cols < 3) return false;
  const int wpt = rb_wpt(rows, cols);
  if (!wpt) return false;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return false;
  const int WPR = (cols + 31) / 32;
  return rb_smem(rows * cols, rows * WPR) + sizeof(RbShared) <= (size_t)optin;
}

template <int WPT>
static int rb_launch(const RbArgs &a, bool sa, cudaStream_t stream) {
  const size_t smem = rb_smem(a.n, a.nw);
  auto kern = sa ? rscan_bs_kernel<WPT, true> : rscan_bs_kernel<WPT, false>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return set_error(GSB_ECUDA, "cudaFuncSetAttribute failed");
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, RB_NT, smem) != cudaSuccess ||
      per_sm < 1)
    return set_error(GSB_ECUDA, "bit-sliced random-scan kernel does not fit on an SM");
  int grid = num_sms() * per_sm;
  if (grid > a.T) grid = a.T;
  kern<<<grid, RB_NT, smem, stream>>>(a);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(GSB_ECUDA, cudaGetErrorString(e));
  return GSB_OK;
}

int rscan_bs_run(int rows, int cols, const int8_t *w_dev, int kind, int sweeps,
                 const uint64_t *table, const uint64_t *seeds, int T, int64_t *best_cut,
                 int32_t *sweeps_exec, uint8_t *best_bits, int *err_ws, cudaStream_t stream) {
  if (!rscan_bs_fits(rows, cols))
    return set_error(GSB_EUNSUPPORTED, "torus too large for the random-scan engine");
  RbArgs a;
  a.rows = rows;
  a.cols = cols;
  a.n = rows * cols;
  a.WPR = (cols + 31) / 32;
  a.nw = rows * a.WPR;
  a.lb = (cols - 1) & 31;
  a.w = w_dev;
  a.table = table;
  a.sweeps = sweeps;
  a.seeds = seeds;
  a.T = T;
  a.best_cut = best_cut;
  a.sweeps_exec = sweeps_exec;
  a.best_bits = best_bits;
  a.nbytes = (a.n + 7) / 8;
  a.err = err_ws;
  a.blocks = (unsigned long long *)((char *)err_ws + 8);
  const bool sa = kind == GSB_ANNEALING;
  switch (rb_wpt(rows, cols)) {
    case 1: return rb_launch<1>(a, sa, stream);
    case 2: return rb_launch<2>(a, sa, stream);
    case 3: return rb_launch<3>(a, sa, stream);
    case 4: return rb_launch<4>(a, sa, stream);
    case 5: return rb_launch<5>(a, sa, stream);
    case 6: return rb_launch<6>(a, sa, stream);
    case 7: return rb_launch<7>(a, sa, stream);
    default: return rb_launch<8>(a, sa, stream);
  }
}

}  // namespace gsb
