// refexact.cu -- reference-exact sweep engine: bit-for-bit
// gsetbench.solvers.run_trial (solvers.py:91-140) on the GPU.
//
// The trial consumes numpy's default_rng(seed) PCG64 stream exactly as the
// reference does (gsb_device.cuh): n next32 draws for the initial spins
// (solvers.py:96), per sweep a Fisher-Yates permutation with masked rejection
// (solvers.py:110), and one next64 per Delta<0 visit for SA (solvers.py:118),
// accepted iff (next64 >> 11) < K[t][-Delta] with K = ceil(exp(Delta/T)*2^53)
// from the host (bit-identical to `random() < math.exp(delta/temp)`).
//
// v0 layout: one thread per trial, per-trial spins/best/permutation in global
// memory (trial-major).  Correctness baseline for the warp-cooperative engine.
#include <cub/device/device_scan.cuh>
#include <cstdint>

#include "gsb_device.cuh"
#include "gsb_internal.h"

namespace gsb {

struct Pcg {
  u128 s, inc;
  int has32;
  uint32_t buf;
  __device__ __forceinline__ uint64_t next64() {
    s = s * pcg_mult() + inc;
    return pcg_out(s);
  }
  __device__ __forceinline__ uint32_t next32() {
    if (has32) {
      has32 = 0;
      return buf;
    }
    uint64_t x = next64();
    has32 = 1;
    buf = (uint32_t)(x >> 32);
    return (uint32_t)x;
  }
  __device__ __forceinline__ uint32_t interval(uint32_t max) {
    uint32_t mask = max;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    uint32_t v;
    while ((v = (next32() & mask)) > max) {
    }
    return v;
  }
};

struct TorusG {
  int rows, cols;
  const int8_t *w;
  __device__ __forceinline__ int delta(const int8_t *s, int i) const {
    int r = i / cols, c = i - r * cols;
    int cr = c + 1 == cols ? 0 : c + 1, cl = c == 0 ? cols - 1 : c - 1;
    int rd = r + 1 == rows ? 0 : r + 1, ru = r == 0 ? rows - 1 : r - 1;
    int acc = w[2 * i] * s[r * cols + cr] + w[2 * i + 1] * s[rd * cols + c] +
              w[2 * (r * cols + cl)] * s[r * cols + cl] + w[2 * (ru * cols + c) + 1] * s[ru * cols + c];
    return acc * s[i];
  }
  __device__ long long cut(const int8_t *s) const {
    long long cc = 0;
    int n = rows * cols;
    for (int x = 0; x < n; x++) {
      int r = x / cols, c = x - r * cols;
      int right = r * cols + (c + 1 == cols ? 0 : c + 1);
      int down = (r + 1 == rows ? 0 : r + 1) * cols + c;
      if (s[x] != s[right]) cc += w[2 * x];
      if (s[x] != s[down]) cc += w[2 * x + 1];
    }
    return cc;
  }
};

struct CsrG {
  int n;
  const int64_t *off;
  const int32_t *nbr;
  const int32_t *wt;
  __device__ __forceinline__ long long delta(const int8_t *s, int i) const {
    long long acc = 0;
    for (int64_t e = off[i]; e < off[i + 1]; e++) acc += (long long)wt[e] * s[nbr[e]];
    return acc * s[i];
  }
  __device__ long long cut(const int8_t *s) const {
    long long cc = 0;
    for (int v = 0; v < n; v++)
      for (int64_t e = off[v]; e < off[v + 1]; e++)
        if (nbr[e] > v && s[v] != s[nbr[e]]) cc += wt[e];
    return cc;
  }
};

template <class G>
__global__ void ref_thread_kernel(G g, int n, int kind, int sweeps, const uint64_t *table,
                                  int dmax, const uint64_t *seeds, int T, int64_t *best_cut,
                                  int32_t *sweeps_exec, uint8_t *best_bits, int8_t *spins_ws,
                                  int8_t *best_ws, uint32_t *perm_ws, int *err) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  int8_t *s = spins_ws + (size_t)t * n;
  int8_t *bs = best_ws + (size_t)t * n;
  uint32_t *a = perm_ws + (size_t)t * n;
  Pcg g_;
  pcg_seed(seeds[t], g_.s, g_.inc);
  g_.has32 = 0;
  g_.buf = 0;
  for (int v = 0; v < n; v++) s[v] = (g_.next32() >> 31) ? 1 : -1;  // solvers.py:96
  long long cur = g.cut(s);                                          // :101
  long long best = cur;
  for (int v = 0; v < n; v++) bs[v] = s[v];
  int executed = 0;
  const bool sa = kind == GSB_ANNEALING;
  for (int sweep = 0; sweep < sweeps; sweep++) {
    for (int i = 0; i < n; i++) a[i] = i;
    for (int i = n - 1; i >= 1; i--) {  // rng.permutation(n), :110
      uint32_t j = g_.interval((uint32_t)i);
      uint32_t tmp = a[i];
      a[i] = a[j];
      a[j] = tmp;
    }
    bool flipped = false;
    const uint64_t *K = sa ? table + (size_t)sweep * dmax : nullptr;
    for (int k = 0; k < n; k++) {
      int i = (int)a[k];
      long long d = g.delta(s, i);  // :111-115
      bool accept;
      if (sa) {
        accept = d >= 0;
        if (!accept) {
          uint64_t x = g_.next64() >> 11;  // rng.random(), :118
          long long md = -d;
          accept = md <= dmax && x < K[md - 1];
        }
      } else {
        accept = d > 0;
      }
      if (accept) {
        s[i] = (int8_t)-s[i];
        cur += d;
        flipped = true;
        if (cur > best) {  // :125-127
          best = cur;
          for (int v = 0; v < n; v++) bs[v] = s[v];
        }
      }
    }
    executed = sweep + 1;
    if (!sa && !flipped) break;
  }
  if (g.cut(bs) != best) atomicExch(err, GSB_EINTEGRITY);  // :132-133
  best_cut[t] = best;
  sweeps_exec[t] = executed;
  uint8_t *out = best_bits + (size_t)t * ((n + 7) / 8);
  for (int byte = 0; byte < (n + 7) / 8; byte++) {
    uint32_t v = 0;
    for (int q = 0; q < 8; q++) {
      int x = byte * 8 + q;
      if (x < n && bs[x] > 0) v |= 1u << (7 - q);
    }
    out[byte] = (uint8_t)v;
  }
}

size_t ref_workspace_bytes(int n, int64_t m_adj, int T) {
  size_t b = 4096;                        // jump-ahead table of the warp engine
  b += align_up((size_t)T * n, 256);      // spins
  b += align_up((size_t)T * n, 256);      // best
  b += align_up((size_t)T * n * 4, 256);  // permutation
  if (m_adj > 0) {
    b += align_up(((size_t)n + 1) * 8, 256);  // off
    b += align_up((size_t)m_adj * 4, 256);    // nbr
    b += align_up((size_t)m_adj * 4, 256);    // wt
    b += align_up(((size_t)n + 1) * 8, 256);  // fill cursor
    b += 1 << 20;                             // cub scan scratch
  }
  return b;
}

struct RefWs {
  int8_t *spins, *best;
  uint32_t *perm;
  char *rest;
};

static RefWs carve(void *ws, int n, int T) {
  char *p = (char *)ws;
  RefWs r;
  r.spins = (int8_t *)p;
  p += align_up((size_t)T * n, 256);
  r.best = (int8_t *)p;
  p += align_up((size_t)T * n, 256);
  r.perm = (uint32_t *)p;
  p += align_up((size_t)T * n * 4, 256);
  r.rest = p;
  return r;
}

int ref_run_torus(int rows, int cols, const int8_t *w_dev, int kind, int sweeps,
                  const uint64_t *table, int dmax, const uint64_t *seeds, int T,
                  int64_t *best_cut, int32_t *sweeps_exec, uint8_t *best_bits, void *ws,
                  size_t ws_bytes, int *err_ws, cudaStream_t stream) {
  int n = rows * cols;
  if (ws_bytes < ref_workspace_bytes(n, 0, T)) return set_error(GSB_ENOMEM, "workspace too small");
  RefWs r = carve(ws, n, T);
  TorusG g{rows, cols, w_dev};
  ref_thread_kernel<TorusG><<<(T + 63) / 64, 64, 0, stream>>>(
      g, n, kind, sweeps, table, dmax, seeds, T, best_cut, sweeps_exec, best_bits, r.spins,
      r.best, r.perm, err_ws);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GSB_OK : set_error(GSB_ECUDA, cudaGetErrorString(e));
}

__global__ void csr_count_kernel(int64_t m, const int32_t *eu, const int32_t *ev,
                                 unsigned long long *deg) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x) {
    atomicAdd(deg + eu[k] + 1, 1ull);
    atomicAdd(deg + ev[k] + 1, 1ull);
  }
}

__global__ void csr_fill_kernel(int64_t m, const int32_t *eu, const int32_t *ev, const int32_t *ew,
                                unsigned long long *fill, int32_t *nbr, int32_t *wt) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long a = atomicAdd(fill + eu[k], 1ull);
    nbr[a] = ev[k];
    wt[a] = ew[k];
    unsigned long long b = atomicAdd(fill + ev[k], 1ull);
    nbr[b] = eu[k];
    wt[b] = ew[k];
  }
}

int ref_run_graph(const gsb_graph *gr, int kind, int sweeps, const uint64_t *table, int dmax,
                  const uint64_t *seeds, int T, int64_t *best_cut, int32_t *sweeps_exec,
                  uint8_t *best_bits, void *ws, size_t ws_bytes, int *err_ws,
                  cudaStream_t stream) {
  int n = gr->n;
  int64_t madj = 2 * gr->m;
  if (ws_bytes < ref_workspace_bytes(n, madj > 0 ? madj : 1, T))
    return set_error(GSB_ENOMEM, "workspace too small");
  RefWs r = carve(ws, n, T);
  char *p = r.rest;
  int64_t *off = (int64_t *)p;
  p += align_up(((size_t)n + 1) * 8, 256);
  int32_t *nbr = (int32_t *)p;
  p += align_up((size_t)(madj > 0 ? madj : 1) * 4, 256);
  int32_t *wt = (int32_t *)p;
  p += align_up((size_t)(madj > 0 ? madj : 1) * 4, 256);
  unsigned long long *fill = (unsigned long long *)p;
  p += align_up(((size_t)n + 1) * 8, 256);
  void *scratch = p;
  size_t scratch_bytes = 1 << 20;
  if (cudaMemsetAsync(off, 0, ((size_t)n + 1) * 8, stream) != cudaSuccess)
    return set_error(GSB_ECUDA, "memset failed");
  if (gr->m > 0)
    csr_count_kernel<<<256, 256, 0, stream>>>(gr->m, gr->eu_dev, gr->ev_dev,
                                              (unsigned long long *)off);
  size_t need = 0;
  cub::DeviceScan::InclusiveSum(nullptr, need, (unsigned long long *)off,
                                (unsigned long long *)off, n + 1, stream);
  if (need > scratch_bytes) return set_error(GSB_ENOMEM, "cub scratch too small");
  cub::DeviceScan::InclusiveSum(scratch, need, (unsigned long long *)off,
                                (unsigned long long *)off, n + 1, stream);
  cudaMemcpyAsync(fill, off, ((size_t)n + 1) * 8, cudaMemcpyDeviceToDevice, stream);
  if (gr->m > 0)
    csr_fill_kernel<<<256, 256, 0, stream>>>(gr->m, gr->eu_dev, gr->ev_dev, gr->ew_dev, fill, nbr,
                                             wt);
  CsrG g{n, off, nbr, wt};
  ref_thread_kernel<CsrG><<<(T + 63) / 64, 64, 0, stream>>>(
      g, n, kind, sweeps, table, dmax, seeds, T, best_cut, sweeps_exec, best_bits, r.spins,
      r.best, r.perm, err_ws);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GSB_OK : set_error(GSB_ECUDA, cudaGetErrorString(e));
}

}  // namespace gsb
