// evaluate.cu -- exact cut / energy evaluator (evaluate.py:35-49), torus weight
// generation (instances.py:203-224) and the multi-GPU best-key helper.
#include <cstdint>
#include <cstring>

#include "gsb_device.cuh"
#include "gsb_internal.h"

namespace gsb {

__device__ __forceinline__ int get_bit(const uint8_t *__restrict__ b, int x) {
  return (b[x >> 3] >> (7 - (x & 7))) & 1;
}

// 32 stream bits starting at bit `off` of an MSB-first packed bitstring
// (bit 31 of the result = stream bit off); reads two 32-bit words, the second
// only if it exists.
__device__ __forceinline__ uint32_t stream32(const uint8_t *__restrict__ b, int nbytes, int off) {
  const int W = off >> 5, sh = off & 31;
  auto be = [&](int w) -> uint32_t {
    const int o = 4 * w;
    if (o + 4 <= nbytes) {
      uint32_t v;
      memcpy(&v, b + o, 4);  // rows of `bits` are nbytes apart: not always 4-byte aligned
      return __byte_perm(v, 0u, 0x0123);
    }
    uint32_t v = 0;
    for (int i = 0; i < 4; i++)
      if (o + i < nbytes) v |= (uint32_t)b[o + i] << (24 - 8 * i);
    return v;
  };
  const uint32_t hi = be(W);
  return sh ? __funnelshift_l(be(W + 1), hi, sh) : hi;
}

// K1, the bit-sliced evaluator: one thread per (row, 32-column
// chunk); the chunk's coupling sign planes are built once and reused for
// every trial of the slab blockIdx.y covers.  Per trial and chunk: three
// 32-bit windows of the MSB-first bitstring (the sites, their right and their
// down neighbours) and four popcounts.  cut = sum over edges with differing
// spins of w; energy = W - 2 cut (evaluate.py:10-12).  A chunk with a weight
// other than +-1 takes the per-site path (any int8 weights stay exact).
__global__ void __launch_bounds__(256)
    torus_cut_energy_kernel(int rows, int cols, int WPR, const int8_t *__restrict__ w,
                            const uint8_t *__restrict__ bits, int nbytes, int T, int slab,
                            unsigned long long *cut, unsigned long long *energy) {
  __shared__ long long red[8];
  const int chunk = blockIdx.x * blockDim.x + threadIdx.x;
  const int nchunks = rows * WPR;
  const bool act = chunk < nchunks;
  const int r = act ? chunk / WPR : 0, k = act ? chunk - r * WPR : 0;
  const int c0 = 32 * k, vb = act ? min(32, cols - c0) : 0;
  const uint32_t valid = vb == 0 ? 0u : (vb == 32 ? ~0u : ~0u << (32 - vb));
  const int rd = r + 1 == rows ? 0 : r + 1;
  // sign planes, MSB-first like the stream: bit 31 - b = site (r, c0 + b)
  uint32_t negR = 0, negD = 0;
  bool unit = true;
  long long wsum = 0;
  for (int b = 0; b < vb; b++) {
    const int x = r * cols + c0 + b;
    const int wr = w[2 * x], wd = w[2 * x + 1];
    negR |= (uint32_t)(wr < 0) << (31 - b);
    negD |= (uint32_t)(wd < 0) << (31 - b);
    unit = unit && (wr == 1 || wr == -1) && (wd == 1 || wd == -1);
    wsum += wr + wd;
  }
  const bool wraps = act && c0 + vb == cols;  // the chunk holds the row's last column
  const int t0 = blockIdx.y * slab, t1 = min(T, t0 + slab);
  for (int t = t0; t < t1; t++) {
    const uint8_t *bt = bits + (size_t)t * nbytes;
    long long c = 0;
    if (act) {
      const int off = r * cols + c0;
      const uint32_t X = stream32(bt, nbytes, off);
      uint32_t R = stream32(bt, nbytes, off + 1);
      if (wraps) {  // right neighbour of the last column is column 0 of the row
        const uint32_t first = stream32(bt, nbytes, r * cols) >> 31;
        const int pos = 32 - vb;  // bit of the last valid column
        R = (R & ~(1u << pos)) | (first << pos);
      }
      const uint32_t D = stream32(bt, nbytes, rd * cols + c0);
      if (unit) {
        const uint32_t xr = (X ^ R) & valid, xd = (X ^ D) & valid;
        c = __popc(xr & ~negR) - __popc(xr & negR) + __popc(xd & ~negD) - __popc(xd & negD);
      } else {
        for (int b = 0; b < vb; b++) {
          const int x = r * cols + c0 + b;
          const uint32_t m = 1u << (31 - b);
          if ((X ^ R) & m) c += w[2 * x];
          if ((X ^ D) & m) c += w[2 * x + 1];
        }
      }
    }
    long long ws = wsum;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      c += __shfl_xor_sync(0xffffffffu, c, o);
      ws += __shfl_xor_sync(0xffffffffu, ws, o);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // energy = W - 2 cut: reduce c and (ws - 2c) over the block
    if (lane == 0) red[warp] = c;
    __syncthreads();
    long long cb = 0;
    if (threadIdx.x < 8) cb = red[threadIdx.x];
    __syncthreads();
    if (lane == 0) red[warp] = ws;
    __syncthreads();
    long long wb = 0;
    if (threadIdx.x < 8) wb = red[threadIdx.x];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        cb += __shfl_xor_sync(0xffffffffu, cb, o);
        wb += __shfl_xor_sync(0xffffffffu, wb, o);
      }
      if (lane == 0) {
        atomicAdd(cut + t, (unsigned long long)cb);
        atomicAdd(energy + t, (unsigned long long)(wb - 2 * cb));
      }
    }
  }
}

__global__ void graph_cut_energy_kernel(int64_t m, const int32_t *__restrict__ eu,
                                        const int32_t *__restrict__ ev,
                                        const int32_t *__restrict__ ew,
                                        const uint8_t *__restrict__ bits, int nbytes,
                                        unsigned long long *cut, unsigned long long *energy) {
  const uint8_t *b = bits + (size_t)blockIdx.y * nbytes;
  long long c = 0, e = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x) {
    int su = get_bit(b, eu[k]), sv = get_bit(b, ev[k]);
    long long wk = ew[k];
    if (su != sv) c += wk;
    e += (su == sv) ? wk : -wk;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    c += __shfl_xor_sync(0xffffffffu, c, o);
    e += __shfl_xor_sync(0xffffffffu, e, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(cut + blockIdx.y, (unsigned long long)c);
    atomicAdd(energy + blockIdx.y, (unsigned long long)e);
  }
}

int torus_cut_energy(int rows, int cols, const int8_t *w, const uint8_t *bits, int T,
                     int64_t *cut, int64_t *energy, cudaStream_t stream) {
  if (T <= 0) return GSB_OK;
  int n = rows * cols;
  if (cudaMemsetAsync(cut, 0, sizeof(int64_t) * T, stream) != cudaSuccess ||
      cudaMemsetAsync(energy, 0, sizeof(int64_t) * T, stream) != cudaSuccess)
    return set_error(GSB_ECUDA, "memset failed");
  const int WPR = (cols + 31) / 32;
  const int bx = (rows * WPR + 255) / 256;
  // trials per block: enough blocks to fill the SMs, slabs as long as that allows
  // (a thread builds its chunk's sign planes once per slab)
  int slabs = (2 * num_sms() + bx - 1) / bx;
  if (slabs < 1) slabs = 1;
  if (slabs > T) slabs = T;
  if (slabs > 65535) slabs = 65535;
  const int slab = (T + slabs - 1) / slabs;
  dim3 grid(bx, (T + slab - 1) / slab);
  torus_cut_energy_kernel<<<grid, 256, 0, stream>>>(rows, cols, WPR, w, bits, (n + 7) / 8, T, slab,
                                                    (unsigned long long *)cut,
                                                    (unsigned long long *)energy);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GSB_OK : set_error(GSB_ECUDA, cudaGetErrorString(e));
}

int graph_cut_energy(const gsb_graph *g, const uint8_t *bits, int T, int64_t *cut,
                     int64_t *energy, cudaStream_t stream) {
  if (T <= 0) return GSB_OK;
  if (cudaMemsetAsync(cut, 0, sizeof(int64_t) * T, stream) != cudaSuccess ||
      cudaMemsetAsync(energy, 0, sizeof(int64_t) * T, stream) != cudaSuccess)
    return set_error(GSB_ECUDA, "memset failed");
  int64_t bx = (g->m + 255) / 256;
  if (bx > 1024) bx = 1024;
  if (bx < 1) bx = 1;
  dim3 grid((unsigned)bx, T);
  graph_cut_energy_kernel<<<grid, 256, 0, stream>>>(g->m, g->eu_dev, g->ev_dev, g->ew_dev, bits,
                                                    (g->n + 7) / 8, (unsigned long long *)cut,
                                                    (unsigned long long *)energy);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GSB_OK : set_error(GSB_ECUDA, cudaGetErrorString(e));
}

// weight k = 2*bit31(next32 #k) - 1; next32 #k is the low (k even) or high
// (k odd) half of PCG64 output k>>1.  Thread i owns outputs [i*L, (i+1)*L).
__global__ void torus_weights_kernel(u128 s0, u128 inc, int64_t nout, int64_t L,
                                     int8_t *__restrict__ w) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t first = i * L;
  if (first >= nout) return;
  u128 A, C;
  pcg_jump_coeffs((uint64_t)first, inc, A, C);
  u128 s = A * s0 + C;
  int64_t last = first + L < nout ? first + L : nout;
  const u128 M = pcg_mult();
  for (int64_t o = first; o < last; o++) {
    s = s * M + inc;
    uint64_t x = pcg_out(s);
    w[2 * o] = (x >> 31) & 1 ? 1 : -1;
    w[2 * o + 1] = (x >> 63) ? 1 : -1;
  }
}

int torus_weights(int rows, int cols, uint64_t seed, int8_t *w, cudaStream_t stream) {
  u128 s0, inc;
  pcg_seed(seed, s0, inc);
  int64_t n = (int64_t)rows * cols;
  int64_t nout = n;  // 2n weights = n outputs
  int64_t L = 64;
  int64_t threads = (nout + L - 1) / L;
  int64_t blocks = (threads + 255) / 256;
  torus_weights_kernel<<<(unsigned)blocks, 256, 0, stream>>>(s0, inc, nout, L, w);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GSB_OK : set_error(GSB_ECUDA, cudaGetErrorString(e));
}

__global__ void best_key_kernel(const int64_t *cut, int T, int64_t first, int64_t *key) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < T) {
    uint64_t idx = (uint64_t)(first + t);
    key[t] = (int64_t)(((uint64_t)cut[t] << 32) | (0xFFFFFFFFull - (idx & 0xFFFFFFFFull)));
  }
}

int best_key(const int64_t *best_cut, int T, int64_t first, int64_t *key, cudaStream_t stream) {
  if (T <= 0) return GSB_OK;
  best_key_kernel<<<(T + 255) / 256, 256, 0, stream>>>(best_cut, T, first, key);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GSB_OK : set_error(GSB_ECUDA, cudaGetErrorString(e));
}

// Philox4x32-10 throughput microbenchmark: every thread evaluates
// `blocks_per_thread` independent blocks (2 streams interleaved for ILP: the
// fastest mix in tools/philox_mb.cu) and XOR-folds the outputs.
// Grid = SMs x 8 CTAs x 256 threads.
__global__ void __launch_bounds__(256) philox_bench_kernel(int64_t n, uint32_t *sink) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t k0 = 0x12345678u ^ blockIdx.x, k1 = 0x9abcdef0u;  // uniform key, as in a trial
  uint32_t acc = 0;
  const int iters = (int)(n / 2);
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int q = 0; q < 2; q++) {
      const P4 r = philox10(P4{tid, (uint32_t)i, (uint32_t)q, 1u}, k0, k1);
      acc ^= r.x ^ r.y ^ r.z ^ r.w;
    }
  }
  if (acc == 0x8badf00du) sink[tid & 255] = acc;  // keep the work alive
}

int philox_bench_threads() { return num_sms() * 8 * 256; }

// ALU-pipe probe: 8 independent LOP3 chains per thread (3-input boolean
// functions, the instruction the bit-sliced sweep kernels are made of);
// n = LOP3 per thread.  SMs x 8 x 256 threads, as the Philox probe.
__global__ void __launch_bounds__(256) lop3_bench_kernel(int64_t n, uint32_t *sink) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t a0 = tid, a1 = tid * 3u + 1u, a2 = tid ^ 0x5bd1e995u, a3 = ~tid, a4 = tid + 77u,
           a5 = tid * 7u, a6 = tid ^ 0xdeadbeefu, a7 = tid - 13u;
  const uint32_t m = 0x9e3779b9u ^ blockIdx.x, k = 0x85ebca6bu + threadIdx.x;
  const int iters = (int)(n / 32);
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int r = 0; r < 4; r++) {
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a0) : "r"(m), "r"(a1));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0xE8;" : "+r"(a1) : "r"(k), "r"(a2));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x69;" : "+r"(a2) : "r"(m), "r"(a3));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0xCA;" : "+r"(a3) : "r"(k), "r"(a4));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x8E;" : "+r"(a4) : "r"(m), "r"(a5));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0xBE;" : "+r"(a5) : "r"(k), "r"(a6));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0xB4;" : "+r"(a6) : "r"(m), "r"(a7));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0xD8;" : "+r"(a7) : "r"(k), "r"(a0));
    }
  }
  const uint32_t acc = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
  if (acc == 0x8badf00du) sink[tid & 255] = acc;  // keep the work alive
}

int lop3_bench(int64_t lop3_per_thread, uint32_t *sink, cudaStream_t stream) {
  const int nsm = num_sms();
  if (nsm <= 0) return set_error(GSB_ECUDA, "no CUDA device");
  lop3_bench_kernel<<<nsm * 8, 256, 0, stream>>>(lop3_per_thread, sink);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GSB_OK : set_error(GSB_ECUDA, cudaGetErrorString(e));
}

int philox_bench(int64_t blocks_per_thread, uint32_t *sink, cudaStream_t stream) {
  const int nsm = num_sms();
  if (nsm <= 0) return set_error(GSB_ECUDA, "no CUDA device");
  philox_bench_kernel<<<nsm * 8, 256, 0, stream>>>(blocks_per_thread, sink);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GSB_OK : set_error(GSB_ECUDA, cudaGetErrorString(e));
}

}  // namespace gsb
