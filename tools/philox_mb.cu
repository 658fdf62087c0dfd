// philox_mb.cu -- micro-benchmark (development tool): Philox4x32-10 block rate
// with the 32x32->64 products issued as IMAD.WIDE vs split IMAD.HI + IMAD.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/philox_mb tools/philox_mb.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct P4 { uint32_t x, y, z, w; };

template <int MODE>
__device__ __forceinline__ void mw(uint32_t a, uint32_t b, uint32_t breg, uint32_t &hi, uint32_t &lo) {
  if (MODE == 0) {
    hi = __umulhi(a, b);
    lo = a * b;
  } else if (MODE == 1) {
    asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(hi) : "r"(a), "r"(b));
    asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(lo) : "r"(a), "r"(breg));
  } else {
    // hi from IMAD.HI, lo from the product's low word via IMAD with a register copy
    hi = __umulhi(a, b);
    lo = a * breg;
  }
}

template <int MODE>
__device__ __forceinline__ P4 philox(P4 c, uint32_t k0, uint32_t k1, uint32_t m0r, uint32_t m1r) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    uint32_t hi0, lo0, hi1, lo1;
    mw<MODE>(c.x, 0xD2511F53u, m0r, hi0, lo0);
    mw<MODE>(c.z, 0xCD9E8D57u, m1r, hi1, lo1);
    P4 n{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    c = n;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

template <int MODE, int ILP>
__global__ void bench(int iters, uint32_t m0r, uint32_t m1r, uint32_t *out) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  const uint32_t k0 = 0x1234567u ^ blockIdx.x, k1 = 0x89abcdefu;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < ILP; u++) {
      P4 o = philox<MODE>(P4{tid, (uint32_t)i, (uint32_t)u, 1u}, k0, k1, m0r, m1r);
      acc ^= o.x ^ o.y ^ o.z ^ o.w;
    }
  }
  if (acc == 0x9u) out[0] = tid;
}

template <int MODE, int ILP>
void run(const char *name, int blocks, int threads, int iters) {
  uint32_t *out;
  cudaMalloc(&out, 4);
  bench<MODE, ILP><<<blocks, threads>>>(iters, 0xD2511F53u, 0xCD9E8D57u, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  bench<MODE, ILP><<<blocks, threads>>>(iters, 0xD2511F53u, 0xCD9E8D57u, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double nb = (double)blocks * threads * iters * ILP;
  printf("%-28s blocks=%d thr=%d ilp=%d: %.3e Philox blocks/s\n", name, blocks, threads, ILP,
         nb / (ms * 1e-3));
  cudaFree(out);
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int occ : {4, 8, 16}) {
    run<0, 2>("IMAD.WIDE", nsm * occ, 256, 2000);
    run<1, 2>("asm mul.hi + mul.lo", nsm * occ, 256, 2000);
    run<2, 2>("umulhi + mul(reg)", nsm * occ, 256, 2000);
    run<0, 4>("IMAD.WIDE", nsm * occ, 256, 1000);
    run<2, 4>("umulhi + mul(reg)", nsm * occ, 256, 1000);
  }
  return 0;
}
