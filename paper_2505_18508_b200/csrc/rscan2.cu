// rscan2.cu -- random-scan engine (kinds *_random_scan): host side.
//
// Team shape selection and launch of rscan2_kernel<NW, RB, SA>
// (rscan2_kernel.cuh has the algorithm; rscan2_nw{1,2,4,7,8,9,13}.cu the
// instantiations).  NW warps per trial in {1, 2, 4, 7, 8}, RB rows per lane in
// {1, 2, 3, 4, 5, 7}: a torus fits when rows <= NW * floor(32 / WPR) * RB for
// some shape, WPR = ceil(cols / 32) <= 32; teams of 9 and 13 warps with
// two rows per lane add occupancy for 100-row tori of 5 and 7 words per row
// (configs 3 and 4), never reach.
#include <cuda_runtime.h>

#include <mutex>

#include "rscan2_kernel.cuh"

namespace gsb {

struct Rs2Shape {
  int NW, RB, NBu, nbig, per_sm;
};

static const int kRbSet[] = {1, 2, 3, 4, 5, 7};
static const int kNwSet[] = {1, 2, 4, 7, 8, 9, 13};

static const void *rs2_kernel(int nw, int rb, bool sa) {
  switch (nw) {
    case 1:
      return rs2_kernel_nw1(rb, sa);
    case 2:
      return rs2_kernel_nw2(rb, sa);
    case 4:
      return rs2_kernel_nw4(rb, sa);
    case 7:
      return rs2_kernel_nw7(rb, sa);
    case 8:
      return rs2_kernel_nw8(rb, sa);
    case 9:
      return rs2_kernel_nw9(rb, sa);
    case 13:
      return rs2_kernel_nw13(rb, sa);
    default:
      return nullptr;
  }
}

// tie queue capacity: ties per sweep ~ n / 64 (4 comparisons of 2^-8 per site)
static int rs2_tqcap(int n) {
  int cap = n / 32;
  return cap < 128 ? 128 : cap;
}

// row-block counts with blocks of RB or RB - 1 rows
static bool rs2_blocks(int rows, int RB, int maxblocks, int &NBu, int &nbig) {
  for (int nb = (rows + RB - 1) / RB; nb <= maxblocks; nb++) {
    if (RB == 1) {
      if (nb == rows) {
        NBu = nb;
        nbig = nb;
        return true;
      }
      continue;
    }
    const int big = rows - nb * (RB - 1);  // blocks with RB rows
    if (big >= 1 && big <= nb) {
      NBu = nb;
      nbig = big;
      return true;
    }
    if (big < 1) break;
  }
  return false;
}

// resident CTAs per SM of an instantiation at a dynamic shared memory size
// (cached; -1 = does not fit)
static int rs2_occupancy(int nw, int rb, bool sa, size_t smem) {
  static std::mutex mu;
  struct Key {
    int dev, nw, rb, sa;
    size_t smem;
    int occ;
  };
  static Key cache[512];
  static int ncache = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  const void *kern = rs2_kernel(nw, rb, sa);
  if (!kern) return -1;
  // every call: the limit may have to rise for this size (allow_dynamic_smem)
  if (allow_dynamic_smem(kern, smem) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  std::lock_guard<std::mutex> lk(mu);
  for (int i = 0; i < ncache; i++)
    if (cache[i].dev == dev && cache[i].nw == nw && cache[i].rb == rb && cache[i].sa == (int)sa &&
        cache[i].smem == smem)
      return cache[i].occ;
  int occ = -1, per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, smem) == cudaSuccess &&
      per_sm >= 1)
    occ = per_sm;
  cudaGetLastError();
  if (ncache < 512) cache[ncache++] = Key{dev, nw, rb, (int)sa, smem, occ};
  return occ;
}

// test-only overrides (gsb_test_rscan_shape, gsb_test_rscan_limits)
static int g_force_nw = 0, g_force_rb = 0, g_test_tqcap = 0, g_test_lcap = 0, g_force_slices = 0;

void rscan2_force_shape(int nw, int rb) {
  g_force_nw = nw;
  g_force_rb = rb;
}

void rscan2_force_slices(int nslice) { g_force_slices = nslice; }

void rscan2_test_limits(int tqcap, int lcap) {
  g_test_tqcap = tqcap;
  g_test_lcap = lcap > RS2_CAP ? RS2_CAP : lcap;
}

// Team shape for T trials.  Cost model (arbitrary units, fitted to B200 runs
// of configs 1-4): with w = k * NW warps resident per SM the SM's throughput
// saturates like w / (w + 12), so a wave of k resident trials per SM takes
//   RB * (k * NW + 12) * (1 + 0.03 log2 NW)
// (work k * NW * RB over that throughput; a small barrier cost per extra
// warp), summed over the waves the occupancy allows.  `occupancy` false (no
// device): only feasibility, first fit.
static bool rs2_shape(int rows, int cols, int T, int nsm, bool sa, bool occupancy, Rs2Shape &sh) {
  const int WPR = (cols + 31) / 32;
  if (WPR > 32 || rows * WPR > 2048) return false;  // tie items carry 11-bit word indices
  const int BPW = 32 / WPR;
  const int n = rows * cols, nstream = (n + 31) / 32, tqcap = rs2_tqcap(n);
  bool found = false;
  double bestcost = 0;
  for (int nw : kNwSet) {
    for (int RB : kRbSet) {
      if (occupancy && g_force_nw > 0 && (nw != g_force_nw || RB != g_force_rb)) continue;
      if (nw > 8 && (RB != 2 || !occupancy)) continue;  // wide teams: two rows per lane only
      int NBu, nbig;
      if (!rs2_blocks(rows, RB, nw * BPW, NBu, nbig)) continue;
      if (!occupancy) {
        sh = Rs2Shape{nw, RB, NBu, nbig, 1};
        return true;
      }
      const int per_sm = rs2_occupancy(nw, RB, sa, rs2_smem_bytes(nw, RB, tqcap, nstream));
      if (per_sm < 1) continue;
      const long long tps = ((long long)T + nsm - 1) / nsm;  // trials per SM
      const long long full = tps / per_sm, rem = tps % per_sm;
      const double bar =
          1.0 + 0.03 * (nw == 1 ? 0 : nw == 2 ? 1 : nw == 4 ? 2 : nw <= 9 ? 3 : 3.7);  // ~log2 NW
      auto wave = [&](long long k) { return (double)RB * ((double)k * nw + 12.0) * bar; };
      const double cost = (double)full * wave(per_sm) + (rem ? wave(rem) : 0.0);
      if (!found || cost < bestcost - 1e-9) {
        found = true;
        bestcost = cost;
        sh = Rs2Shape{nw, RB, NBu, nbig, per_sm};
      }
    }
  }
  return found;
}

// Sweep slices for an annealing launch of T trials on `grid` resident teams
// (Rs2Args::nslice).  Unsliced, team b runs trials b, b + grid, ...: the launch
// ends on a part-filled wave (config 2: 1024 trials on 444 seats = 2.31 waves,
// run as 3) and on the teams whose trials happened to need the most
// best-so-far work.  Cut into slices drawn from a counter, the seats stay full
// until the work runs out.  Measured on B200 (tools/slices_ab.py): config 2
// +18 %, configs 3 / 4 (2000 / 1000 sweeps) +10 % / +8 %, flat from ~13 slices
// up to slices of 8 sweeps.
static int rs2_slices(int T, int nsm, const Rs2Shape &sh, int sweeps, bool sa) {
  if (!sa) return 1;  // greedy trials stop early; nothing to balance
  if (g_force_slices > 0) return g_force_slices > sweeps ? sweeps : g_force_slices;
  if ((long long)T <= (long long)nsm * sh.per_sm) return 1;  // a seat per trial
  const int c = sweeps / 32;
  return c < 1 ? 1 : c > 16 ? 16 : c;
}

size_t rscan2_workspace_bytes(int rows, int cols, int T) {
  const size_t WPR = (size_t)(cols + 31) / 32;
  const size_t flags = ((size_t)T * 4 + 15) & ~(size_t)15;
  return flags + (size_t)T * 4 * (4 + 2 * (size_t)rows * WPR);
}

bool rscan2_fits(int rows, int cols) {
  Rs2Shape sh;
  if (rows < 3 || cols < 3) return false;
  return rs2_shape(rows, cols, 1, 148, true, false, sh);
}

bool rscan2_shape(int rows, int cols, int T, int *nw, int *rb) {
  Rs2Shape sh;
  if (rows < 3 || cols < 3 || T < 1 || !rs2_shape(rows, cols, T, num_sms(), true, true, sh))
    return false;
  *nw = sh.NW;
  *rb = sh.RB;
  return true;
}

int rscan2_run(int rows, int cols, const int8_t *w_dev, int kind, int sweeps,
               const uint64_t *table, const uint64_t *seeds, int T, int64_t *best_cut,
               int32_t *sweeps_exec, uint8_t *best_bits, void *ws, int *err_ws,
               unsigned long long *stats, cudaStream_t stream) {
  Rs2Shape sh;
  const bool sa = kind == GSB_ANNEALING;
  const int nsm = num_sms();
  if (nsm < 1) return set_error(GSB_ECUDA, "no CUDA device");
  if (rows < 3 || cols < 3 || !rs2_shape(rows, cols, T, nsm, sa, true, sh))
    return set_error(GSB_EUNSUPPORTED, "torus too large for the random-scan engine");
  Rs2Args a;
  a.rows = rows;
  a.cols = cols;
  a.n = rows * cols;
  a.WPR = (cols + 31) / 32;
  a.NBu = sh.NBu;
  a.nbig = sh.nbig;
  a.lastvalid = cols - 32 * (a.WPR - 1);
  a.w = w_dev;
  a.table = table;
  a.sweeps = sweeps;
  a.seeds = seeds;
  a.T = T;
  a.best_cut = best_cut;
  a.sweeps_exec = sweeps_exec;
  a.best_bits = best_bits;
  a.nbytes = (a.n + 7) / 8;
  a.nstream = (a.n + 31) / 32;
  a.tqcap = rs2_tqcap(a.n);
  a.lcap = RS2_CAP;
  if (g_test_tqcap > 0 && g_test_tqcap < a.tqcap) a.tqcap = g_test_tqcap;  // smem sized for the default
  if (g_test_lcap > 0) a.lcap = g_test_lcap;
  a.m_one = 1u;
  a.m_two = 2u;
  a.m_neg = 0xFFFFFFFFu;
  a.m_last = 1u << (a.lastvalid - 1);
  a.err = err_ws;
  a.stats = stats;
  // sweep slices: work counter in the zeroed error block (after the counters),
  // flags and parked states in the workspace
  a.nslice = rs2_slices(T, nsm, sh, sweeps, sa);
  a.slice_len = (sweeps + a.nslice - 1) / a.nslice;
  a.nslice = (sweeps + a.slice_len - 1) / a.slice_len;
  a.dynamic = a.nslice > 1 || (long long)T > (long long)nsm * sh.per_sm;
  a.sl_shift = 0;
  while ((1LL << a.sl_shift) < T) a.sl_shift++;
  a.sl_ctr = (uint32_t *)((char *)err_ws + 96);
  a.sl_flag = (uint32_t *)ws;
  a.sl_state = (uint32_t *)((char *)ws + (((size_t)T * 4 + 15) & ~(size_t)15));
  if (a.nslice > 1 &&
      cudaMemsetAsync(a.sl_flag, 0, (size_t)T * 4, stream) != cudaSuccess)
    return set_error(GSB_ECUDA, "memset failed");
  const size_t smem = rs2_smem_bytes(sh.NW, sh.RB, rs2_tqcap(a.n), a.nstream);
  const void *kern = rs2_kernel(sh.NW, sh.RB, sa);
  if (!kern) return set_error(GSB_EUNSUPPORTED, "no random-scan kernel for this team shape");
  long long grid = (long long)nsm * sh.per_sm;
  if (grid > T) grid = T;
  void *params[] = {&a};
  const cudaError_t e = cudaLaunchKernel(kern, dim3((unsigned)grid), dim3((unsigned)(sh.NW * 32)),
                                         params, smem, stream);
  if (e != cudaSuccess) return set_error(GSB_ECUDA, cudaGetErrorString(e));
  return GSB_OK;
}

}  // namespace gsb
