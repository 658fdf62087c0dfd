// abi.cu -- the C ABI of libgsb_cuda.so (include/gsb.h).
//
// Host-side glue only: argument validation (mirrors SolverConfig.__post_init__,
// solvers.py:43-59, and TorusSpec, instances.py:190-196), schedule tables
// (solvers.py:84-88, :118), workspace carving and kernel dispatch.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "gsb_internal.h"

namespace gsb {

static thread_local std::string g_err;

int set_error(int code, const char *msg) {
  g_err = msg ? msg : "";
  return code;
}

int num_sms() {
  static std::mutex mu;
  static std::vector<int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  std::lock_guard<std::mutex> lk(mu);
  if ((int)cache.size() <= dev) cache.resize(dev + 1, 0);
  if (cache[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    cache[dev] = v;
  }
  return cache[dev];
}

cudaError_t allow_dynamic_smem(const void *kern, size_t bytes) {
  struct Entry {
    int dev;
    const void *kern;
    size_t max_bytes;
  };
  static std::mutex mu;
  static std::vector<Entry> seen;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  Entry *hit = nullptr;
  for (auto &en : seen)
    if (en.dev == dev && en.kern == kern) hit = &en;
  if (hit && hit->max_bytes >= bytes) return cudaSuccess;
  if (bytes > 48 * 1024 || hit) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
  }
  if (hit)
    hit->max_bytes = bytes;
  else
    seen.push_back(Entry{dev, kern, bytes});
  return cudaSuccess;
}

static bool torus_ok(const gsb_torus *t) {
  return t && t->rows >= 3 && t->cols >= 3 && t->w_dev &&
         (int64_t)t->rows * t->cols < (int64_t)1 << 30;
}

static size_t err_bytes() { return 256; }

// Stream-ordered pool for the host-buffer entry point: keeps its reservation
// between calls (release threshold = max) so repeated calls do not remap
// device memory.  One pool per device, created on first use.
static cudaError_t pool_alloc(void **p, size_t bytes, cudaStream_t stream) {
  static std::mutex mu;
  static std::vector<cudaMemPool_t> pools;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lk(mu);
    if ((int)pools.size() <= dev) pools.resize(dev + 1, nullptr);
    if (!pools[dev]) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      e = cudaMemPoolCreate(&pools[dev], &props);
      if (e != cudaSuccess) return e;
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pool = pools[dev];
  }
  return cudaMallocFromPoolAsync(p, bytes, pool, stream);
}

}  // namespace gsb

using namespace gsb;

extern "C" {

const char *gsb_last_error(void) { return g_err.c_str(); }

int gsb_abi_version(void) { return GSB_ABI_VERSION; }

int gsb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int gsb_mix_seeds(uint64_t master, int64_t first, int32_t T, uint64_t *out) {
  if (first < 0 || T < 0 || (!out && T > 0)) return set_error(GSB_EINVAL, "bad arguments");
  for (int32_t t = 0; t < T; t++) {  // campaign.py:50-53
    uint64_t z = master + (uint64_t)(first + t + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    out[t] = z ^ (z >> 31);
  }
  return GSB_OK;
}

int gsb_torus_weights(int32_t rows, int32_t cols, uint64_t seed, int8_t *w_dev, void *stream) {
  if (rows < 3 || cols < 3 || !w_dev)
    return set_error(GSB_EINVAL, "torus must be at least 3x3");
  return torus_weights(rows, cols, seed, w_dev, (cudaStream_t)stream);
}

int gsb_torus_cut_energy(const gsb_torus *inst, const uint8_t *bits, int32_t T, int64_t *cut,
                         int64_t *energy, void *stream) {
  if (!torus_ok(inst) || T < 0 || (T > 0 && (!bits || !cut || !energy)))
    return set_error(GSB_EINVAL, "bad arguments");
  return torus_cut_energy(inst->rows, inst->cols, inst->w_dev, bits, T, cut, energy,
                          (cudaStream_t)stream);
}

int gsb_graph_cut_energy(const gsb_graph *g, const uint8_t *bits, int32_t T, int64_t *cut,
                         int64_t *energy, void *stream) {
  if (!g || g->n < 1 || g->m < 0 || T < 0 || (T > 0 && (!bits || !cut || !energy)))
    return set_error(GSB_EINVAL, "bad arguments");
  return graph_cut_energy(g, bits, T, cut, energy, (cudaStream_t)stream);
}

int gsb_schedule_table(int engine, int32_t sweeps, double t0, double t1, int32_t dmax,
                       uint64_t *table) {
  if (sweeps < 1 || dmax < 1 || !table) return set_error(GSB_EINVAL, "bad arguments");
  if (!(0.0 < t1 && t1 < t0)) return set_error(GSB_EINVAL, "need 0 < temp_end < temp_start");
  int bits;
  if (engine == GSB_ENGINE_REFERENCE)
    bits = 53;
  else if (engine == GSB_ENGINE_CHECKERBOARD || engine == GSB_ENGINE_CHECKERBOARD_TILED ||
           engine == GSB_ENGINE_CHECKERBOARD_CLUSTER || engine == GSB_ENGINE_RANDOM_SCAN ||
           engine == GSB_ENGINE_RANDOM_SCAN_LARGE)
    bits = 32;
  else
    return set_error(GSB_EINVAL, "unknown engine");
  for (int32_t t = 0; t < sweeps; t++) {
    // solvers.py:84-88 (Python float ops are these libm calls)
    double temp = sweeps == 1 ? t0 : t0 * std::pow(t1 / t0, (double)t / (double)(sweeps - 1));
    for (int32_t d = 1; d <= dmax; d++) {
      double p = std::exp((double)(-d) / temp);  // math.exp(delta / temp), solvers.py:118
      double x = std::ceil(std::ldexp(p, bits));
      table[(size_t)t * dmax + (d - 1)] = (uint64_t)x;
    }
  }
  return GSB_OK;
}

size_t gsb_torus_workspace_bytes(const gsb_torus *inst, int engine, int32_t sweeps, int32_t T) {
  (void)sweeps;
  if (!inst) return 0;
  int n = inst->rows * inst->cols;
  size_t b = err_bytes();
  if (engine == GSB_ENGINE_RANDOM_SCAN || engine == GSB_ENGINE_RANDOM_SCAN_LARGE) {
    // rscan2 parks trials between sweep slices; the large-torus engine keeps the
    // planes of up to 8 trials in the workspace
    if (engine == GSB_ENGINE_RANDOM_SCAN_LARGE || !rscan2_fits(inst->rows, inst->cols))
      b += rscan_big_workspace_bytes(inst->rows, inst->cols, T);
    else
      b += rscan2_workspace_bytes(inst->rows, inst->cols, T);
  } else if (engine == GSB_ENGINE_CHECKERBOARD && checker_fits(inst->rows, inst->cols)) {
    b += checker_workspace_bytes(inst->rows, inst->cols);
  } else if ((engine == GSB_ENGINE_CHECKERBOARD || engine == GSB_ENGINE_CHECKERBOARD_CLUSTER) &&
             checker_cluster_fits(inst->rows, inst->cols)) {
    b += checker_cluster_workspace_bytes(inst->rows, inst->cols);
  } else if (engine == GSB_ENGINE_CHECKERBOARD || engine == GSB_ENGINE_CHECKERBOARD_TILED ||
             engine == GSB_ENGINE_CHECKERBOARD_CLUSTER) {
    b += checker_hbm_workspace_bytes(inst->rows, inst->cols, T, num_sms());
  } else {
    b += ref_workspace_bytes(n, 0, T);
  }
  return b;
}

static int finish_check(int *err_dev, cudaStream_t stream) {
  int h = 0;
  if (cudaMemcpyAsync(&h, err_dev, sizeof(int), cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
      cudaStreamSynchronize(stream) != cudaSuccess)
    return set_error(GSB_ECUDA, cudaGetErrorString(cudaGetLastError()));
  if (h == GSB_EINTEGRITY)
    return set_error(GSB_EINTEGRITY, "internal cut accounting drifted from recomputation");
  if (h != 0) return set_error(h, "device error");
  return GSB_OK;
}

int gsb_torus_sweep(const gsb_torus *inst, int engine, int kind, int32_t sweeps,
                    const uint64_t *table, const uint64_t *seeds, int32_t T, int64_t *best_cut,
                    int32_t *sweeps_exec, uint8_t *best_bits, void *ws, size_t ws_bytes,
                    void *stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!torus_ok(inst)) return set_error(GSB_EINVAL, "torus must be at least 3x3");
  if (kind != GSB_GREEDY && kind != GSB_ANNEALING) return set_error(GSB_EINVAL, "unknown kind");
  if (sweeps < 1) return set_error(GSB_EINVAL, "sweeps must be positive");
  if (T < 0) return set_error(GSB_EINVAL, "T must be non-negative");
  if (T == 0) return GSB_OK;
  if (!seeds || !best_cut || !sweeps_exec || !best_bits || !ws)
    return set_error(GSB_EINVAL, "null buffer");
  if (kind == GSB_ANNEALING && !table) return set_error(GSB_EINVAL, "annealing needs a table");
  if (ws_bytes < gsb_torus_workspace_bytes(inst, engine, sweeps, T))
    return set_error(GSB_ENOMEM, "workspace too small");
  int *err = (int *)ws;
  char *rest = (char *)ws + err_bytes();
  size_t rest_bytes = ws_bytes - err_bytes();
  if (cudaMemsetAsync(err, 0, 128, stream) != cudaSuccess)
    return set_error(GSB_ECUDA, "memset failed");
  int rc;
  if (engine == GSB_ENGINE_CHECKERBOARD || engine == GSB_ENGINE_CHECKERBOARD_TILED ||
      engine == GSB_ENGINE_CHECKERBOARD_CLUSTER) {
    if ((inst->rows & 1) || (inst->cols & 1))
      return set_error(GSB_EUNSUPPORTED,
                       "checkerboard kinds need even torus dimensions (bipartite torus)");
    if (engine == GSB_ENGINE_CHECKERBOARD && checker_fits(inst->rows, inst->cols)) {
      rc = checker_run(inst->rows, inst->cols, inst->w_dev, kind, sweeps, table, seeds, T,
                       best_cut, sweeps_exec, best_bits, rest, err, stream);
    } else if (engine != GSB_ENGINE_CHECKERBOARD_TILED &&
               checker_cluster_fits(inst->rows, inst->cols)) {
      rc = checker_cluster_run(inst->rows, inst->cols, inst->w_dev, kind, sweeps, table, seeds, T,
                               best_cut, sweeps_exec, best_bits, rest, err, stream);
    } else if (engine != GSB_ENGINE_CHECKERBOARD_CLUSTER &&
               checker_hbm_fits(inst->rows, inst->cols)) {
      rc = checker_hbm_run(inst->rows, inst->cols, inst->w_dev, kind, sweeps, table, seeds, T,
                           best_cut, sweeps_exec, best_bits, rest, err, stream);
    } else {
      return set_error(GSB_EUNSUPPORTED, "torus too large for the checkerboard engines");
    }
  } else if (engine == GSB_ENGINE_RANDOM_SCAN && rscan2_fits(inst->rows, inst->cols)) {
    rc = rscan2_run(inst->rows, inst->cols, inst->w_dev, kind, sweeps, table, seeds, T, best_cut,
                    sweeps_exec, best_bits, rest, err, (unsigned long long *)((char *)err + 16),
                    stream);
  } else if (engine == GSB_ENGINE_RANDOM_SCAN || engine == GSB_ENGINE_RANDOM_SCAN_LARGE) {
    rc = rscan_big_run(inst->rows, inst->cols, inst->w_dev, kind, sweeps, table, seeds, T,
                       best_cut, sweeps_exec, best_bits, rest, err, stream);
  } else if (engine == GSB_ENGINE_REFERENCE && ref_warp_fits(inst->rows, inst->cols)) {
    rc = ref_warp_run(inst->rows, inst->cols, inst->w_dev, kind, sweeps, table, seeds, T, best_cut,
                      sweeps_exec, best_bits, rest, err, stream);
  } else if (engine == GSB_ENGINE_REFERENCE) {
    rc = ref_run_torus(inst->rows, inst->cols, inst->w_dev, kind, sweeps, table, 4, seeds, T,
                       best_cut, sweeps_exec, best_bits, rest, rest_bytes, err, stream);
  } else {
    return set_error(GSB_EINVAL, "unknown engine");
  }
  return rc;
}

int gsb_rscan_fits(int32_t rows, int32_t cols) {
  return rscan2_fits(rows, cols) ? 1 : rscan_big_fits(rows, cols) ? 2 : 0;
}

int gsb_rscan_shape(int32_t rows, int32_t cols, int32_t T, int32_t *warps, int32_t *rows_per_lane) {
  if (!warps || !rows_per_lane) return set_error(GSB_EINVAL, "null argument");
  int nw = 0, rb = 0;
  if (!rscan2_shape(rows, cols, T, &nw, &rb))
    return set_error(GSB_EUNSUPPORTED, "torus too large for the random-scan engine");
  *warps = nw;
  *rows_per_lane = rb;
  return GSB_OK;
}

int gsb_test_checker_shape(int32_t warps, int32_t variant) {
  if (!(warps == 0 || warps == 1 || warps == 2 || warps == 4 || warps == 8 || warps == 16) ||
      variant < 0 || variant > 2)
    return set_error(GSB_EINVAL, "bad checkerboard team shape");
  checker_force_shape(warps, variant);
  return GSB_OK;
}

int gsb_test_cluster_size(int32_t ctas) {
  if (ctas < 0 || ctas > 16 || (ctas & (ctas - 1))) return set_error(GSB_EINVAL, "bad cluster size");
  checker_cluster_force_size(ctas);
  return GSB_OK;
}

int gsb_test_rscan_shape(int32_t warps, int32_t rows_per_lane) {
  if ((warps == 0) != (rows_per_lane == 0) || warps < 0 || rows_per_lane < 0)
    return set_error(GSB_EINVAL, "bad team shape");
  rscan2_force_shape(warps, rows_per_lane);
  return GSB_OK;
}

int gsb_test_rscan_limits(int32_t tie_queue_cap, int32_t list_cap) {
  if (tie_queue_cap < 0 || list_cap < 0) return set_error(GSB_EINVAL, "bad limits");
  rscan2_test_limits(tie_queue_cap, list_cap);
  return GSB_OK;
}

int gsb_test_rscan_slices(int32_t slices) {
  if (slices < 0) return set_error(GSB_EINVAL, "bad slice count");
  rscan2_force_slices(slices);
  return GSB_OK;
}

int gsb_workspace_rscan_stats(const void *ws, void *stream, uint64_t *out4) {
  if (!ws || !out4) return set_error(GSB_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemcpyAsync(out4, (const char *)ws + 16, 32, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return set_error(GSB_ECUDA, cudaGetErrorString(cudaGetLastError()));
  return GSB_OK;
}

int gsb_workspace_counters(const void *ws, void *stream, uint64_t *philox_blocks) {
  if (!ws || !philox_blocks) return set_error(GSB_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemcpyAsync(philox_blocks, (const char *)ws + 8, 8, cudaMemcpyDeviceToHost, st) !=
          cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return set_error(GSB_ECUDA, cudaGetErrorString(cudaGetLastError()));
  return GSB_OK;
}

int gsb_philox_bench(int64_t blocks_per_thread, uint32_t *sink_dev, void *stream) {
  if (blocks_per_thread < 1 || !sink_dev) return set_error(GSB_EINVAL, "bad arguments");
  return philox_bench(blocks_per_thread, sink_dev, (cudaStream_t)stream);
}

int gsb_lop3_bench(int64_t lop3_per_thread, uint32_t *sink_dev, void *stream) {
  if (lop3_per_thread < 32 || !sink_dev) return set_error(GSB_EINVAL, "bad arguments");
  return lop3_bench(lop3_per_thread, sink_dev, (cudaStream_t)stream);
}

int gsb_workspace_status(const void *ws, void *stream) {
  if (!ws) return set_error(GSB_EINVAL, "null workspace");
  return finish_check((int *)ws, (cudaStream_t)stream);
}

size_t gsb_graph_workspace_bytes(const gsb_graph *g, int32_t sweeps, int32_t T) {
  (void)sweeps;
  if (!g) return 0;
  return err_bytes() + ref_workspace_bytes(g->n, g->m > 0 ? 2 * g->m : 1, T);
}

int gsb_graph_sweep(const gsb_graph *g, int kind, int32_t sweeps, const uint64_t *table,
                    int32_t dmax, const uint64_t *seeds, int32_t T, int64_t *best_cut,
                    int32_t *sweeps_exec, uint8_t *best_bits, void *ws, size_t ws_bytes,
                    void *stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!g || g->n < 1 || g->m < 0) return set_error(GSB_EINVAL, "bad graph");
  if (kind != GSB_GREEDY && kind != GSB_ANNEALING) return set_error(GSB_EINVAL, "unknown kind");
  if (sweeps < 1) return set_error(GSB_EINVAL, "sweeps must be positive");
  if (T <= 0) return T == 0 ? GSB_OK : set_error(GSB_EINVAL, "T must be non-negative");
  if (kind == GSB_ANNEALING && (!table || dmax < 1))
    return set_error(GSB_EINVAL, "annealing needs a table");
  if (ws_bytes < gsb_graph_workspace_bytes(g, sweeps, T))
    return set_error(GSB_ENOMEM, "workspace too small");
  int *err = (int *)ws;
  if (cudaMemsetAsync(err, 0, sizeof(int), stream) != cudaSuccess)
    return set_error(GSB_ECUDA, "memset failed");
  return ref_run_graph(g, kind, sweeps, table, dmax < 1 ? 1 : dmax, seeds, T, best_cut,
                       sweeps_exec, best_bits, (char *)ws + err_bytes(), ws_bytes - err_bytes(),
                       err, stream);
}

int gsb_torus_sweep_host(int32_t rows, int32_t cols, const int8_t *w_host, int engine, int kind,
                         int32_t sweeps, double t0, double t1, const uint64_t *seeds_host,
                         int32_t T, int64_t *best_cut_host, int32_t *sweeps_exec_host,
                         uint8_t *best_bits_host, void *stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (rows < 3 || cols < 3 || !w_host) return set_error(GSB_EINVAL, "torus must be at least 3x3");
  if (T < 0 || sweeps < 1) return set_error(GSB_EINVAL, "bad arguments");
  if (T == 0) return GSB_OK;
  const int n = rows * cols;
  const size_t nbytes = (size_t)(n + 7) / 8;
  std::vector<uint64_t> table;
  if (kind == GSB_ANNEALING) {
    table.resize((size_t)sweeps * 4);
    int rc = gsb_schedule_table(engine, sweeps, t0, t1, 4, table.data());
    if (rc) return rc;
  }
  int8_t *w = nullptr;
  uint64_t *tab = nullptr, *seeds = nullptr;
  int64_t *bc = nullptr;
  int32_t *se = nullptr;
  uint8_t *bits = nullptr;
  void *ws = nullptr;
  gsb_torus inst{rows, cols, nullptr};
  size_t wsb = gsb_torus_workspace_bytes(&inst, engine, sweeps, T);
  int rc = GSB_OK;
#define GSB_TRY(x)                                                   \
  do {                                                               \
    cudaError_t e_ = (x);                                            \
    if (e_ != cudaSuccess) {                                         \
      rc = set_error(GSB_ECUDA, cudaGetErrorString(e_));             \
      goto done;                                                     \
    }                                                                \
  } while (0)
  GSB_TRY(pool_alloc((void **)&w, (size_t)2 * n, stream));
  GSB_TRY(pool_alloc((void **)&seeds, sizeof(uint64_t) * T, stream));
  GSB_TRY(pool_alloc((void **)&bc, sizeof(int64_t) * T, stream));
  GSB_TRY(pool_alloc((void **)&se, sizeof(int32_t) * T, stream));
  GSB_TRY(pool_alloc((void **)&bits, nbytes * T, stream));
  GSB_TRY(pool_alloc(&ws, wsb, stream));
  if (!table.empty()) {
    GSB_TRY(pool_alloc((void **)&tab, sizeof(uint64_t) * table.size(), stream));
    GSB_TRY(cudaMemcpyAsync(tab, table.data(), sizeof(uint64_t) * table.size(),
                            cudaMemcpyHostToDevice, stream));
  }
  GSB_TRY(cudaMemcpyAsync(w, w_host, (size_t)2 * n, cudaMemcpyHostToDevice, stream));
  GSB_TRY(cudaMemcpyAsync(seeds, seeds_host, sizeof(uint64_t) * T, cudaMemcpyHostToDevice, stream));
  inst.w_dev = w;
  rc = gsb_torus_sweep(&inst, engine, kind, sweeps, tab, seeds, T, bc, se, bits, ws, wsb, stream);
  if (rc) goto done;
  rc = finish_check((int *)ws, stream);
  if (rc) goto done;
  GSB_TRY(cudaMemcpyAsync(best_cut_host, bc, sizeof(int64_t) * T, cudaMemcpyDeviceToHost, stream));
  GSB_TRY(cudaMemcpyAsync(sweeps_exec_host, se, sizeof(int32_t) * T, cudaMemcpyDeviceToHost, stream));
  GSB_TRY(cudaMemcpyAsync(best_bits_host, bits, nbytes * T, cudaMemcpyDeviceToHost, stream));
  GSB_TRY(cudaStreamSynchronize(stream));
done:
  cudaFreeAsync(w, stream);
  cudaFreeAsync(seeds, stream);
  cudaFreeAsync(bc, stream);
  cudaFreeAsync(se, stream);
  cudaFreeAsync(bits, stream);
  cudaFreeAsync(ws, stream);
  if (tab) cudaFreeAsync(tab, stream);
  cudaStreamSynchronize(stream);
#undef GSB_TRY
  return rc;
}

int gsb_best_key(const int64_t *best_cut, int32_t T, int64_t first, int64_t *key, void *stream) {
  if (T < 0 || first < 0) return set_error(GSB_EINVAL, "bad arguments");
  return best_key(best_cut, T, first, key, (cudaStream_t)stream);
}

}  // extern "C"
