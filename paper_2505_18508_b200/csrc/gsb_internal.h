// gsb_internal.h -- internal declarations shared by the .cu files of libgsb_cuda.so
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "../../include/gsb.h"

namespace gsb {

int set_error(int code, const char *msg);
int num_sms();
// Allow `kern` at least `bytes` of dynamic shared memory on the current device.
// The limit is only ever raised and the bookkeeping is mutex-guarded: host
// threads launching the same instantiation for tori of different sizes cannot
// lower it under each other.  Returns cudaSuccess or the CUDA error.
cudaError_t allow_dynamic_smem(const void *kern, size_t bytes);

// checkerboard engine (checker.cu)
int checker_words(int rows, int cols, int *WPR, int *nw);
bool checker_fits(int rows, int cols);
size_t checker_workspace_bytes(int rows, int cols);
int checker_run(int rows, int cols, const int8_t *w_dev, int kind, int sweeps,
                const uint64_t *table, const uint64_t *seeds, int T, int64_t *best_cut,
                int32_t *sweeps_exec, uint8_t *best_bits, void *ws, int *err_ws,
                cudaStream_t stream);

void checker_force_shape(int warps, int variant);
void checker_cluster_force_size(int c);

void checker_masks_kernel_launch(int rows, int cols, int WPR, const int8_t *w, uint4 *masks,
                                 uint4 *geo, cudaStream_t stream);
// HBM-tiled checkerboard engine (checker_hbm.cu)
bool checker_hbm_fits(int rows, int cols);
size_t checker_hbm_workspace_bytes(int rows, int cols, int T, int nsm);
int checker_hbm_run(int rows, int cols, const int8_t *w_dev, int kind, int sweeps,
                    const uint64_t *table, const uint64_t *seeds, int T, int64_t *best_cut,
                    int32_t *sweeps_exec, uint8_t *best_bits, void *ws, int *err_ws,
                    cudaStream_t stream);

// cluster checkerboard engine (checker_cluster.cu)
bool checker_cluster_fits(int rows, int cols);
size_t checker_cluster_workspace_bytes(int rows, int cols);
int checker_cluster_run(int rows, int cols, const int8_t *w_dev, int kind, int sweeps,
                        const uint64_t *table, const uint64_t *seeds, int T, int64_t *best_cut,
                        int32_t *sweeps_exec, uint8_t *best_bits, void *ws, int *err_ws,
                        cudaStream_t stream);

// random-scan engine (rscan2.cu)
bool rscan2_fits(int rows, int cols);
bool rscan2_shape(int rows, int cols, int T, int *nw, int *rb);
void rscan2_force_shape(int nw, int rb);
void rscan2_test_limits(int tqcap, int lcap);
void rscan2_force_slices(int nslice);
size_t rscan2_workspace_bytes(int rows, int cols, int T);
int rscan2_run(int rows, int cols, const int8_t *w_dev, int kind, int sweeps,
               const uint64_t *table, const uint64_t *seeds, int T, int64_t *best_cut,
               int32_t *sweeps_exec, uint8_t *best_bits, void *ws, int *err_ws,
               unsigned long long *stats, cudaStream_t stream);

// random-scan engine for tori beyond rscan2's teams (rscan_big.cu: planes in global memory)
bool rscan_big_fits(int rows, int cols);
size_t rscan_big_workspace_bytes(int rows, int cols, int T);
int rscan_big_run(int rows, int cols, const int8_t *w_dev, int kind, int sweeps,
                  const uint64_t *table, const uint64_t *seeds, int T, int64_t *best_cut,
                  int32_t *sweeps_exec, uint8_t *best_bits, void *ws, int *err_ws,
                  cudaStream_t stream);

// reference-exact engines (refexact.cu: any graph; refexact_warp.cu: tori, n < 2^16)
bool ref_warp_fits(int rows, int cols);
int ref_warp_run(int rows, int cols, const int8_t *w_dev, int kind, int sweeps,
                 const uint64_t *table, const uint64_t *seeds, int T, int64_t *best_cut,
                 int32_t *sweeps_exec, uint8_t *best_bits, void *ws, int *err_ws,
                 cudaStream_t stream);
size_t ref_workspace_bytes(int n, int64_t m_adj, int T);
int ref_run_torus(int rows, int cols, const int8_t *w_dev, int kind, int sweeps,
                  const uint64_t *table, int dmax, const uint64_t *seeds, int T,
                  int64_t *best_cut, int32_t *sweeps_exec, uint8_t *best_bits, void *ws,
                  size_t ws_bytes, int *err_ws, cudaStream_t stream);
int ref_run_graph(const gsb_graph *g, int kind, int sweeps, const uint64_t *table, int dmax,
                  const uint64_t *seeds, int T, int64_t *best_cut, int32_t *sweeps_exec,
                  uint8_t *best_bits, void *ws, size_t ws_bytes, int *err_ws,
                  cudaStream_t stream);

// evaluator / generators (evaluate.cu)
int torus_cut_energy(int rows, int cols, const int8_t *w, const uint8_t *bits, int T,
                     int64_t *cut, int64_t *energy, cudaStream_t stream);
int graph_cut_energy(const gsb_graph *g, const uint8_t *bits, int T, int64_t *cut,
                     int64_t *energy, cudaStream_t stream);
int torus_weights(int rows, int cols, uint64_t seed, int8_t *w, cudaStream_t stream);
int best_key(const int64_t *best_cut, int T, int64_t first, int64_t *key, cudaStream_t stream);
int philox_bench(int64_t blocks_per_thread, uint32_t *sink, cudaStream_t stream);
int philox_bench_threads();
int lop3_bench(int64_t lop3_per_thread, uint32_t *sink, cudaStream_t stream);

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace gsb
