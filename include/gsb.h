/*
 * gsb.h -- C ABI of the B200 sweep engine (libgsb_cuda.so).
 *
 * Drop-in boundary for the reference's hot path.  The reference is pure
 * Python (gsetbench, /root/reference/pkg/src/gsetbench); its "FFI" for this
 * path is the Python call surface itself, so each entry point below names the
 * reference function it replaces.  The Python package paper_2505_18508_b200
 * binds these with ctypes (INTEGRATION.md shows the binding).
 *
 * Conventions
 *  - Plain pointers and sizes only.  `*_dev` pointers are device memory on the
 *    current CUDA device, `stream` is a cudaStream_t passed as void* (NULL =
 *    legacy default stream).  The caller owns every buffer; the library keeps
 *    no state between calls apart from a per-device property cache.
 *  - Return 0 on success or a negative GSB_E* code; gsb_last_error() returns a
 *    thread-local message for the last failure on the calling thread.
 *  - Spin bitstrings ("bits") are packed MSB-first by variable id: byte b, bit
 *    (7-j) is variable 8b+j+1 (1-based), 1 = spin +1, pad bits 0 -- so
 *    bytes(bits[:ceil(n/8)]).hex()[:ceil(n/4)] == gsetbench.codec.encode_hex
 *    (codec.py:64-83).
 *  - Torus weights `w` are int8 [rows*cols*2]: w[2x] = weight of the edge from
 *    site x to its right neighbour, w[2x+1] to its down neighbour, x = r*cols+c
 *    (0-based) -- exactly the emission order of generate_torus
 *    (instances.py:211-223).
 */
#ifndef GSB_H
#define GSB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSB_ABI_VERSION 1

/* error codes */
#define GSB_OK 0
#define GSB_EINVAL -1    /* invalid argument (Python: ValueError)           */
#define GSB_ECUDA -2     /* CUDA runtime failure (Python: RuntimeError)      */
#define GSB_EINTEGRITY -3 /* cut accounting drift, solvers.py:132-133        */
#define GSB_ENOMEM -4    /* workspace too small / allocation failed          */
#define GSB_EUNSUPPORTED -5 /* instance shape not supported by the engine    */

/* solver kinds: solvers.py:27-29 (+ engine selects the sweep order / RNG) */
#define GSB_GREEDY 0
#define GSB_ANNEALING 1

/* engines */
#define GSB_ENGINE_REFERENCE 0    /* numpy-PCG64 + random permutation: bit-exact with run_trial */
#define GSB_ENGINE_CHECKERBOARD 1 /* Philox4x32-10 + colour order (DESIGN.md contract)        */
#define GSB_ENGINE_CHECKERBOARD_TILED 2 /* same contract, forces the HBM-tiled engine (used
                                           automatically when the torus exceeds a cluster) */
#define GSB_ENGINE_CHECKERBOARD_CLUSTER 3 /* same contract, forces the cluster engine (one trial
                                             over the shared memory of a CTA cluster; used
                                             automatically when the torus exceeds one SM) */
#define GSB_ENGINE_RANDOM_SCAN 4  /* Philox4x32-10 + the reference's random visit order
                                     (i.i.d. 32-bit priorities, DESIGN.md random-scan contract):
                                     solvers.py:107-127 with the same law, best-so-far of the
                                     sequential scan exact; tori up to 8 warps x 7 rows per lane */

#define GSB_ENGINE_RANDOM_SCAN_LARGE 5 /* same contract and results as RANDOM_SCAN, forces the
                                         engine for tori beyond one SM (planes in global
                                         memory, one cooperative kernel per 8 trials; used
                                         automatically when the torus exceeds the teams) */

typedef struct gsb_torus {
    int32_t rows, cols;  /* TorusSpec.rows/cols (instances.py:186-187), >= 3 */
    const int8_t *w_dev; /* [rows*cols*2] device pointer, see above           */
} gsb_torus;

typedef struct gsb_graph { /* general instance, ProblemInstance (instances.py:19-62) */
    int32_t n;             /* vertices 1..n                                           */
    int64_t m;             /* edges                                                   */
    const int32_t *eu_dev; /* [m] 0-based endpoint u (u < v), edge order as .edges     */
    const int32_t *ev_dev; /* [m] 0-based endpoint v                                  */
    const int32_t *ew_dev; /* [m] integer weight                                      */
} gsb_graph;

/* ---- library ---- */
const char *gsb_last_error(void);
int gsb_abi_version(void);
/* number of CUDA devices visible (0 if none) */
int gsb_device_count(void);

/* ---- seeds / instances ---- */
/* campaign.mix_seed (campaign.py:39-53) for indices first..first+T-1, host out */
int gsb_mix_seeds(uint64_t master_seed, int64_t first_index, int32_t T, uint64_t *seeds_out);

/* generate_torus weights (instances.py:221-223): numpy default_rng(seed)
 * .integers(0, 2, 2n)*2-1, computed on the device with PCG64 jump-ahead. */
int gsb_torus_weights(int32_t rows, int32_t cols, uint64_t seed, int8_t *w_dev, void *stream);

/* ---- evaluator (evaluate.py:35-49) ---- */
/* cut_value / ising_energy of T packed bitstrings [T][ceil(n/8)] */
int gsb_torus_cut_energy(const gsb_torus *inst, const uint8_t *bits_dev, int32_t T,
                         int64_t *cut_dev, int64_t *energy_dev, void *stream);
int gsb_graph_cut_energy(const gsb_graph *g, const uint8_t *bits_dev, int32_t T,
                         int64_t *cut_dev, int64_t *energy_dev, void *stream);

/* ---- schedule (solvers.py:84-88, :118) ---- */
/* Host-side acceptance thresholds, computed with the platform libm exactly as
 * the reference's math.exp / float ** do.  Table layout [sweeps][dmax] uint64:
 *  reference engine:    K[t][d-1] = ceil(exp(-d / T_t) * 2^53)  (accept iff next64>>11 < K)
 *  checkerboard engine: K[t][d-1] = ceil(exp(-d / T_t) * 2^32)  (accept iff u32 < K)
 * dmax = 4 for the +-1 torus.  Greedy needs no table (pass NULL). */
int gsb_schedule_table(int engine, int32_t sweeps, double temp_start, double temp_end,
                       int32_t dmax, uint64_t *table_host);

/* ---- the hot path: batched trials (solvers.py:91-140 x campaign.py:324-429) ----
 * T independent trials, trial t keyed by seeds_dev[t] (the SolverConfig.seed
 * of run_trial, i.e. mix_seed(master, index) in a campaign).  Outputs per
 * trial: best_cut, sweeps_executed and the best bitstring.  Results depend
 * only on (instance, engine, kind, sweeps, temperatures, seed) -- never on T,
 * the trial's position in the batch or the device count. */
size_t gsb_torus_workspace_bytes(const gsb_torus *inst, int engine, int32_t sweeps,
                                 int32_t T);
int gsb_torus_sweep(const gsb_torus *inst, int engine, int kind, int32_t sweeps,
                    const uint64_t *table_dev, const uint64_t *seeds_dev, int32_t T,
                    int64_t *best_cut_dev, int32_t *sweeps_executed_dev, uint8_t *best_bits_dev,
                    void *workspace_dev, size_t workspace_bytes, void *stream);

/* Which random-scan engine a rows x cols torus gets: 1 = the register-resident
 * teams (cols <= 1024 and rows <= 8 * floor(32 / ceil(cols / 32)) * 7), 2 = the
 * large-torus engine (n < 2^28), 0 = none. */
int gsb_rscan_fits(int32_t rows, int32_t cols);

/* Team shape the random-scan engine launches for T trials of a rows x cols
 * torus (one CTA of *warps warps per trial, *rows_per_lane rows per lane);
 * needs a device (SM count).  Introspection for tests and profiles. */
int gsb_rscan_shape(int32_t rows, int32_t cols, int32_t T, int32_t *warps, int32_t *rows_per_lane);

/* TEST-ONLY: force the checkerboard engine's team shape for later launches of
 * this process: warps per trial (1, 2, 4, 8, 16; 0 = automatic) and the
 * one-warp kernel variant (0 = automatic, 1 = 128-register, 2 = the 8-per-SM
 * variant the engine picks when the trials fill fewer than 8 warps per SM), so
 * parity tests can run the benchmark's instantiations on a handful of trials.
 * gsb_test_cluster_size forces the cluster engine's CTA count (0 = automatic). */
int gsb_test_checker_shape(int32_t warps, int32_t variant);
int gsb_test_cluster_size(int32_t ctas);

/* TEST-ONLY: force the team shape (warps per trial, rows per lane) of later
 * random-scan launches of this process, so parity tests can reach every kernel
 * instantiation at small trial counts; (0, 0) restores the automatic choice.
 * A shape that cannot hold the torus makes the sweep return GSB_EUNSUPPORTED. */
int gsb_test_rscan_shape(int32_t warps, int32_t rows_per_lane);

/* TEST-ONLY: shrink the random-scan engine's tie queue and step-4b event list
 * (0 = default) so parity tests reach their overflow paths (ties decided by
 * the owning lane, candidate buckets split over passes, ordered extraction). */
int gsb_test_rscan_limits(int32_t tie_queue_cap, int32_t list_cap);

/* TEST-ONLY: force the number of sweep slices of annealing random-scan launches
 * (0 = the launcher's choice: slices only when the trials exceed the resident
 * teams and the schedule is long).  Results never depend on it. */
int gsb_test_rscan_slices(int32_t slices);

/* Counters of the last random-scan sweep call on this workspace: out4[0] =
 * rounds (summed over trials), [1] sweeps whose best-so-far needed the bucket
 * pass, [2] candidate buckets sorted exactly, [3] top-byte ties resolved by
 * low bits.  Synchronises `stream`. */
int gsb_workspace_rscan_stats(const void *workspace_dev, void *stream, uint64_t *out4);

/* The sweep calls are asynchronous on `stream`.  The integrity guard of
 * solvers.py:132-133 (best_cut == cut of the best bitstring, recomputed on
 * the device) is recorded in the workspace; gsb_workspace_status synchronises
 * `stream` and returns GSB_OK or GSB_EINTEGRITY for the last sweep call that
 * used this workspace. */
int gsb_workspace_status(const void *workspace_dev, void *stream);

/* Statistics of the last checkerboard sweep on this workspace: the number of
 * Philox4x32-10 blocks the contract required (init + 8 planes per word and
 * half-sweep + the per-site tail groups).  Synchronises `stream`. */
int gsb_workspace_counters(const void *workspace_dev, void *stream, uint64_t *philox_blocks);

/* Philox4x32-10 throughput probe (roofline denominator): launches
 * SMs x 8 x 256 threads, each evaluating blocks_per_thread blocks. */
int gsb_philox_bench(int64_t blocks_per_thread, uint32_t *sink_dev, void *stream);

/* ALU-pipe throughput probe (roofline denominator of the bit-sliced kernels):
 * SMs x 8 x 256 threads, each issuing lop3_per_thread LOP3 (8 independent
 * chains; a multiple of 32). */
int gsb_lop3_bench(int64_t lop3_per_thread, uint32_t *sink_dev, void *stream);

/* reference engine on a general graph (any integer weights, dmax = max_i sum_j |w_ij|) */
size_t gsb_graph_workspace_bytes(const gsb_graph *g, int32_t sweeps, int32_t T);
int gsb_graph_sweep(const gsb_graph *g, int kind, int32_t sweeps, const uint64_t *table_dev,
                    int32_t dmax, const uint64_t *seeds_dev, int32_t T, int64_t *best_cut_dev,
                    int32_t *sweeps_executed_dev, uint8_t *best_bits_dev, void *workspace_dev,
                    size_t workspace_bytes, void *stream);

/* Host-buffer convenience entry (the e2e path): weights, seeds and outputs in
 * host memory; the library allocates device memory, copies in, runs
 * gsb_torus_sweep on `stream` and copies the results back (synchronous). */
int gsb_torus_sweep_host(int32_t rows, int32_t cols, const int8_t *w_host, int engine, int kind,
                         int32_t sweeps, double temp_start, double temp_end,
                         const uint64_t *seeds_host, int32_t T, int64_t *best_cut_host,
                         int32_t *sweeps_executed_host, uint8_t *best_bits_host, void *stream);

/* ---- multi-GPU reduction helper ----
 * key[t] = (best_cut[t] << 32) | (0xFFFFFFFF - (first_index + t)) as int64 and
 * the argmax over the batch (highest cut wins, ties -> lowest trial index);
 * the caller all-reduces the key (NCCL max) and broadcasts the winner's bits. */
int gsb_best_key(const int64_t *best_cut_dev, int32_t T, int64_t first_index, int64_t *key_dev,
                 void *stream);

#ifdef __cplusplus
}
#endif
#endif
