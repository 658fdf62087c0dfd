/*
 * gsb_oracle.h -- CPU restatement of the reference sweep hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product path (paper_2505_18508_b200, libgsb_cuda.so) never
 * links or calls it.
 *
 * Two trial semantics are restated here:
 *
 *  (1) "reference-exact": gsetbench.solvers.run_trial
 *      (/root/reference/pkg/src/gsetbench/solvers.py:91-140) with numpy's
 *      default_rng stream (SeedSequence -> PCG64, third-party numpy, verified
 *      against numpy 2.3.5 through tests/golden/rng_kat.json) -- sequential
 *      random-permutation sweeps, Delta from the neighbour sum, SA acceptance
 *      `u < exp(Delta/T)` with u = (next64 >> 11) * 2^-53, best-so-far on strict
 *      improvement, greedy early stop.  Pinned bit-for-bit against the Python
 *      reference by tests/golden/trials_small.json, graphs_small.json,
 *      c1_full.json and the c2/c3/c4 samples.
 *
 *  (2) "checkerboard" (Philox): the same trial with exactly two changes, the
 *      sweep order (all colour-0 sites of the bipartite torus in increasing id,
 *      then all colour-1 sites) and the RNG (counter-based Philox4x32-10 keyed by
 *      the trial seed).  DESIGN.md section "Checkerboard contract" is the
 *      normative statement; this file is its executable form.
 *
 *  (3) "random scan" (Philox): solvers.py:107-127 unchanged -- a fresh
 *      uniformly random visit order every sweep, scanned sequentially --
 *      with the permutation drawn as i.i.d. 32-bit Philox priorities (sites
 *      sorted by (priority, id)) and the acceptance uniforms from Philox: the
 *      reference's dynamics in law.
 */
#ifndef GSB_ORACLE_H
#define GSB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { GSO_GREEDY = 0, GSO_ANNEALING = 1 };

typedef struct {
    uint64_t state_hi, state_lo;
    uint64_t inc_hi, inc_lo;
    int has_uint32;
    uint32_t uinteger;
} gso_pcg64;

/* numpy: np.random.default_rng(seed) for 0 <= seed < 2^64 */
void gso_pcg64_seed(gso_pcg64 *g, uint64_t seed);
uint64_t gso_pcg64_next64(gso_pcg64 *g);
uint32_t gso_pcg64_next32(gso_pcg64 *g);
/* numpy Generator.integers(0, 2) element / permutation(n) / random() */
void gso_pcg64_permutation(gso_pcg64 *g, int64_t n, int64_t *out);
double gso_pcg64_random(gso_pcg64 *g);

/* campaign.py:39-53 */
uint64_t gso_mix_seed(uint64_t master, uint64_t index);

/* instances.py:203-224: w[2x] = right edge of site x, w[2x+1] = down edge */
void gso_torus_weights(int rows, int cols, uint64_t seed, int8_t *w);
/* edge list of generate_torus in emission order (0-based endpoints, u<v) */
void gso_torus_edges(int rows, int cols, const int8_t *w, int32_t *eu, int32_t *ev,
                     int64_t *ew);

/* evaluate.py:35-49 on an edge list; spins are int8 +-1 */
int64_t gso_cut(int64_t m, const int32_t *eu, const int32_t *ev, const int64_t *ew,
                const int8_t *spins);
int64_t gso_energy(int64_t m, const int32_t *eu, const int32_t *ev, const int64_t *ew,
                   const int8_t *spins);

/* solvers.py:84-88 */
double gso_temperature(int sweeps, double t0, double t1, int sweep_index);

/* Philox4x32-10 block function (Salmon et al. 2011; Random123) */
void gso_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* reference-exact trial on a general graph (edge list, any integer weights).
 * Returns 0, or -1 on the integrity-guard failure of solvers.py:132-133. */
int gso_run_trial_ref(int32_t n, int64_t m, const int32_t *eu, const int32_t *ev,
                      const int64_t *ew, int kind, int32_t sweeps, uint64_t seed,
                      double t0, double t1, int64_t *best_cut, int8_t *best_spins,
                      int32_t *sweeps_executed);

/* checkerboard (Philox) trial on a rows x cols torus, rows and cols even. */
int gso_run_trial_checker(int32_t rows, int32_t cols, const int8_t *w, int kind,
                          int32_t sweeps, uint64_t seed, double t0, double t1,
                          int64_t *best_cut, int8_t *best_spins, int32_t *sweeps_executed);

/* random-scan (Philox) trial on any rows x cols torus (rows, cols >= 3): the
 * reference's random-order sweep with priorities drawn from Philox, executed
 * level by level. */
int gso_run_trial_rscan(int32_t rows, int32_t cols, const int8_t *w, int kind, int32_t sweeps,
                        uint64_t seed, double t0, double t1, int64_t *best_cut,
                        int8_t *best_spins, int32_t *sweeps_executed);

/* batched, multi-threaded (pthreads) versions: trial t uses seeds[t];
 * best_spins is [T][n] (may be NULL).  Returns 0 or the first failure. */
int gso_run_trials_ref(int32_t n, int64_t m, const int32_t *eu, const int32_t *ev,
                       const int64_t *ew, int kind, int32_t sweeps, int32_t T,
                       const uint64_t *seeds, double t0, double t1, int64_t *best_cut,
                       int8_t *best_spins, int32_t *sweeps_executed, int nthreads);
int gso_run_trials_checker(int32_t rows, int32_t cols, const int8_t *w, int kind,
                           int32_t sweeps, int32_t T, const uint64_t *seeds, double t0,
                           double t1, int64_t *best_cut, int8_t *best_spins,
                           int32_t *sweeps_executed, int nthreads);
int gso_run_trials_rscan(int32_t rows, int32_t cols, const int8_t *w, int kind, int32_t sweeps,
                         int32_t T, const uint64_t *seeds, double t0, double t1,
                         int64_t *best_cut, int8_t *best_spins, int32_t *sweeps_executed,
                         int nthreads);

#ifdef __cplusplus
}
#endif
#endif
