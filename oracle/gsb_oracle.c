/*
 * gsb_oracle.c -- CPU restatement of the reference sweep hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see gsb_oracle.h).  Plain C, no SIMD tricks: each
 * function mirrors the reference line by line and cites it.
 *
 * Third-party arithmetic restated here (numpy, not under /root/reference; the
 * reference pins only numpy>=1.24, pkg/pyproject.toml:10; this restatement is
 * pinned to numpy 2.3.5 by tests/golden/rng_kat.json):
 *   - numpy.random.SeedSequence (O'Neill's seed_seq hash: hashmix/mix, pool 4)
 *   - PCG64 (XSL-RR 128/64, numpy pcg64_set_seed / pcg64_next32 buffering)
 *   - Generator.integers(0, 2) = Lemire bounded draw, range 2 -> bit 31 of next32
 *   - Generator.permutation(n) = arange + Fisher-Yates with masked rejection
 *     (random_interval), i = n-1 .. 1
 *   - Generator.random() = (next64 >> 11) * 2^-53
 */
#include "gsb_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------ */
/* SeedSequence -> PCG64                                               */
/* ------------------------------------------------------------------ */
#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u

static uint32_t ss_hashmix(uint32_t value, uint32_t *hc) {
    value ^= *hc;
    *hc *= SS_MULT_A;
    value *= *hc;
    value ^= value >> 16;
    return value;
}

static uint32_t ss_mix(uint32_t x, uint32_t y) {
    uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
    r ^= r >> 16;
    return r;
}

static const u128 PCG_MULT =
    ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;

static u128 pcg_state(const gso_pcg64 *g) { return ((u128)g->state_hi << 64) | g->state_lo; }
static u128 pcg_inc(const gso_pcg64 *g) { return ((u128)g->inc_hi << 64) | g->inc_lo; }
static void pcg_set(gso_pcg64 *g, u128 s) {
    g->state_hi = (uint64_t)(s >> 64);
    g->state_lo = (uint64_t)s;
}

void gso_pcg64_seed(gso_pcg64 *g, uint64_t seed) {
    /* SeedSequence(entropy=seed): entropy as little-endian uint32 words */
    uint32_t ent[2];
    int nent;
    if (seed == 0) {
        ent[0] = 0;
        nent = 1;
    } else if (seed >> 32) {
        ent[0] = (uint32_t)seed;
        ent[1] = (uint32_t)(seed >> 32);
        nent = 2;
    } else {
        ent[0] = (uint32_t)seed;
        nent = 1;
    }
    uint32_t pool[4];
    uint32_t hc = SS_INIT_A;
    for (int i = 0; i < 4; i++) pool[i] = ss_hashmix(i < nent ? ent[i] : 0u, &hc);
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
    /* generate_state(4, uint64) = 8 uint32 words, little-endian pairs */
    uint32_t words[8];
    uint32_t hb = SS_INIT_B;
    for (int i = 0; i < 8; i++) {
        uint32_t v = pool[i % 4];
        v ^= hb;
        hb *= SS_MULT_B;
        v *= hb;
        v ^= v >> 16;
        words[i] = v;
    }
    uint64_t val[4];
    for (int i = 0; i < 4; i++) val[i] = (uint64_t)words[2 * i] | ((uint64_t)words[2 * i + 1] << 32);
    /* pcg64_set_seed: s = val[0]:val[1], i = val[2]:val[3];
       pcg_setseq_128_srandom_r: state=0; inc=(i<<1)|1; step; state+=s; step */
    u128 s = ((u128)val[0] << 64) | val[1];
    u128 i = ((u128)val[2] << 64) | val[3];
    u128 inc = (i << 1) | 1u;
    u128 st = 0;
    st = st * PCG_MULT + inc;
    st += s;
    st = st * PCG_MULT + inc;
    pcg_set(g, st);
    g->inc_hi = (uint64_t)(inc >> 64);
    g->inc_lo = (uint64_t)inc;
    g->has_uint32 = 0;
    g->uinteger = 0;
}

uint64_t gso_pcg64_next64(gso_pcg64 *g) {
    u128 st = pcg_state(g) * PCG_MULT + pcg_inc(g);
    pcg_set(g, st);
    uint64_t x = (uint64_t)(st >> 64) ^ (uint64_t)st;
    unsigned rot = (unsigned)(st >> 122);
    return (x >> rot) | (x << ((-rot) & 63));
}

uint32_t gso_pcg64_next32(gso_pcg64 *g) {
    if (g->has_uint32) {
        g->has_uint32 = 0;
        return g->uinteger;
    }
    uint64_t nx = gso_pcg64_next64(g);
    g->has_uint32 = 1;
    g->uinteger = (uint32_t)(nx >> 32);
    return (uint32_t)nx;
}

/* numpy distributions.c random_interval, 32-bit branch (max < 2^32 here) */
static uint32_t random_interval32(gso_pcg64 *g, uint32_t max) {
    if (max == 0) return 0;
    uint32_t mask = max;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    uint32_t v;
    while ((v = (gso_pcg64_next32(g) & mask)) > max) {
    }
    return v;
}

void gso_pcg64_permutation(gso_pcg64 *g, int64_t n, int64_t *out) {
    for (int64_t i = 0; i < n; i++) out[i] = i;
    for (int64_t i = n - 1; i >= 1; i--) {
        int64_t j = random_interval32(g, (uint32_t)i);
        int64_t t = out[i];
        out[i] = out[j];
        out[j] = t;
    }
}

double gso_pcg64_random(gso_pcg64 *g) {
    return (double)(gso_pcg64_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}

/* ------------------------------------------------------------------ */
/* campaign.py:39-53                                                   */
/* ------------------------------------------------------------------ */
uint64_t gso_mix_seed(uint64_t master, uint64_t index) {
    uint64_t z = master + (index + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* ------------------------------------------------------------------ */
/* instances.py:203-224                                                */
/* ------------------------------------------------------------------ */
void gso_torus_weights(int rows, int cols, uint64_t seed, int8_t *w) {
    gso_pcg64 g;
    gso_pcg64_seed(&g, seed);
    int64_t m = 2 * (int64_t)rows * cols;
    /* rng.integers(0, 2, size=m) * 2 - 1 (instances.py:221-222) */
    for (int64_t k = 0; k < m; k++) w[k] = (gso_pcg64_next32(&g) >> 31) ? 1 : -1;
}

void gso_torus_edges(int rows, int cols, const int8_t *w, int32_t *eu, int32_t *ev,
                     int64_t *ew) {
    int64_t k = 0;
    for (int r = 0; r < rows; r++)
        for (int c = 0; c < cols; c++) {
            int32_t v = r * cols + c;
            int32_t right = r * cols + (c + 1) % cols;
            int32_t down = ((r + 1) % rows) * cols + c;
            int32_t nb[2] = {right, down};
            for (int e = 0; e < 2; e++, k++) {
                /* from_edges canonicalises u < v (instances.py:88-89) */
                int32_t a = v, b = nb[e];
                if (a > b) {
                    int32_t t = a;
                    a = b;
                    b = t;
                }
                eu[k] = a;
                ev[k] = b;
                ew[k] = w[k];
            }
        }
}

/* ------------------------------------------------------------------ */
/* evaluate.py:35-49                                                   */
/* ------------------------------------------------------------------ */
int64_t gso_cut(int64_t m, const int32_t *eu, const int32_t *ev, const int64_t *ew,
                const int8_t *s) {
    int64_t c = 0;
    for (int64_t e = 0; e < m; e++)
        if (s[eu[e]] != s[ev[e]]) c += ew[e];
    return c;
}

int64_t gso_energy(int64_t m, const int32_t *eu, const int32_t *ev, const int64_t *ew,
                   const int8_t *s) {
    int64_t E = 0;
    for (int64_t e = 0; e < m; e++) E += ew[e] * s[eu[e]] * s[ev[e]];
    return E;
}

/* solvers.py:84-88 */
double gso_temperature(int sweeps, double t0, double t1, int sweep_index) {
    if (sweeps == 1) return t0;
    double frac = (double)sweep_index / (double)(sweeps - 1);
    return t0 * pow(t1 / t0, frac);
}

/* ------------------------------------------------------------------ */
/* Philox4x32-10                                                       */
/* ------------------------------------------------------------------ */
void gso_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; r++) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c0 = n0;
        c1 = n1;
        c2 = n2;
        c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

/* ------------------------------------------------------------------ */
/* reference-exact trial: solvers.py:91-140                            */
/* ------------------------------------------------------------------ */
typedef struct {
    int32_t n;
    int64_t *off; /* CSR offsets [n+1] */
    int32_t *nbr;
    int64_t *wt;
} csr_t;

static int csr_build(csr_t *g, int32_t n, int64_t m, const int32_t *eu, const int32_t *ev,
                     const int64_t *ew) {
    g->n = n;
    g->off = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    g->nbr = (int32_t *)malloc(sizeof(int32_t) * (size_t)(2 * m + 1));
    g->wt = (int64_t *)malloc(sizeof(int64_t) * (size_t)(2 * m + 1));
    if (!g->off || !g->nbr || !g->wt) return -1;
    for (int64_t e = 0; e < m; e++) {
        g->off[eu[e] + 1]++;
        g->off[ev[e] + 1]++;
    }
    for (int32_t i = 0; i < n; i++) g->off[i + 1] += g->off[i];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    memcpy(fill, g->off, sizeof(int64_t) * (size_t)(n + 1));
    /* adjacency order as instances.py:55-56 (edge order, u side then v side) */
    for (int64_t e = 0; e < m; e++) {
        g->nbr[fill[eu[e]]] = ev[e];
        g->wt[fill[eu[e]]++] = ew[e];
        g->nbr[fill[ev[e]]] = eu[e];
        g->wt[fill[ev[e]]++] = ew[e];
    }
    free(fill);
    return 0;
}

static void csr_free(csr_t *g) {
    free(g->off);
    free(g->nbr);
    free(g->wt);
}

static int trial_ref_csr(const csr_t *G, int64_t m, const int32_t *eu, const int32_t *ev,
                         const int64_t *ew, int kind, int32_t sweeps, uint64_t seed, double t0,
                         double t1, int64_t *best_cut, int8_t *best_spins,
                         int32_t *sweeps_executed) {
    int32_t n = G->n;
    gso_pcg64 g;
    gso_pcg64_seed(&g, seed); /* solvers.py:94 */
    int8_t *s = (int8_t *)malloc((size_t)n);
    int8_t *bs = (int8_t *)malloc((size_t)n);
    int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    for (int32_t i = 0; i < n; i++) s[i] = (gso_pcg64_next32(&g) >> 31) ? 1 : -1; /* :96 */
    int64_t current = gso_cut(m, eu, ev, ew, s); /* :101 */
    int64_t best = current;
    memcpy(bs, s, (size_t)n);
    /* best_spins = tuple(spins) at every new best (:125-127), materialised once
       per sweep from the sweep's flip log (same snapshot, O(n) per sweep) */
    int32_t *flog = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int32_t executed = 0;
    int annealing = kind == GSO_ANNEALING;
    for (int32_t sweep = 0; sweep < sweeps; sweep++) { /* :107 */
        double temp = annealing ? gso_temperature(sweeps, t0, t1, sweep) : 0.0;
        int flipped = 0;
        int64_t nlog = 0, nbest = -1;
        gso_pcg64_permutation(&g, n, perm); /* :110 */
        for (int32_t k = 0; k < n; k++) {
            int32_t i = (int32_t)perm[k];
            int64_t delta = 0;
            for (int64_t e = G->off[i]; e < G->off[i + 1]; e++) delta += G->wt[e] * s[G->nbr[e]];
            delta *= s[i]; /* :111-115 */
            int accept;
            if (annealing)
                accept = delta >= 0 ||
                         gso_pcg64_random(&g) < exp((double)delta / temp); /* :118 */
            else
                accept = delta > 0; /* :120 */
            if (accept) {
                s[i] = (int8_t)-s[i];
                current += delta;
                flipped = 1;
                flog[nlog++] = i;
                if (current > best) { /* :125-127 */
                    best = current;
                    nbest = nlog;
                }
            }
        }
        if (nbest >= 0) {
            memcpy(bs, s, (size_t)n);
            for (int64_t f = nbest; f < nlog; f++) bs[flog[f]] = (int8_t)-bs[flog[f]];
        }
        executed = sweep + 1;
        if (!annealing && !flipped) break; /* :129-130 */
    }
    free(flog);
    int rc = 0;
    if (best != gso_cut(m, eu, ev, ew, bs)) rc = -1; /* :132-133 */
    *best_cut = best;
    if (best_spins) memcpy(best_spins, bs, (size_t)n);
    *sweeps_executed = executed;
    free(s);
    free(bs);
    free(perm);
    return rc;
}

int gso_run_trial_ref(int32_t n, int64_t m, const int32_t *eu, const int32_t *ev,
                      const int64_t *ew, int kind, int32_t sweeps, uint64_t seed, double t0,
                      double t1, int64_t *best_cut, int8_t *best_spins,
                      int32_t *sweeps_executed) {
    csr_t G;
    if (csr_build(&G, n, m, eu, ev, ew)) return -2;
    int rc = trial_ref_csr(&G, m, eu, ev, ew, kind, sweeps, seed, t0, t1, best_cut, best_spins,
                           sweeps_executed);
    csr_free(&G);
    return rc;
}

/* ------------------------------------------------------------------ */
/* checkerboard (Philox) trial -- DESIGN.md "Checkerboard contract"     */
/* ------------------------------------------------------------------ */
/* Uniform of site (r, k) of colour p at sweep t (contract v2):
 *   wi = r*WPR + (k>>5), b = k & 31,
 *   planes j = 0..7: word (j & 3) of Philox(key, (wi, t, 2p + (j >> 2), 1));
 *   u bits 31..24 = bit b of planes 0..7 (plane 0 = MSB);
 *   u bits 23..0  = (word (b & 3) of Philox(key, (wi, t, 4 + 8p + (b >> 2), 1))) >> 8. */
typedef struct {
    uint32_t key[2];
    int32_t t, p, wi;
    uint32_t planes[8];
    uint32_t tail[32];
} plane_cache;

static uint32_t checker_uniform(plane_cache *pc, int32_t t, int32_t p, int32_t wi, int bit) {
    if (pc->t != t || pc->p != p || pc->wi != wi) {
        for (int g = 0; g < 2; g++) {
            uint32_t ctr[4] = {(uint32_t)wi, (uint32_t)t, (uint32_t)(2 * p + g), 1u};
            gso_philox4x32_10(ctr, pc->key, &pc->planes[4 * g]);
        }
        for (int q = 0; q < 8; q++) {
            uint32_t ctr[4] = {(uint32_t)wi, (uint32_t)t, (uint32_t)(4 + 8 * p + q), 1u};
            gso_philox4x32_10(ctr, pc->key, &pc->tail[4 * q]);
        }
        pc->t = t;
        pc->p = p;
        pc->wi = wi;
    }
    uint32_t u = 0;
    for (int j = 0; j < 8; j++) u |= ((pc->planes[j] >> bit) & 1u) << (31 - j);
    u |= pc->tail[bit] >> 8;
    return u;
}

static int trial_checker(int32_t rows, int32_t cols, const int8_t *w, const int32_t *eu,
                         const int32_t *ev, const int64_t *ew, int kind, int32_t sweeps,
                         uint64_t seed, double t0, double t1, int64_t *best_cut,
                         int8_t *best_spins, int32_t *sweeps_executed) {
    if ((rows & 1) || (cols & 1) || rows < 4 || cols < 4) return -3;
    int32_t n = rows * cols, H = cols / 2, WPR = (H + 31) / 32;
    int64_t m = 2 * (int64_t)n;
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    int8_t *s = (int8_t *)malloc((size_t)n);
    int8_t *bs = (int8_t *)malloc((size_t)n);
    /* initial spins: site (r,k) of colour p takes bit (k&31) of word 0 of
       Philox(key, (wi, 0, p, 0)) */
    for (int32_t r = 0; r < rows; r++)
        for (int32_t c = 0; c < cols; c++) {
            int32_t p = (r + c) & 1, k = c >> 1, wi = r * WPR + (k >> 5);
            uint32_t ctr[4] = {(uint32_t)wi, 0u, (uint32_t)p, 0u}, o[4];
            gso_philox4x32_10(ctr, key, o);
            s[r * cols + c] = ((o[0] >> (k & 31)) & 1u) ? 1 : -1;
        }
    int64_t current = gso_cut(m, eu, ev, ew, s);
    int64_t best = current;
    memcpy(bs, s, (size_t)n);
    /* best_spins = tuple(spins) at every new best (solvers.py:125-127),
       materialised once per half-sweep: the flips of the half-sweep are logged
       and, if the best improved in it, bs = s minus the flips after the last
       improvement (same snapshot, O(n) per half-sweep instead of per event). */
    int32_t *flog = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int64_t nlog = 0, nbest = -1;
    int32_t executed = 0;
    int annealing = kind == GSO_ANNEALING;
    plane_cache pc;
    pc.key[0] = key[0];
    pc.key[1] = key[1];
    pc.t = -1;
    for (int32_t sweep = 0; sweep < sweeps; sweep++) {
        double temp = annealing ? gso_temperature(sweeps, t0, t1, sweep) : 0.0;
        int flipped = 0;
        for (int32_t p = 0; p < 2; p++) {
            nlog = 0;
            nbest = -1;
            for (int32_t r = 0; r < rows; r++)
                for (int32_t k = 0; k < H; k++) {
                    int32_t c = 2 * k + ((r + p) & 1);
                    int32_t i = r * cols + c;
                    int32_t cl = (c + cols - 1) % cols, cr = (c + 1) % cols;
                    int32_t ru = (r + rows - 1) % rows, rd = (r + 1) % rows;
                    int64_t delta = (int64_t)w[2 * i] * s[r * cols + cr] +
                                    (int64_t)w[2 * i + 1] * s[rd * cols + c] +
                                    (int64_t)w[2 * (r * cols + cl)] * s[r * cols + cl] +
                                    (int64_t)w[2 * (ru * cols + c) + 1] * s[ru * cols + c];
                    delta *= s[i];
                    int accept;
                    if (annealing) {
                        accept = delta >= 0;
                        if (!accept) {
                            uint32_t u = checker_uniform(&pc, sweep, p, r * WPR + (k >> 5), k & 31);
                            accept = (double)u * (1.0 / 4294967296.0) < exp((double)delta / temp);
                        }
                    } else {
                        accept = delta > 0;
                    }
                    if (accept) {
                        s[i] = (int8_t)-s[i];
                        current += delta;
                        flipped = 1;
                        flog[nlog++] = i;
                        if (current > best) {
                            best = current;
                            nbest = nlog;
                        }
                    }
                }
            if (nbest >= 0) {
                memcpy(bs, s, (size_t)n);
                for (int64_t f = nbest; f < nlog; f++) bs[flog[f]] = (int8_t)-bs[flog[f]];
            }
        }
        executed = sweep + 1;
        if (!annealing && !flipped) break;
    }
    free(flog);
    int rc = 0;
    if (best != gso_cut(m, eu, ev, ew, bs)) rc = -1;
    *best_cut = best;
    if (best_spins) memcpy(best_spins, bs, (size_t)n);
    *sweeps_executed = executed;
    free(s);
    free(bs);
    return rc;
}

/* ------------------------------------------------------------------ */
/* random-scan (Philox) trial -- DESIGN.md "Random-scan contract" (v2)  */
/* ------------------------------------------------------------------ */
/* The reference's sweep visits the sites in a fresh uniformly random order
 * (solvers.py:110) and, for each, computes Delta, accepts and flips
 * (solvers.py:111-127).  This restatement keeps solvers.py:107-127 line by
 * line and changes only where the randomness comes from: the permutation of
 * sweep t is the sites sorted by (priority, id), the priorities i.i.d. 32-bit
 * Philox values, and the acceptance uniform of a site is its own 32-bit
 * Philox value.  Layout of the draws (key = (lo32(seed), hi32(seed)),
 * TAG = 5, WPR = ceil(cols / 32), site (r, c): word wi = r*WPR + (c >> 5),
 * bit b = c & 31, id = r*cols + c):
 *   initial spin:  bit b of word 0 of Philox(key, (wi, 0, 31, TAG)) (1 = +1);
 *   priority(t):   bits 31..24 = bit b of planes j = 0..7 (plane 0 = MSB),
 *                  plane j = word (j & 3) of Philox(key, (wi, t, j >> 2, TAG));
 *                  bits 23..0 = word (b & 3) of Philox(key, (wi, t, 2 + (b >> 2), TAG)) >> 8;
 *   uniform(t):    the same with q = 10 + (j >> 2) for the planes and
 *                  q = 12 + (b >> 2) for the low bits;
 *   accept Delta < 0 iff uniform * 2^-32 < exp(Delta / T_t).
 * The GPU engine runs the same order level by level and recovers the
 * best-so-far of this sequential scan exactly (rscan2.cu). */
#define RS_TAG 5u

typedef struct {
    uint32_t p;
    int32_t v;
} prio_t;

static int prio_cmp(const void *a, const void *b) {
    const prio_t *x = (const prio_t *)a, *y = (const prio_t *)b;
    if (x->p != y->p) return x->p < y->p ? -1 : 1;
    return x->v < y->v ? -1 : (x->v > y->v);
}

/* The 32 Philox values of word wi at sweep t (one per bit b): bits 31..24 from
 * the planes of blocks q0, q0+1, bits 23..0 from word (b & 3) of block
 * q0 + 2 + (b >> 2), shifted right by 8. */
static void rs_values(const uint32_t key[2], uint32_t wi, uint32_t t, uint32_t q0,
                      uint32_t out[32]) {
    uint32_t pl[8], o[4];
    for (uint32_t g = 0; g < 2; g++) {
        uint32_t ctr[4] = {wi, t, q0 + g, RS_TAG};
        gso_philox4x32_10(ctr, key, o);
        for (int j = 0; j < 4; j++) pl[4 * g + j] = o[j];
    }
    for (int b = 0; b < 32; b++) {
        uint32_t hi = 0;
        for (int j = 0; j < 8; j++) hi |= ((pl[j] >> b) & 1u) << (31 - j);
        out[b] = hi;
    }
    for (uint32_t g = 0; g < 8; g++) {
        uint32_t ctr[4] = {wi, t, q0 + 2u + g, RS_TAG};
        gso_philox4x32_10(ctr, key, o);
        for (int j = 0; j < 4; j++) out[4 * g + j] |= o[j] >> 8;
    }
}

static int trial_rscan(int32_t rows, int32_t cols, const int8_t *w, const int32_t *eu,
                       const int32_t *ev, const int64_t *ew, int kind, int32_t sweeps,
                       uint64_t seed, double t0, double t1, int64_t *best_cut,
                       int8_t *best_spins, int32_t *sweeps_executed) {
    int32_t n = rows * cols, WPR = (cols + 31) / 32;
    int64_t m = 2 * (int64_t)n;
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    int8_t *s = (int8_t *)malloc((size_t)n);
    int8_t *bs = (int8_t *)malloc((size_t)n);
    prio_t *pr = (prio_t *)malloc(sizeof(prio_t) * (size_t)n);
    int32_t *flog = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int32_t nwords = rows * WPR;
    uint32_t *uval = (uint32_t *)malloc(sizeof(uint32_t) * 32 * (size_t)nwords);
    int32_t *ustamp = (int32_t *)malloc(sizeof(int32_t) * (size_t)nwords);
    uint32_t vals[32];
    for (int32_t v = 0; v < n; v++) {
        int32_t r = v / cols, c = v % cols;
        uint32_t ctr[4] = {(uint32_t)(r * WPR + (c >> 5)), 0u, 31u, RS_TAG}, o[4];
        gso_philox4x32_10(ctr, key, o);
        s[v] = ((o[0] >> (c & 31)) & 1u) ? 1 : -1;
    }
    int64_t current = gso_cut(m, eu, ev, ew, s); /* solvers.py:101 */
    int64_t best = current;                      /* solvers.py:102-103 */
    memcpy(bs, s, (size_t)n);
    int32_t executed = 0;
    int annealing = kind == GSO_ANNEALING;
    for (int32_t sweep = 0; sweep < sweeps; sweep++) {
        double temp = annealing ? gso_temperature(sweeps, t0, t1, sweep) : 0.0;
        /* the sweep's order (solvers.py:110): sites sorted by (priority, id) */
        for (int32_t wi = 0; wi < nwords; wi++) {
            int32_t r = wi / WPR, c0 = 32 * (wi % WPR);
            rs_values(key, (uint32_t)wi, (uint32_t)sweep, 0u, vals);
            for (int b = 0; b < 32 && c0 + b < cols; b++) {
                int32_t v = r * cols + c0 + b;
                pr[v].p = vals[b];
                pr[v].v = v;
            }
            ustamp[wi] = -1;
        }
        qsort(pr, (size_t)n, sizeof(prio_t), prio_cmp);
        int flipped = 0;
        int64_t nlog = 0, nbest = -1;
        for (int32_t i = 0; i < n; i++) { /* solvers.py:111-127 */
            int32_t v = pr[i].v, r = v / cols, c = v % cols;
            int32_t cl = (c + cols - 1) % cols, cr = (c + 1) % cols;
            int32_t ru = (r + rows - 1) % rows, rd = (r + 1) % rows;
            int64_t delta = (int64_t)w[2 * v] * s[r * cols + cr] +
                            (int64_t)w[2 * v + 1] * s[rd * cols + c] +
                            (int64_t)w[2 * (r * cols + cl)] * s[r * cols + cl] +
                            (int64_t)w[2 * (ru * cols + c) + 1] * s[ru * cols + c];
            delta *= s[v];
            int accept;
            if (annealing) {
                accept = delta >= 0;
                if (!accept) {
                    int32_t wi = r * WPR + (c >> 5);
                    if (ustamp[wi] != sweep) {
                        rs_values(key, (uint32_t)wi, (uint32_t)sweep, 10u, uval + 32 * (size_t)wi);
                        ustamp[wi] = sweep;
                    }
                    uint32_t u = uval[32 * (size_t)wi + (c & 31)];
                    accept = (double)u * (1.0 / 4294967296.0) < exp((double)delta / temp);
                }
            } else {
                accept = delta > 0;
            }
            if (accept) {
                s[v] = (int8_t)-s[v];
                current += delta;
                flipped = 1;
                flog[nlog++] = v;
                if (current > best) {
                    best = current;
                    nbest = nlog;
                }
            }
        }
        if (nbest >= 0) { /* snapshot at the last improvement of the sweep */
            memcpy(bs, s, (size_t)n);
            for (int64_t f = nbest; f < nlog; f++) bs[flog[f]] = (int8_t)-bs[flog[f]];
        }
        executed = sweep + 1;
        if (!annealing && !flipped) break;
    }
    int rc = 0;
    if (best != gso_cut(m, eu, ev, ew, bs)) rc = -1;
    *best_cut = best;
    if (best_spins) memcpy(best_spins, bs, (size_t)n);
    *sweeps_executed = executed;
    free(s); free(bs); free(pr); free(flog); free(uval); free(ustamp);
    return rc;
}

typedef struct {
    int32_t rows, cols;
    const int8_t *w;
    int32_t *eu, *ev;
    int64_t *ew;
    int64_t m;
} torus_edges_t;

static int torus_edges_alloc(torus_edges_t *te, int32_t rows, int32_t cols, const int8_t *w) {
    te->rows = rows;
    te->cols = cols;
    te->w = w;
    te->m = 2 * (int64_t)rows * cols;
    te->eu = (int32_t *)malloc(sizeof(int32_t) * (size_t)te->m);
    te->ev = (int32_t *)malloc(sizeof(int32_t) * (size_t)te->m);
    te->ew = (int64_t *)malloc(sizeof(int64_t) * (size_t)te->m);
    if (!te->eu || !te->ev || !te->ew) return -1;
    gso_torus_edges(rows, cols, w, te->eu, te->ev, te->ew);
    return 0;
}

static void torus_edges_free(torus_edges_t *te) {
    free(te->eu);
    free(te->ev);
    free(te->ew);
}

int gso_run_trial_checker(int32_t rows, int32_t cols, const int8_t *w, int kind,
                          int32_t sweeps, uint64_t seed, double t0, double t1,
                          int64_t *best_cut, int8_t *best_spins, int32_t *sweeps_executed) {
    torus_edges_t te;
    if (torus_edges_alloc(&te, rows, cols, w)) return -2;
    int rc = trial_checker(rows, cols, w, te.eu, te.ev, te.ew, kind, sweeps, seed, t0, t1,
                           best_cut, best_spins, sweeps_executed);
    torus_edges_free(&te);
    return rc;
}

int gso_run_trial_rscan(int32_t rows, int32_t cols, const int8_t *w, int kind, int32_t sweeps,
                        uint64_t seed, double t0, double t1, int64_t *best_cut,
                        int8_t *best_spins, int32_t *sweeps_executed) {
    torus_edges_t te;
    if (torus_edges_alloc(&te, rows, cols, w)) return -2;
    int rc = trial_rscan(rows, cols, w, te.eu, te.ev, te.ew, kind, sweeps, seed, t0, t1,
                         best_cut, best_spins, sweeps_executed);
    torus_edges_free(&te);
    return rc;
}

/* ------------------------------------------------------------------ */
/* batched, multi-threaded                                              */
/* ------------------------------------------------------------------ */
typedef struct {
    int mode; /* 0 ref, 1 checker, 2 random scan */
    const csr_t *G;
    int64_t m;
    const int32_t *eu, *ev;
    const int64_t *ew;
    int32_t rows, cols;
    const int8_t *w;
    int kind;
    int32_t sweeps, T, n;
    const uint64_t *seeds;
    double t0, t1;
    int64_t *best_cut;
    int8_t *best_spins;
    int32_t *sweeps_executed;
    int nthreads, tid;
    int rc;
} job_t;

static void *job_run(void *arg) {
    job_t *j = (job_t *)arg;
    j->rc = 0;
    for (int32_t t = j->tid; t < j->T; t += j->nthreads) {
        int8_t *bs = j->best_spins ? j->best_spins + (int64_t)t * j->n : NULL;
        int rc;
        if (j->mode == 0)
            rc = trial_ref_csr(j->G, j->m, j->eu, j->ev, j->ew, j->kind, j->sweeps, j->seeds[t],
                               j->t0, j->t1, &j->best_cut[t], bs, &j->sweeps_executed[t]);
        else if (j->mode == 1)
            rc = trial_checker(j->rows, j->cols, j->w, j->eu, j->ev, j->ew, j->kind, j->sweeps,
                               j->seeds[t], j->t0, j->t1, &j->best_cut[t], bs,
                               &j->sweeps_executed[t]);
        else
            rc = trial_rscan(j->rows, j->cols, j->w, j->eu, j->ev, j->ew, j->kind, j->sweeps,
                             j->seeds[t], j->t0, j->t1, &j->best_cut[t], bs,
                             &j->sweeps_executed[t]);
        if (rc && !j->rc) j->rc = rc;
    }
    return NULL;
}

static int run_jobs(job_t *proto, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > proto->T) nthreads = proto->T;
    job_t *jobs = (job_t *)malloc(sizeof(job_t) * (size_t)nthreads);
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int i = 0; i < nthreads; i++) {
        jobs[i] = *proto;
        jobs[i].nthreads = nthreads;
        jobs[i].tid = i;
        pthread_create(&th[i], NULL, job_run, &jobs[i]);
    }
    int rc = 0;
    for (int i = 0; i < nthreads; i++) {
        pthread_join(th[i], NULL);
        if (jobs[i].rc && !rc) rc = jobs[i].rc;
    }
    free(jobs);
    free(th);
    return rc;
}

int gso_run_trials_ref(int32_t n, int64_t m, const int32_t *eu, const int32_t *ev,
                       const int64_t *ew, int kind, int32_t sweeps, int32_t T,
                       const uint64_t *seeds, double t0, double t1, int64_t *best_cut,
                       int8_t *best_spins, int32_t *sweeps_executed, int nthreads) {
    csr_t G;
    if (csr_build(&G, n, m, eu, ev, ew)) return -2;
    job_t p;
    memset(&p, 0, sizeof p);
    p.mode = 0;
    p.G = &G;
    p.m = m;
    p.eu = eu;
    p.ev = ev;
    p.ew = ew;
    p.kind = kind;
    p.sweeps = sweeps;
    p.T = T;
    p.n = n;
    p.seeds = seeds;
    p.t0 = t0;
    p.t1 = t1;
    p.best_cut = best_cut;
    p.best_spins = best_spins;
    p.sweeps_executed = sweeps_executed;
    int rc = run_jobs(&p, nthreads);
    csr_free(&G);
    return rc;
}

static int run_torus_jobs(int mode, int32_t rows, int32_t cols, const int8_t *w, int kind,
                          int32_t sweeps, int32_t T, const uint64_t *seeds, double t0,
                          double t1, int64_t *best_cut, int8_t *best_spins,
                          int32_t *sweeps_executed, int nthreads) {
    torus_edges_t te;
    if (torus_edges_alloc(&te, rows, cols, w)) return -2;
    job_t p;
    memset(&p, 0, sizeof p);
    p.mode = mode;
    p.m = te.m;
    p.eu = te.eu;
    p.ev = te.ev;
    p.ew = te.ew;
    p.rows = rows;
    p.cols = cols;
    p.w = w;
    p.kind = kind;
    p.sweeps = sweeps;
    p.T = T;
    p.n = rows * cols;
    p.seeds = seeds;
    p.t0 = t0;
    p.t1 = t1;
    p.best_cut = best_cut;
    p.best_spins = best_spins;
    p.sweeps_executed = sweeps_executed;
    int rc = run_jobs(&p, nthreads);
    torus_edges_free(&te);
    return rc;
}

int gso_run_trials_checker(int32_t rows, int32_t cols, const int8_t *w, int kind,
                           int32_t sweeps, int32_t T, const uint64_t *seeds, double t0,
                           double t1, int64_t *best_cut, int8_t *best_spins,
                           int32_t *sweeps_executed, int nthreads) {
    return run_torus_jobs(1, rows, cols, w, kind, sweeps, T, seeds, t0, t1, best_cut, best_spins,
                          sweeps_executed, nthreads);
}

int gso_run_trials_rscan(int32_t rows, int32_t cols, const int8_t *w, int kind, int32_t sweeps,
                         int32_t T, const uint64_t *seeds, double t0, double t1,
                         int64_t *best_cut, int8_t *best_spins, int32_t *sweeps_executed,
                         int nthreads) {
    return run_torus_jobs(2, rows, cols, w, kind, sweeps, T, seeds, t0, t1, best_cut, best_spins,
                          sweeps_executed, nthreads);
}
