/*
 * synth.c — seeded, deterministic synthetic workload generator.
 *
 * This module is SHARED INPUT GENERATION ONLY: it produces ASCII query/target pairs, their
 * lengths and the per-pair initial score h0.  It holds none of the method's arithmetic (no
 * scoring, no DP, no packing), so both the CUDA path and the CPU oracle can consume its output
 * without sharing any code with each other.
 *
 * PRNG: SplitMix64.  Every pair owns an independent stream seeded by
 *     state0 = splitmix64_mix(seed ^ (cfg << 56) ^ pair_index)
 * so any slice of a batch can be generated in parallel and reproduced exactly
 * (SURVEY §8(d) "per-pair stream", "per-pair derived seeds").
 *
 * Wgsim-like read model ("in-house sequence read simulator similar to Wgsim";
 * SPEC S:414-463 readsim):
 *   - source bases i.i.d. uniform over ACGT;
 *   - walking the source: with p_ins an insertion of ell random bases, with p_del a deletion of
 *     ell source bases, otherwise copy the next source base, substituted (uniform over the other
 *     three) with probability p_sub; stop when the query reaches its nominal length;
 *   - the target is the consumed source window plus random flanks split uniformly left/right.
 * Optional parity-only N injection at rate p_n on both sides (separate stream).
 *
 * Configs 1..5 are the BASELINE.json configs, exactly as SURVEY §8(d) tabulates them.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

static inline uint64_t sm_mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
typedef struct { uint64_t s; } rng_t;
static inline uint64_t rng_next(rng_t* r) {
    uint64_t z = (r->s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static inline double rng_unif(rng_t* r) { return (double)(rng_next(r) >> 11) * (1.0 / 9007199254740992.0); }
/* uniform integer in [lo, hi] (inclusive) */
static inline int64_t rng_int(rng_t* r, int64_t lo, int64_t hi) {
    if (hi <= lo) return lo;
    return lo + (int64_t)(rng_next(r) % (uint64_t)(hi - lo + 1));
}

/* ---- length distributions ------------------------------------------------------------- */
enum { QD_UNIFORM = 0, QD_LOGUNIFORM = 1, QD_HIST_Q250 = 2 };
enum { TD_ABS_UNIFORM = 0, TD_QLEN_TO_1P5 = 1, TD_FLANK = 2, TD_HIST_R250 = 3 };

typedef struct {
    int qdist, qlo, qhi;
    int tdist, tlo, thi; /* TD_FLANK: flank U{tlo..thi}; others: nominal absolute target length */
    double p_sub, p_ins, p_del;
    int ell_lo, ell_hi;
} profile_t;

/* PAPER.md P:209-220 (fig:histo250, Query-250bp): ybar-interval bins of width 25 from 25. */
static const double HIST_Q250_LO = 25, HIST_Q250_W = 25;
static const double HIST_Q250[10] = {50660999, 54919472, 57779537, 59423447, 62531367,
                                     59729170, 56895730, 53725113, 53759244, 10924482};
/* PAPER.md P:281-291 (fig:histo250, Ref-250bp): bins of width 50 from 50. */
static const double HIST_R250_LO = 50, HIST_R250_W = 50;
static const double HIST_R250[9] = {55909280, 54744255, 57389925, 60560872, 62084911,
                                    59885092, 56663531, 54555046, 58471833 /* + 500-550 bin */};
static const double HIST_R250_LAST = 83776;

static int draw_hist(rng_t* r, const double* w, int nb, double last, double lo, double width) {
    double tot = last;
    for (int b = 0; b < nb; ++b) tot += w[b];
    double u = rng_unif(r) * tot;
    int b = 0;
    for (; b < nb; ++b) {
        if (u < w[b]) break;
        u -= w[b];
    }
    /* b == nb selects the trailing bin (weight `last`) */
    int base = (int)(lo + b * width);
    return (int)rng_int(r, base, base + (int)width - 1);
}

static void config_profile(int cfg, int component, profile_t* p) {
    memset(p, 0, sizeof(*p));
    switch (cfg == 5 ? 50 + component : cfg) {
    case 1: /* 1,000 pairs; qlen 150; tlen U{150..250}; 4% sub, 0.5% ins, 0.5% del, ell 1 */
        *p = (profile_t){QD_UNIFORM, 150, 150, TD_ABS_UNIFORM, 150, 250, 0.04, 0.005, 0.005, 1, 1};
        break;
    case 2: /* 1M pairs; qlen 150; tlen 250; 2% sub; 0.1% ins/del, ell U{1..3} */
        *p = (profile_t){QD_UNIFORM, 150, 150, TD_ABS_UNIFORM, 250, 250, 0.02, 0.001, 0.001, 1, 3};
        break;
    case 3: case 51: /* 500k; qlen log-uniform [100,1000); tlen U{qlen..min(1000,1.5 qlen)} */
        *p = (profile_t){QD_LOGUNIFORM, 100, 1000, TD_QLEN_TO_1P5, 0, 1000, 0.02, 0.001, 0.001, 1, 3};
        break;
    case 4: case 52: /* 100k; qlen U{1000..10000}; tlen = consumed + U{0..500}; 5/5/5%, ell 1 */
        *p = (profile_t){QD_UNIFORM, 1000, 10000, TD_FLANK, 0, 500, 0.05, 0.05, 0.05, 1, 1};
        break;
    case 50: /* dataset-A-like: Fig. 3 histograms, tlen >= qlen, errors as config 2 */
        *p = (profile_t){QD_HIST_Q250, 0, 0, TD_HIST_R250, 0, 0, 0.02, 0.001, 0.001, 1, 3};
        break;
    default: /* unknown: behave as config 1 */
        *p = (profile_t){QD_UNIFORM, 150, 150, TD_ABS_UNIFORM, 150, 250, 0.04, 0.005, 0.005, 1, 1};
    }
}

/* config 5 component of pair k: 90% A-like, 9.9% config-3-like, 0.1% config-4-like.
 * grouped != 0 makes components contiguous (worst case for a length-oblivious split). */
static int config5_component(rng_t* r, int64_t k, int64_t n_total, int grouped) {
    if (grouped) {
        int64_t a = (n_total * 900) / 1000, b = (n_total * 999) / 1000;
        return k < a ? 0 : (k < b ? 1 : 2);
    }
    double u = rng_unif(r);
    return u < 0.9 ? 0 : (u < 0.999 ? 1 : 2);
}

typedef struct {
    int32_t qlen, tlen, h0, left_flank, consumed;
} pair_shape_t;

/* Simulate pair k.  When q/t are NULL only the shape is produced; both passes consume the RNG
 * streams identically so the shape and the bases always agree. */
static void simulate_pair(int cfg, uint64_t seed, int64_t k, int64_t n_total, int grouped, double p_n,
                          pair_shape_t* sh, uint8_t* q, uint8_t* t) {
    static const char B[4] = {'A', 'C', 'G', 'T'};
    uint64_t s0 = sm_mix(seed ^ ((uint64_t)cfg << 56) ^ (uint64_t)k);
    rng_t meta = {sm_mix(s0 ^ 0x1111)}, mut = {sm_mix(s0 ^ 0x2222)}, src = {sm_mix(s0 ^ 0x3333)},
          flank = {sm_mix(s0 ^ 0x4444)}, nrng = {sm_mix(s0 ^ 0x5555)};
    int comp = (cfg == 5) ? config5_component(&meta, k, n_total, grouped) : 0;
    profile_t p;
    config_profile(cfg, comp, &p);

    int qlen;
    if (p.qdist == QD_UNIFORM) qlen = (int)rng_int(&meta, p.qlo, p.qhi);
    else if (p.qdist == QD_LOGUNIFORM) {
        double u = rng_unif(&meta);
        qlen = (int)floor(exp(log((double)p.qlo) + u * (log((double)p.qhi) - log((double)p.qlo))));
    } else qlen = draw_hist(&meta, HIST_Q250, 10, 0.0, HIST_Q250_LO, HIST_Q250_W);
    if (qlen < 1) qlen = 1;

    int tnom = 0, flank_total_fixed = -1;
    switch (p.tdist) {
    case TD_ABS_UNIFORM: tnom = (int)rng_int(&meta, p.tlo, p.thi); break;
    case TD_QLEN_TO_1P5: {
        int hi = (int)floor(1.5 * qlen);
        if (hi > p.thi) hi = p.thi;
        if (hi < qlen) hi = qlen;
        tnom = (int)rng_int(&meta, qlen, hi);
        break;
    }
    case TD_FLANK: flank_total_fixed = (int)rng_int(&meta, p.tlo, p.thi); break;
    case TD_HIST_R250: {
        tnom = draw_hist(&meta, HIST_R250, 9, HIST_R250_LAST, HIST_R250_LO, HIST_R250_W);
        if (tnom < qlen) tnom = qlen;
        break;
    }
    }
    int h0 = 19 + (int)rng_int(&meta, 0, 31); /* BWA minimum seed length 19 x match 1 (§8(d)) */

    /* walk the source window */
    int qi = 0, consumed = 0;
    while (qi < qlen) {
        double u = rng_unif(&mut);
        if (u < p.p_ins) {
            int L = (int)rng_int(&mut, p.ell_lo, p.ell_hi);
            for (int x = 0; x < L && qi < qlen; ++x) {
                int b = (int)(rng_next(&mut) & 3);
                if (q) q[qi] = (uint8_t)B[b];
                ++qi;
            }
        } else if (u < p.p_ins + p.p_del) {
            int L = (int)rng_int(&mut, p.ell_lo, p.ell_hi);
            for (int x = 0; x < L; ++x) {
                int b = (int)(rng_next(&src) & 3);
                if (t) t[consumed] = (uint8_t)B[b]; /* written after the left flank shift below */
                ++consumed;
            }
        } else {
            int b = (int)(rng_next(&src) & 3);
            if (t) t[consumed] = (uint8_t)B[b];
            ++consumed;
            if (rng_unif(&mut) < p.p_sub) b = (b + 1 + (int)rng_int(&mut, 0, 2)) & 3;
            if (q) q[qi] = (uint8_t)B[b];
            ++qi;
        }
    }
    int flank_total = flank_total_fixed >= 0 ? flank_total_fixed : (tnom > consumed ? tnom - consumed : 0);
    int left = (int)rng_int(&flank, 0, flank_total);
    int tlen = consumed + flank_total;
    if (t) {
        /* t[0..consumed) holds the source window; shift it right by `left` and fill flanks */
        memmove(t + left, t, (size_t)consumed);
        for (int x = 0; x < left; ++x) t[x] = (uint8_t)B[rng_next(&flank) & 3];
        for (int x = left + consumed; x < tlen; ++x) t[x] = (uint8_t)B[rng_next(&flank) & 3];
        if (p_n > 0) {
            for (int x = 0; x < qlen; ++x) if (rng_unif(&nrng) < p_n) q[x] = 'N';
            for (int x = 0; x < tlen; ++x) if (rng_unif(&nrng) < p_n) t[x] = 'N';
        }
    }
    sh->qlen = qlen;
    sh->tlen = tlen;
    sh->h0 = h0;
    sh->left_flank = left;
    sh->consumed = consumed;
}

/* ---- threaded drivers ------------------------------------------------------------------- */
typedef struct {
    int cfg, grouped;
    uint64_t seed;
    int64_t first, n, n_total, lo, hi;
    double p_n;
    int32_t *qlen, *tlen, *h0;
    const int64_t *q_off, *t_off;
    uint8_t *q, *t;
    const int64_t* idx; /* optional: global pair index of output i (else first + i) */
} job_t;

static inline int64_t pair_index(const job_t* j, int64_t i) { return j->idx ? j->idx[i] : j->first + i; }

static void* len_worker(void* arg) {
    job_t* j = (job_t*)arg;
    for (int64_t i = j->lo; i < j->hi; ++i) {
        pair_shape_t sh;
        simulate_pair(j->cfg, j->seed, pair_index(j, i), j->n_total, j->grouped, j->p_n, &sh, NULL, NULL);
        j->qlen[i] = sh.qlen;
        j->tlen[i] = sh.tlen;
        if (j->h0) j->h0[i] = sh.h0;
    }
    return NULL;
}
static void* base_worker(void* arg) {
    job_t* j = (job_t*)arg;
    for (int64_t i = j->lo; i < j->hi; ++i) {
        pair_shape_t sh;
        simulate_pair(j->cfg, j->seed, pair_index(j, i), j->n_total, j->grouped, j->p_n, &sh,
                      j->q + j->q_off[i], j->t + j->t_off[i]);
    }
    return NULL;
}
static void run_jobs(job_t proto, int n_threads, void* (*fn)(void*)) {
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    if ((int64_t)n_threads > proto.n) n_threads = proto.n > 0 ? (int)proto.n : 1;
    pthread_t th[256];
    job_t jobs[256];
    for (int k = 0; k < n_threads; ++k) {
        jobs[k] = proto;
        jobs[k].lo = proto.n * k / n_threads;
        jobs[k].hi = proto.n * (k + 1) / n_threads;
        pthread_create(&th[k], NULL, fn, &jobs[k]);
    }
    for (int k = 0; k < n_threads; ++k) pthread_join(th[k], NULL);
}

/* Shapes of pairs [first, first+n) of a batch of n_total pairs (n_total matters only for the
 * grouped config-5 order).  h0 may be NULL. Returns 0. */
EXPORT int synth_lengths(int cfg, uint64_t seed, int64_t first, int64_t n, int64_t n_total, int grouped,
                         int32_t* qlen, int32_t* tlen, int32_t* h0, int n_threads) {
    job_t j = {cfg, grouped, seed, first, n, n_total, 0, 0, 0.0, qlen, tlen, h0, NULL, NULL, NULL, NULL, NULL};
    run_jobs(j, n_threads, len_worker);
    return 0;
}

/* As synth_lengths / synth_bases for an explicit list of global pair indices idx[0..n) (a rank's
 * shard of a partitioned batch): output i is pair idx[i] of the n_total-pair batch. */
EXPORT int synth_lengths_idx(int cfg, uint64_t seed, const int64_t* idx, int64_t n, int64_t n_total, int grouped,
                             int32_t* qlen, int32_t* tlen, int32_t* h0, int n_threads) {
    job_t j = {cfg, grouped, seed, 0, n, n_total, 0, 0, 0.0, qlen, tlen, h0, NULL, NULL, NULL, NULL, idx};
    run_jobs(j, n_threads, len_worker);
    return 0;
}
EXPORT int synth_bases_idx(int cfg, uint64_t seed, const int64_t* idx, int64_t n, int64_t n_total, int grouped,
                           double p_n, const int64_t* q_off, const int64_t* t_off, uint8_t* q_ascii, uint8_t* t_ascii,
                           int n_threads) {
    job_t j = {cfg, grouped, seed, 0, n, n_total, 0, 0, p_n, NULL, NULL, NULL, q_off, t_off, q_ascii, t_ascii, idx};
    run_jobs(j, n_threads, base_worker);
    return 0;
}

/* Bases of the same pairs into caller buffers at the given byte offsets (uppercase ASCII). */
EXPORT int synth_bases(int cfg, uint64_t seed, int64_t first, int64_t n, int64_t n_total, int grouped,
                       double p_n, const int64_t* q_off, const int64_t* t_off, uint8_t* q_ascii,
                       uint8_t* t_ascii, int n_threads) {
    job_t j = {cfg, grouped, seed, first, n, n_total, 0, 0, p_n, NULL, NULL, NULL, q_off, t_off, q_ascii, t_ascii, NULL};
    run_jobs(j, n_threads, base_worker);
    return 0;
}
