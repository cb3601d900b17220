/*
 * oracle.c — CPU oracle for batched affine-gap (Gotoh) seed extension.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load or execute this code.  The product (CUDA) path never links,
 * imports or calls it, and it shares no code, header, table or helper with the product.
 *
 * It is the plain definition, written out: a full (m+1) x (n+1) int32 matrix for each of H, E, F,
 * filled cell by cell in row-major order, followed by a row-major scan for the best cell.
 *
 *   Rows i = target ("reference at i"), 0..m-1; columns j = query, 0..n-1.
 *   Out-of-table cells (row -1, column -1) are the boundary.
 *
 * LOCAL (Eqs. 1-3; SPEC.md S:132-140 cell_update, S:377-391 oracle_align):
 *   E(i,j) = max(0, H(i,j-1) - alpha, E(i,j-1) - beta)              (Eq. 2, clamped: S:135)
 *   F(i,j) = max(0, H(i-1,j) - alpha, F(i-1,j) - beta)              (Eq. 3, clamped)
 *   H(i,j) = max(0, E(i,j), F(i,j), H(i-1,j-1) + S(t_i, q_j))       (Eq. 1)
 *   boundary H = E = F = 0
 *   score = max H; end = smallest (i, j) in row-major order with H = score; (0,0) when score = 0
 *
 * EXTEND (seed-anchored; SURVEY §8(c) reading 7, listed in DESIGN.md):
 *   H(-1,-1) = h0;  H(-1,j) = max(0, h0 - alpha - beta*j);  H(i,-1) = max(0, h0 - alpha - beta*i)
 *   E(i,-1) = F(-1,j) = 0;  E, F as in LOCAL;
 *   D(i,j) = H(i-1,j-1) + S  if H(i-1,j-1) > 0, else 0   ("dead-zero": no fresh local starts)
 *   H(i,j) = max(0, E, F, D)
 *   score = max(h0, max H); end = smallest (i,j) with H = score, the anchor (-1,-1) ranked first.
 *
 * S(t, q) = match if t == q and t != N, else mismatch (N never matches, N-N included: S:123-131).
 * Base codes (oracle's own table): A/a=0 C/c=1 G/g=2 T/t/U/u=3 N/n=4; others invalid.
 *
 * BANDED (reading 16; PAPER.md P:1728-1735 names banded DP only as
 * future work): a per-pair band w >= 0 keeps the cells with |i - j| <= w (the diagonal through the
 * anchor / the table origin, as BWA-MEM's ksw_extend band).  Cells outside the band are not part
 * of the table: they read as H = E = F = 0, exactly like the out-of-table boundary cells of
 * LOCAL, and can never be the best cell.  Boundary row/column values (EXTEND) are unchanged.
 *
 * START coordinates (LOCAL only, reading 15 — the paper defines no
 * start): with (t_end, q_end) chosen by the tie rule above, align the reversed prefixes
 * t' = t[t_end] t[t_end-1] .. t[0] and q' = q[q_end] .. q[0] in LOCAL mode; its end (i', j') by the
 * same tie rule gives t_start = t_end - i', q_start = q_end - j' (the first aligned column of an
 * optimal alignment ending at the end cell; among those, the largest t_start, then the largest
 * q_start).  score 0: start = (0, 0), like the end.
 *
 * Two entry points compute the same thing: oracle_align_full (the definition above, full
 * matrices, guarded at ORACLE_FULL_MAX_CELLS) and oracle_align_rows (the identical loop keeping
 * only rows i-1 and i; used for long pairs; cross-checked against the full one in tests).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

enum { OR_LOCAL = 0, OR_EXTEND = 1 };
enum { OR_OK = 0, OR_EINVALID_BASE = -1, OR_EEMPTY = -2, OR_ETOO_LARGE = -3, OR_EBAD_H0 = -4, OR_ENOMEM = -5, OR_EBAD_BAND = -6 };

#define ORACLE_FULL_MAX_CELLS (1LL << 26)

static int code_of(uint8_t c) {
    switch (c) {
    case 'A': case 'a': return 0;
    case 'C': case 'c': return 1;
    case 'G': case 'g': return 2;
    case 'T': case 't': case 'U': case 'u': return 3;
    case 'N': case 'n': return 4;
    default: return -1;
    }
}

static inline int32_t imax(int32_t a, int32_t b) { return a > b ? a : b; }

static inline int32_t subst(int tc, int qc, int32_t match, int32_t mismatch) {
    return (tc == qc && tc != 4) ? match : mismatch;
}

/* encode both sequences; returns status */
static int encode(const uint8_t* s, int len, int8_t* out) {
    for (int k = 0; k < len; ++k) {
        int c = code_of(s[k]);
        if (c < 0) return OR_EINVALID_BASE;
        out[k] = (int8_t)c;
    }
    return OR_OK;
}

static int check(int n, int m, int mode, int32_t h0) {
    if (n < 1 || m < 1) return OR_EEMPTY;
    if (mode == OR_EXTEND && h0 < 1) return OR_EBAD_H0;
    return OR_OK;
}

/* ---- full-matrix definition ---------------------------------------------------------------- */
/* H, E, F: caller buffers of (m+1)*(n+1) int32 (may be NULL: allocated here). */
static int align_full_impl(const int8_t* qc, int n, const int8_t* tc, int m, int32_t match,
                           int32_t mismatch, int32_t alpha, int32_t beta, int mode, int32_t h0,
                           int32_t* H, int32_t* E, int32_t* F, int32_t out[3]) {
    const long W = n + 1;
#define AT(X, i, j) X[((long)(i) + 1) * W + ((long)(j) + 1)]
    /* boundary row -1 (including the corner) and column -1 */
    for (int j = -1; j < n; ++j) {
        int32_t b = 0;
        if (mode == OR_EXTEND) b = (j == -1) ? h0 : imax(0, h0 - alpha - beta * j);
        AT(H, -1, j) = b;
        AT(E, -1, j) = 0;
        AT(F, -1, j) = 0;
    }
    for (int i = 0; i < m; ++i) {
        AT(H, i, -1) = (mode == OR_EXTEND) ? imax(0, h0 - alpha - beta * i) : 0;
        AT(E, i, -1) = 0;
        AT(F, i, -1) = 0;
    }
    /* Eqs. 1-3, row-major */
    for (int i = 0; i < m; ++i) {
        for (int j = 0; j < n; ++j) {
            int32_t e = imax(0, imax(AT(H, i, j - 1) - alpha, AT(E, i, j - 1) - beta));
            int32_t f = imax(0, imax(AT(H, i - 1, j) - alpha, AT(F, i - 1, j) - beta));
            int32_t hd = AT(H, i - 1, j - 1);
            int32_t d;
            if (mode == OR_LOCAL || hd > 0) d = hd + subst(tc[i], qc[j], match, mismatch);
            else d = 0;
            int32_t h = imax(imax(0, e), imax(f, d));
            AT(E, i, j) = e;
            AT(F, i, j) = f;
            AT(H, i, j) = h;
        }
    }
    /* best cell: strict '>' in row-major order = max score, then smallest i, then smallest j */
    int32_t best = (mode == OR_EXTEND) ? h0 : 0;
    int32_t bi = (mode == OR_EXTEND) ? -1 : 0, bj = (mode == OR_EXTEND) ? -1 : 0;
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j)
            if (AT(H, i, j) > best) {
                best = AT(H, i, j);
                bi = i;
                bj = j;
            }
#undef AT
    out[0] = best;
    out[1] = bj; /* q_end */
    out[2] = bi; /* t_end */
    return OR_OK;
}

/* ---- banded: the same definition with the cells |i - j| > w forced to zero ------------------ */
static int align_banded_impl(const int8_t* qc, int n, const int8_t* tc, int m, int32_t match, int32_t mismatch,
                             int32_t alpha, int32_t beta, int mode, int32_t h0, int32_t w, int32_t out[3]) {
    const long W = n + 1;
    int32_t* H = (int32_t*)malloc(3 * (size_t)(m + 1) * (size_t)W * sizeof(int32_t));
    if (!H) return OR_ENOMEM;
    int32_t* E = H + (size_t)(m + 1) * W;
    int32_t* F = E + (size_t)(m + 1) * W;
#define AT(X, i, j) X[((long)(i) + 1) * W + ((long)(j) + 1)]
    for (int j = -1; j < n; ++j) {
        AT(H, -1, j) = (mode == OR_EXTEND) ? ((j == -1) ? h0 : imax(0, h0 - alpha - beta * j)) : 0;
        AT(E, -1, j) = 0;
        AT(F, -1, j) = 0;
    }
    for (int i = 0; i < m; ++i) {
        AT(H, i, -1) = (mode == OR_EXTEND) ? imax(0, h0 - alpha - beta * i) : 0;
        AT(E, i, -1) = 0;
        AT(F, i, -1) = 0;
    }
    for (int i = 0; i < m; ++i) {
        for (int j = 0; j < n; ++j) {
            if (i - j > w || j - i > w) { /* outside the band: not part of the table */
                AT(E, i, j) = 0;
                AT(F, i, j) = 0;
                AT(H, i, j) = 0;
                continue;
            }
            int32_t e = imax(0, imax(AT(H, i, j - 1) - alpha, AT(E, i, j - 1) - beta));
            int32_t f = imax(0, imax(AT(H, i - 1, j) - alpha, AT(F, i - 1, j) - beta));
            int32_t hd = AT(H, i - 1, j - 1);
            int32_t d;
            if (mode == OR_LOCAL || hd > 0) d = hd + subst(tc[i], qc[j], match, mismatch);
            else d = 0;
            AT(E, i, j) = e;
            AT(F, i, j) = f;
            AT(H, i, j) = imax(imax(0, e), imax(f, d));
        }
    }
    int32_t best = (mode == OR_EXTEND) ? h0 : 0;
    int32_t bi = (mode == OR_EXTEND) ? -1 : 0, bj = (mode == OR_EXTEND) ? -1 : 0;
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j)
            if (AT(H, i, j) > best) {
                best = AT(H, i, j);
                bi = i;
                bj = j;
            }
#undef AT
    free(H);
    out[0] = best;
    out[1] = bj;
    out[2] = bi;
    return OR_OK;
}

/* ---- the same recurrence keeping two rows ---------------------------------------------------- */
static int align_rows_impl(const int8_t* qc, int n, const int8_t* tc, int m, int32_t match,
                           int32_t mismatch, int32_t alpha, int32_t beta, int mode, int32_t h0,
                           int32_t* rowbuf /* 6*(n+1) */, int32_t out[3]) {
    const long W = n + 1;
    int32_t *Hp = rowbuf, *Fp = rowbuf + W, *Hc = rowbuf + 2 * W, *Fc = rowbuf + 3 * W;
    /* previous row = row -1 */
    for (int j = -1; j < n; ++j) {
        Hp[j + 1] = (mode == OR_EXTEND) ? ((j == -1) ? h0 : imax(0, h0 - alpha - beta * j)) : 0;
        Fp[j + 1] = 0;
    }
    int32_t best = (mode == OR_EXTEND) ? h0 : 0;
    int32_t bi = (mode == OR_EXTEND) ? -1 : 0, bj = (mode == OR_EXTEND) ? -1 : 0;
    for (int i = 0; i < m; ++i) {
        Hc[0] = (mode == OR_EXTEND) ? imax(0, h0 - alpha - beta * i) : 0;
        Fc[0] = 0;
        int32_t e_left = 0; /* E(i,-1) */
        for (int j = 0; j < n; ++j) {
            int32_t e = imax(0, imax(Hc[j] - alpha, e_left - beta));
            int32_t f = imax(0, imax(Hp[j + 1] - alpha, Fp[j + 1] - beta));
            int32_t hd = Hp[j];
            int32_t d;
            if (mode == OR_LOCAL || hd > 0) d = hd + subst(tc[i], qc[j], match, mismatch);
            else d = 0;
            int32_t h = imax(imax(0, e), imax(f, d));
            Hc[j + 1] = h;
            Fc[j + 1] = f;
            e_left = e;
            if (h > best) {
                best = h;
                bi = i;
                bj = j;
            }
        }
        int32_t* t = Hp; Hp = Hc; Hc = t;
        t = Fp; Fp = Fc; Fc = t;
    }
    out[0] = best;
    out[1] = bj;
    out[2] = bi;
    return OR_OK;
}

static int prepare(const uint8_t* q, int n, const uint8_t* t, int m, int mode, int32_t h0, int8_t** qc,
                   int8_t** tc) {
    int st = check(n, m, mode, h0);
    if (st) return st;
    *qc = (int8_t*)malloc((size_t)n);
    *tc = (int8_t*)malloc((size_t)m);
    if (!*qc || !*tc) return OR_ENOMEM;
    if (encode(q, n, *qc) || encode(t, m, *tc)) return OR_EINVALID_BASE;
    return OR_OK;
}

/* out = {score, q_end, t_end}.  Returns OR_OK or a negative status. */
EXPORT int oracle_align_full(const uint8_t* q, int n, const uint8_t* t, int m, int32_t match, int32_t mismatch,
                             int32_t alpha, int32_t beta, int mode, int32_t h0, int32_t out[3]) {
    int8_t *qc = NULL, *tc = NULL;
    int st = prepare(q, n, t, m, mode, h0, &qc, &tc);
    if (st == OR_OK && (long long)(m + 1) * (n + 1) > ORACLE_FULL_MAX_CELLS) st = OR_ETOO_LARGE;
    if (st == OR_OK) {
        size_t cells = (size_t)(m + 1) * (size_t)(n + 1);
        int32_t* buf = (int32_t*)malloc(3 * cells * sizeof(int32_t));
        if (!buf) st = OR_ENOMEM;
        else {
            st = align_full_impl(qc, n, tc, m, match, mismatch, alpha, beta, mode, h0, buf, buf + cells,
                                 buf + 2 * cells, out);
            free(buf);
        }
    }
    free(qc);
    free(tc);
    return st;
}

/* Full H/E/F tables for tests: each of size (m+1)*(n+1), row -1 / column -1 included. */
EXPORT int oracle_tables(const uint8_t* q, int n, const uint8_t* t, int m, int32_t match, int32_t mismatch,
                         int32_t alpha, int32_t beta, int mode, int32_t h0, int32_t* H, int32_t* E, int32_t* F,
                         int32_t out[3]) {
    int8_t *qc = NULL, *tc = NULL;
    int st = prepare(q, n, t, m, mode, h0, &qc, &tc);
    if (st == OR_OK)
        st = align_full_impl(qc, n, tc, m, match, mismatch, alpha, beta, mode, h0, H, E, F, out);
    free(qc);
    free(tc);
    return st;
}

EXPORT int oracle_align_rows(const uint8_t* q, int n, const uint8_t* t, int m, int32_t match, int32_t mismatch,
                             int32_t alpha, int32_t beta, int mode, int32_t h0, int32_t out[3]) {
    int8_t *qc = NULL, *tc = NULL;
    int st = prepare(q, n, t, m, mode, h0, &qc, &tc);
    if (st == OR_OK) {
        int32_t* rows = (int32_t*)malloc(6 * (size_t)(n + 1) * sizeof(int32_t));
        if (!rows) st = OR_ENOMEM;
        else {
            st = align_rows_impl(qc, n, tc, m, match, mismatch, alpha, beta, mode, h0, rows, out);
            free(rows);
        }
    }
    free(qc);
    free(tc);
    return st;
}

/* Banded alignment of one pair (w >= 0).  out = {score, q_end, t_end}. */
EXPORT int oracle_align_banded(const uint8_t* q, int n, const uint8_t* t, int m, int32_t match, int32_t mismatch,
                               int32_t alpha, int32_t beta, int mode, int32_t h0, int32_t w, int32_t out[3]) {
    int8_t *qc = NULL, *tc = NULL;
    int st = prepare(q, n, t, m, mode, h0, &qc, &tc);
    if (st == OR_OK && w < 0) st = OR_EBAD_BAND;
    if (st == OR_OK && (long long)(m + 1) * (n + 1) > ORACLE_FULL_MAX_CELLS) st = OR_ETOO_LARGE;
    if (st == OR_OK) st = align_banded_impl(qc, n, tc, m, match, mismatch, alpha, beta, mode, h0, w, out);
    free(qc);
    free(tc);
    return st;
}

typedef struct {
    const uint8_t *q, *t;
    const int64_t *q_off, *t_off;
    const int32_t *h0, *w;
    int64_t n;
    int32_t match, mismatch, alpha, beta;
    int mode;
    int32_t *score, *q_end, *t_end, *status;
    volatile int64_t next;
} banded_batch_t;

static void* banded_worker(void* arg) {
    banded_batch_t* b = (banded_batch_t*)arg;
    for (;;) {
        int64_t k0 = __atomic_fetch_add(&b->next, 16, __ATOMIC_RELAXED);
        if (k0 >= b->n) break;
        int64_t k1 = k0 + 16 < b->n ? k0 + 16 : b->n;
        for (int64_t k = k0; k < k1; ++k) {
            int n = (int)(b->q_off[k + 1] - b->q_off[k]), m = (int)(b->t_off[k + 1] - b->t_off[k]);
            int32_t out[3] = {-1, -2, -2};
            int st = oracle_align_banded(b->q + b->q_off[k], n, b->t + b->t_off[k], m, b->match, b->mismatch,
                                         b->alpha, b->beta, b->mode, b->h0 ? b->h0[k] : 0, b->w[k], out);
            if (st) out[0] = -1, out[1] = -2, out[2] = -2;
            b->score[k] = out[0];
            b->q_end[k] = out[1];
            b->t_end[k] = out[2];
            if (b->status) b->status[k] = st;
        }
    }
    return NULL;
}

EXPORT int oracle_banded_batch(const uint8_t* q, const int64_t* q_off, const uint8_t* t, const int64_t* t_off,
                               const int32_t* h0, const int32_t* w, int64_t n, int32_t match, int32_t mismatch,
                               int32_t alpha, int32_t beta, int mode, int32_t* score, int32_t* q_end,
                               int32_t* t_end, int32_t* status, int n_threads) {
    banded_batch_t b = {q, t, q_off, t_off, h0, w, n, match, mismatch, alpha, beta, mode,
                        score, q_end, t_end, status, 0};
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 512) n_threads = 512;
    pthread_t th[512];
    for (int k = 0; k < n_threads; ++k) pthread_create(&th[k], NULL, banded_worker, &b);
    for (int k = 0; k < n_threads; ++k) pthread_join(th[k], NULL);
    return n_threads;
}

/* ---- start coordinates by the reverse DP (LOCAL) ------------------------------------------ */
/* out = {score, q_end, t_end, q_start, t_start}. */
EXPORT int oracle_start(const uint8_t* q, int n, const uint8_t* t, int m, int32_t match, int32_t mismatch,
                        int32_t alpha, int32_t beta, int32_t out[5]) {
    int8_t *qc = NULL, *tc = NULL;
    int st = prepare(q, n, t, m, OR_LOCAL, 0, &qc, &tc);
    int32_t* rows = NULL;
    int8_t *qr = NULL, *tr = NULL;
    if (st == OR_OK) {
        rows = (int32_t*)malloc(6 * (size_t)(n + 1) * sizeof(int32_t));
        qr = (int8_t*)malloc((size_t)n);
        tr = (int8_t*)malloc((size_t)m);
        if (!rows || !qr || !tr) st = OR_ENOMEM;
    }
    if (st == OR_OK) {
        int32_t fw[3], rv[3];
        align_rows_impl(qc, n, tc, m, match, mismatch, alpha, beta, OR_LOCAL, 0, rows, fw);
        out[0] = fw[0];
        out[1] = fw[1];
        out[2] = fw[2];
        out[3] = 0;
        out[4] = 0;
        if (fw[0] > 0) {
            const int qe = fw[1], te = fw[2];
            for (int j = 0; j <= qe; ++j) qr[j] = qc[qe - j];
            for (int i = 0; i <= te; ++i) tr[i] = tc[te - i];
            align_rows_impl(qr, qe + 1, tr, te + 1, match, mismatch, alpha, beta, OR_LOCAL, 0, rows, rv);
            out[3] = qe - rv[1];
            out[4] = te - rv[2];
        }
    }
    free(rows);
    free(qr);
    free(tr);
    free(qc);
    free(tc);
    return st;
}

/* Batch form: q_start / t_start of every pair (LOCAL), pthreads over pairs. */
typedef struct {
    const uint8_t *q, *t;
    const int64_t *q_off, *t_off;
    int64_t n;
    int32_t match, mismatch, alpha, beta;
    int32_t *score, *q_end, *t_end, *q_start, *t_start, *status;
    volatile int64_t next;
} start_batch_t;

static void* start_worker(void* arg) {
    start_batch_t* b = (start_batch_t*)arg;
    for (;;) {
        int64_t k0 = __atomic_fetch_add(&b->next, 16, __ATOMIC_RELAXED);
        if (k0 >= b->n) break;
        int64_t k1 = k0 + 16 < b->n ? k0 + 16 : b->n;
        for (int64_t k = k0; k < k1; ++k) {
            int n = (int)(b->q_off[k + 1] - b->q_off[k]), m = (int)(b->t_off[k + 1] - b->t_off[k]);
            int32_t out[5] = {-1, -2, -2, -2, -2};
            int st = oracle_start(b->q + b->q_off[k], n, b->t + b->t_off[k], m, b->match, b->mismatch, b->alpha,
                                  b->beta, out);
            if (st) out[0] = -1, out[1] = out[2] = out[3] = out[4] = -2;
            b->score[k] = out[0];
            b->q_end[k] = out[1];
            b->t_end[k] = out[2];
            b->q_start[k] = out[3];
            b->t_start[k] = out[4];
            if (b->status) b->status[k] = st;
        }
    }
    return NULL;
}

EXPORT int oracle_start_batch(const uint8_t* q, const int64_t* q_off, const uint8_t* t, const int64_t* t_off,
                              int64_t n, int32_t match, int32_t mismatch, int32_t alpha, int32_t beta,
                              int32_t* score, int32_t* q_end, int32_t* t_end, int32_t* q_start, int32_t* t_start,
                              int32_t* status, int n_threads) {
    start_batch_t b = {q, t, q_off, t_off, n, match, mismatch, alpha, beta,
                       score, q_end, t_end, q_start, t_start, status, 0};
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 512) n_threads = 512;
    pthread_t th[512];
    for (int k = 0; k < n_threads; ++k) pthread_create(&th[k], NULL, start_worker, &b);
    for (int k = 0; k < n_threads; ++k) pthread_join(th[k], NULL);
    return n_threads;
}

/* ---- batch driver: pthreads, dynamic pair scheduling ------------------------------------------ */
typedef struct {
    const uint8_t *q, *t;
    const int64_t *q_off, *t_off;
    const int32_t* h0;
    int64_t n;
    int32_t match, mismatch, alpha, beta;
    int mode;
    int force_rows;
    int32_t *score, *q_end, *t_end, *status;
    volatile int64_t next;
} batch_t;

static void* batch_worker(void* arg) {
    batch_t* b = (batch_t*)arg;
    for (;;) {
        int64_t k0 = __atomic_fetch_add(&b->next, 16, __ATOMIC_RELAXED);
        if (k0 >= b->n) break;
        int64_t k1 = k0 + 16 < b->n ? k0 + 16 : b->n;
        for (int64_t k = k0; k < k1; ++k) {
            int n = (int)(b->q_off[k + 1] - b->q_off[k]), m = (int)(b->t_off[k + 1] - b->t_off[k]);
            int32_t out[3] = {-1, -2, -2};
            int32_t h0 = b->h0 ? b->h0[k] : 0;
            int st;
            if (!b->force_rows && (long long)(m + 1) * (n + 1) <= (1LL << 22))
                st = oracle_align_full(b->q + b->q_off[k], n, b->t + b->t_off[k], m, b->match, b->mismatch,
                                       b->alpha, b->beta, b->mode, h0, out);
            else
                st = oracle_align_rows(b->q + b->q_off[k], n, b->t + b->t_off[k], m, b->match, b->mismatch,
                                       b->alpha, b->beta, b->mode, h0, out);
            if (st) out[0] = -1, out[1] = -2, out[2] = -2;
            b->score[k] = out[0];
            b->q_end[k] = out[1];
            b->t_end[k] = out[2];
            if (b->status) b->status[k] = st;
        }
    }
    return NULL;
}

/* Align pairs k = 0..n-1 (query k = q[q_off[k] .. q_off[k+1]), likewise target).  Pairs with
 * (m+1)(n+1) <= 2^22 use the full-matrix definition, longer ones the two-row form (or all pairs
 * with force_rows).  Per-pair status (may be NULL). Returns the number of threads used. */
EXPORT int oracle_align_batch(const uint8_t* q, const int64_t* q_off, const uint8_t* t, const int64_t* t_off,
                              const int32_t* h0, int64_t n, int32_t match, int32_t mismatch, int32_t alpha,
                              int32_t beta, int mode, int32_t* score, int32_t* q_end, int32_t* t_end,
                              int32_t* status, int n_threads, int force_rows) {
    batch_t b = {q, t, q_off, t_off, h0, n, match, mismatch, alpha, beta, mode, force_rows,
                 score, q_end, t_end, status, 0};
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 512) n_threads = 512;
    pthread_t th[512];
    for (int k = 0; k < n_threads; ++k) pthread_create(&th[k], NULL, batch_worker, &b);
    for (int k = 0; k < n_threads; ++k) pthread_join(th[k], NULL);
    return n_threads;
}
