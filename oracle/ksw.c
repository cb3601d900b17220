/*
 * ksw.c — CPU oracle of the BWA-MEM-compatible seed extension.
 *
 * TEST INFRASTRUCTURE ONLY (same rules as oracle.c): only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it; the CUDA product shares nothing.
 *
 * PAPER.md does not define this operation: its real-world inputs are BWA-MEM seeds
 * and it notes the field "has grown to value quality over speed" with BWA-MEM the de facto
 * standard.  DESIGN.md reading 17 takes BWA-MEM's public extension algorithm
 * (ksw_extend2 of bwa's ksw.c) as the definition and restates it; this file follows it step by
 * step, in its order and notation:
 *
 *   scores  S(x,y) = a if x == y < 4; -b if x != y, both < 4; -1 if either is N   (bwa_fill_scmat)
 *   gaps    a deletion (target base, vertical) of length k costs o_del + k*e_del, an insertion
 *           (query base, horizontal) o_ins + k*e_ins; oe_del = o_del + e_del, oe_ins = o_ins + e_ins
 *   row -1  eh[0].h = h0; eh[j].h = max(0, h0 - oe_ins - (j-1)*e_ins) while the previous value
 *           exceeds e_ins (eh[j].h holds H(-1, j-1)); eh[j].e = 0
 *   band    w is lowered to max(1, (n*max_S + end_bonus - o_ins)/e_ins + 1) and to the same bound
 *           with (o_del, e_del); row i only covers columns [max(beg, i-w), min(end, i+w+1, n))
 *   row i   h1 = max(0, h0 - (o_del + e_del*(i+1))) if beg == 0 else 0;  f = 0;  for each column j:
 *             M = eh[j].h (= H(i-1,j-1)); e = eh[j].e (= E(i,j)); eh[j].h = h1 (= H(i,j-1))
 *             M = M ? M + S(t_i, q_j) : 0          (no fresh starts: a dead cell kills the diagonal)
 *             h = max(M, e, f); h1 = h;  row max m / its LAST column mj (ties -> larger j)
 *             eh[j].e = max(e - e_del, max(M - oe_del, 0))   (E(i+1,j): gaps open from M only)
 *             f       = max(f - e_ins, max(M - oe_ins, 0))   (F(i,j+1))
 *           eh[end].h = h1, eh[end].e = 0
 *           if end == n: gscore/max_ie take (h1, i) when h1 >= gscore (ties -> later row)
 *           if m == 0: stop
 *           if m > max: max = m, (max_i, max_j) = (i, mj), max_off = max(max_off, |mj - i|)
 *           else if zdrop > 0 and the drop max - m, less the gap-length term
 *             ((i - max_i) - (mj - max_j)) * e_del   (when i - max_i > mj - max_j), else
 *             ((mj - max_j) - (i - max_i)) * e_ins,  exceeds zdrop: stop
 *           beg = first j in [beg, end) whose (eh[j].h, eh[j].e) is not (0, 0);
 *           end = min(n, 2 + the last j in [beg, end] whose (eh[j].h, eh[j].e) is not (0, 0))
 *           (eh[] entries beyond end keep the values an earlier row left there — the next row may
 *           read one of them, exactly as ksw_extend2 does)
 *   result  score = max, qle = max_j + 1, tle = max_i + 1, gtle = max_ie + 1, gscore, max_off
 *           (qle = tle = 0 when no cell beats h0; gscore = -1 / gtle = 0 when no row reached n)
 *
 * The BWA-MEM caller then keeps the local extension (score, qle, tle) unless gscore > 0 and
 * gscore > score - end_bonus, in which case it takes the end-to-end one (gscore, n, gtle); that
 * choice is returned as `clip` (0: end-to-end, 1: local).
 *
 * KSW_NO_TRIM (flags bit 0, for the pins only): skip the beg/end update (every row spans the
 * band).  That is the plain recurrence the brute-force path enumeration of the tests checks.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

enum { KSW_OK = 0, KSW_EINVALID_BASE = -1, KSW_EEMPTY = -2, KSW_EBAD_H0 = -4, KSW_ENOMEM = -5, KSW_EBAD_PARAM = -7 };
enum { KSW_NO_TRIM = 1 };

static int ksw_code(uint8_t c) {
    switch (c) {
    case 'A': case 'a': return 0;
    case 'C': case 'c': return 1;
    case 'G': case 'g': return 2;
    case 'T': case 't': case 'U': case 'u': return 3;
    case 'N': case 'n': return 4;
    default: return -1;
    }
}

typedef struct {
    int32_t h, e;
} ksw_eh;

/* out[7]: score, qle, tle, gtle, gscore, max_off, clip.  htab (pins only, may be NULL): m*n int32,
 * H(i,j) of every computed cell, -1 elsewhere; rows after a stop stay -1. */
static int ksw_impl(const uint8_t* q, int n, const uint8_t* t, int m, int32_t a, int32_t b, int32_t o_del,
                    int32_t e_del, int32_t o_ins, int32_t e_ins, int32_t w, int32_t end_bonus, int32_t zdrop,
                    int32_t h0, int32_t flags, int32_t* out, int32_t* htab) {
    if (n < 1 || m < 1) return KSW_EEMPTY;
    if (h0 < 1) return KSW_EBAD_H0;
    if (a < 1 || b < 1 || o_del < 0 || e_del < 1 || o_ins < 0 || e_ins < 1 || w < 0 || end_bonus < 0)
        return KSW_EBAD_PARAM;
    int8_t* qc = (int8_t*)malloc((size_t)n);
    int8_t* tc = (int8_t*)malloc((size_t)m);
    ksw_eh* eh = (ksw_eh*)calloc((size_t)n + 1, sizeof(ksw_eh));
    if (!qc || !tc || !eh) {
        free(qc); free(tc); free(eh);
        return KSW_ENOMEM;
    }
    for (int k = 0; k < n; ++k) {
        const int c = ksw_code(q[k]);
        if (c < 0) { free(qc); free(tc); free(eh); return KSW_EINVALID_BASE; }
        qc[k] = (int8_t)c;
    }
    for (int k = 0; k < m; ++k) {
        const int c = ksw_code(t[k]);
        if (c < 0) { free(qc); free(tc); free(eh); return KSW_EINVALID_BASE; }
        tc[k] = (int8_t)c;
    }
    const int32_t oe_del = o_del + e_del, oe_ins = o_ins + e_ins;
    if (htab)
        for (int64_t k = 0; k < (int64_t)m * n; ++k) htab[k] = -1;
    /* row -1 */
    eh[0].h = h0;
    eh[1].h = h0 > oe_ins ? h0 - oe_ins : 0;
    for (int j = 2; j <= n && eh[j - 1].h > e_ins; ++j) eh[j].h = eh[j - 1].h - e_ins;
    /* band adjustment (max_S = a: the largest entry of the 5x5 matrix, since a >= 1 > -1) */
    int max_ins = (int)((double)(n * a + end_bonus - o_ins) / e_ins + 1.);
    if (max_ins < 1) max_ins = 1;
    if (w > max_ins) w = max_ins;
    int max_del = (int)((double)(n * a + end_bonus - o_del) / e_del + 1.);
    if (max_del < 1) max_del = 1;
    if (w > max_del) w = max_del;
    int32_t max = h0, max_i = -1, max_j = -1, max_ie = -1, gscore = -1, max_off = 0;
    int beg = 0, end = n;
    for (int i = 0; i < m; ++i) {
        int32_t f = 0, h1, mrow = 0;
        int mj = -1;
        if (flags & KSW_NO_TRIM) {  /* pins only: every row spans the band */
            beg = 0;
            end = n;
        }
        if (beg < i - w) beg = i - w;
        if (end > i + w + 1) end = i + w + 1;
        if (end > n) end = n;
        if (beg == 0) {
            h1 = h0 - (o_del + e_del * (i + 1));
            if (h1 < 0) h1 = 0;
        } else
            h1 = 0;
        int j;
        for (j = beg; j < end; ++j) {
            int32_t M = eh[j].h, e = eh[j].e;
            eh[j].h = h1;
            const int32_t s = (tc[i] == 4 || qc[j] == 4) ? -1 : (tc[i] == qc[j] ? a : -b);
            M = M ? M + s : 0;
            int32_t h = M > e ? M : e;
            h = h > f ? h : f;
            h1 = h;
            if (htab) htab[(int64_t)i * n + j] = h;
            mj = mrow > h ? mj : j;
            mrow = mrow > h ? mrow : h;
            int32_t tt = M - oe_del;
            tt = tt > 0 ? tt : 0;
            e -= e_del;
            e = e > tt ? e : tt;
            eh[j].e = e;
            tt = M - oe_ins;
            tt = tt > 0 ? tt : 0;
            f -= e_ins;
            f = f > tt ? f : tt;
        }
        eh[end].h = h1;
        eh[end].e = 0;
        if (j == n) {
            max_ie = gscore > h1 ? max_ie : i;
            gscore = gscore > h1 ? gscore : h1;
        }
        if (mrow == 0) break;
        if (mrow > max) {
            max = mrow;
            max_i = i;
            max_j = mj;
            const int off = mj > i ? mj - i : i - mj;
            max_off = max_off > off ? max_off : off;
        } else if (zdrop > 0) {
            if (i - max_i > mj - max_j) {
                if (max - mrow - ((i - max_i) - (mj - max_j)) * e_del > zdrop) break;
            } else {
                if (max - mrow - ((mj - max_j) - (i - max_i)) * e_ins > zdrop) break;
            }
        }
        if (!(flags & KSW_NO_TRIM)) {
            for (j = beg; j < end && eh[j].h == 0 && eh[j].e == 0; ++j) {
            }
            beg = j;
            for (j = end; j >= beg && eh[j].h == 0 && eh[j].e == 0; --j) {
            }
            end = j + 2 < n ? j + 2 : n;
        }
    }
    free(qc);
    free(tc);
    free(eh);
    out[0] = max;
    out[1] = max_j + 1;
    out[2] = max_i + 1;
    out[3] = max_ie + 1;
    out[4] = gscore;
    out[5] = max_off;
    out[6] = (gscore <= 0 || gscore <= max - end_bonus) ? 1 : 0;
    return KSW_OK;
}

EXPORT int oracle_ksw_extend(const uint8_t* q, int n, const uint8_t* t, int m, int32_t a, int32_t b, int32_t o_del,
                             int32_t e_del, int32_t o_ins, int32_t e_ins, int32_t w, int32_t end_bonus, int32_t zdrop,
                             int32_t h0, int32_t flags, int32_t* out) {
    return ksw_impl(q, n, t, m, a, b, o_del, e_del, o_ins, e_ins, w, end_bonus, zdrop, h0, flags, out, 0);
}

EXPORT int oracle_ksw_table(const uint8_t* q, int n, const uint8_t* t, int m, int32_t a, int32_t b, int32_t o_del,
                            int32_t e_del, int32_t o_ins, int32_t e_ins, int32_t w, int32_t end_bonus, int32_t zdrop,
                            int32_t h0, int32_t flags, int32_t* out, int32_t* htab) {
    return ksw_impl(q, n, t, m, a, b, o_del, e_del, o_ins, e_ins, w, end_bonus, zdrop, h0, flags, out, htab);
}

/* ---- batch over pairs (pthreads, dynamic index) ---------------------------------------------- */
typedef struct {
    const uint8_t *qa, *ta;
    const int64_t *qo, *to;
    const int32_t* h0;
    int64_t n;
    int32_t p[9]; /* a, b, o_del, e_del, o_ins, e_ins, w, end_bonus, zdrop */
    int32_t flags;
    int32_t* out; /* [7][n] */
    int32_t* status;
    volatile int64_t next;
} ksw_batch_t;

static void* ksw_worker(void* arg) {
    ksw_batch_t* B = (ksw_batch_t*)arg;
    for (;;) {
        const int64_t k = __sync_fetch_and_add(&B->next, 1);
        if (k >= B->n) break;
        int32_t r[7] = {0, 0, 0, 0, 0, 0, 0};
        const int st = oracle_ksw_extend(B->qa + B->qo[k], (int)(B->qo[k + 1] - B->qo[k]), B->ta + B->to[k],
                                         (int)(B->to[k + 1] - B->to[k]), B->p[0], B->p[1], B->p[2], B->p[3], B->p[4],
                                         B->p[5], B->p[6], B->p[7], B->p[8], B->h0[k], B->flags, r);
        for (int c = 0; c < 7; ++c) B->out[(int64_t)c * B->n + k] = st == KSW_OK ? r[c] : -1;
        B->status[k] = st;
    }
    return 0;
}

EXPORT int oracle_ksw_batch(const uint8_t* qa, const int64_t* qo, const uint8_t* ta, const int64_t* to,
                            const int32_t* h0, int64_t n, const int32_t* params /* 9 */, int32_t flags, int32_t* out,
                            int32_t* status, int threads) {
    ksw_batch_t B;
    B.qa = qa; B.ta = ta; B.qo = qo; B.to = to; B.h0 = h0; B.n = n; B.flags = flags; B.out = out; B.status = status;
    B.next = 0;
    memcpy(B.p, params, sizeof(B.p));
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    int started = 0;
    for (int i = 1; i < threads; ++i)
        if (pthread_create(&th[started], 0, ksw_worker, &B) == 0) ++started;
    ksw_worker(&B);
    for (int i = 0; i < started; ++i) pthread_join(th[i], 0);
    return started + 1;
}
