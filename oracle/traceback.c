/*
 * traceback.c — CPU oracle of the CIGAR traceback (reading 18).
 *
 * TEST INFRASTRUCTURE ONLY (same rules as oracle.c): only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it; the CUDA product shares nothing.
 *
 * The paper returns score and end coordinates only; SPEC puts traceback out of scope
 * (S:16).  Reading 18: the alignment of a LOCAL result is the global alignment of the
 * substrings t[t_start..t_end] x q[q_start..q_end] (start from reading 15, end from the tie rule),
 * under the same affine scheme (alpha = first gap base, beta = each further one), whose optimal
 * score equals the local score.  Among several optimal alignments one is chosen by tracing back
 * from the end cell with a fixed preference:
 *
 *   Gotoh, global, rows i = target, columns j = query, 0-based inside the substrings:
 *     H(-1,-1) = 0;  H(-1,j) = -(alpha + beta*j);  H(i,-1) = -(alpha + beta*i)
 *     E(i,j) = max(H(i,j-1) - alpha, E(i,j-1) - beta)      E(i,-1) = -inf   (insertion: query base)
 *     F(i,j) = max(H(i-1,j) - alpha, F(i-1,j) - beta)      F(-1,j) = -inf   (deletion: target base)
 *     H(i,j) = max(H(i-1,j-1) + S(t_i, q_j), E(i,j), F(i,j))
 *   The chosen alignment is the optimal one whose op string, read from the END, is smallest with
 *   M < D < I (match/mismatch first, then deletion = target base, then insertion = query base).
 *   Tracing back from (M-1, N-1) in state H, that is:
 *     H at (i,j):  'M' to (i-1,j-1) if H == H(i-1,j-1) + S;  else state F if H == F;  else state E
 *     E at (i,j):  'I'; to (i,j-1) in state H if E == H(i,j-1) - alpha, else in E (opening first is
 *                  never larger: the next op from H is then M or D, both < I)
 *     F at (i,j):  'D'; if only one of open (F == H(i-1,j) - alpha) / extend (F == F(i-1,j) - beta)
 *                  holds, take it; if both hold, extend when state H at (i-1,j) would next emit I
 *                  (neither its M nor its F test holds; D < I), else open
 *     H at (-1,j): j+1 'I';  H at (i,-1): i+1 'D'
 * The CIGAR is the op sequence in forward order, run-length encoded as BAM does:
 * element = (run length << 4) | op, op M = 0, I = 1, D = 2.
 */
#include <stdint.h>
#include <stdlib.h>

#define EXPORT __attribute__((visibility("default")))

enum { TB_OK = 0, TB_EINVALID_BASE = -1, TB_EEMPTY = -2, TB_ENOMEM = -5, TB_ERANGE = -8, TB_ECAP = -9 };

static int tb_code(uint8_t c) {
    switch (c) {
    case 'A': case 'a': return 0;
    case 'C': case 'c': return 1;
    case 'G': case 'g': return 2;
    case 'T': case 't': case 'U': case 'u': return 3;
    case 'N': case 'n': return 4;
    default: return -1;
    }
}

#define TB_NEG (-(1 << 29))

/* ops: caller buffer of `cap` uint32; out[0] = number of CIGAR elements, out[1] = global score. */
EXPORT int oracle_traceback(const uint8_t* q, int n, const uint8_t* t, int m, int32_t match, int32_t mismatch,
                            int32_t alpha, int32_t beta, int32_t t_start, int32_t t_end, int32_t q_start,
                            int32_t q_end, uint32_t* ops, int cap, int32_t* out) {
    if (n < 1 || m < 1) return TB_EEMPTY;
    if (t_start < 0 || q_start < 0 || t_end >= m || q_end >= n || t_start > t_end || q_start > q_end) return TB_ERANGE;
    const int M = t_end - t_start + 1, N = q_end - q_start + 1;
    const size_t W = (size_t)N + 1;
    int32_t* H = (int32_t*)malloc(sizeof(int32_t) * (size_t)(M + 1) * W);
    int32_t* E = (int32_t*)malloc(sizeof(int32_t) * (size_t)(M + 1) * W);
    int32_t* F = (int32_t*)malloc(sizeof(int32_t) * (size_t)(M + 1) * W);
    char* rev = (char*)malloc((size_t)M + (size_t)N + 2);
    if (!H || !E || !F || !rev) {
        free(H); free(E); free(F); free(rev);
        return TB_ENOMEM;
    }
    int st = TB_OK;
    for (int k = 0; k < n && st == TB_OK; ++k)
        if (tb_code(q[k]) < 0) st = TB_EINVALID_BASE;
    for (int k = 0; k < m && st == TB_OK; ++k)
        if (tb_code(t[k]) < 0) st = TB_EINVALID_BASE;
    if (st != TB_OK) {
        free(H); free(E); free(F); free(rev);
        return st;
    }
    /* index (i+1, j+1): row 0 / column 0 are the boundary i = -1 / j = -1 */
#define AT(X, i, j) X[(size_t)((i) + 1) * W + (size_t)((j) + 1)]
    AT(H, -1, -1) = 0;
    AT(E, -1, -1) = TB_NEG;
    AT(F, -1, -1) = TB_NEG;
    for (int j = 0; j < N; ++j) {
        AT(H, -1, j) = -(alpha + beta * j);
        AT(E, -1, j) = TB_NEG;
        AT(F, -1, j) = TB_NEG;
    }
    for (int i = 0; i < M; ++i) {
        AT(H, i, -1) = -(alpha + beta * i);
        AT(E, i, -1) = TB_NEG;
        AT(F, i, -1) = TB_NEG;
        const int tc = tb_code(t[t_start + i]);
        for (int j = 0; j < N; ++j) {
            const int qc = tb_code(q[q_start + j]);
            const int32_t s = (tc == qc && tc != 4) ? match : mismatch;
            int32_t e = AT(H, i, j - 1) - alpha, e2 = AT(E, i, j - 1) - beta;
            e = e > e2 ? e : e2;
            int32_t f = AT(H, i - 1, j) - alpha, f2 = AT(F, i - 1, j) - beta;
            f = f > f2 ? f : f2;
            int32_t h = AT(H, i - 1, j - 1) + s;
            h = h > e ? h : e;
            h = h > f ? h : f;
            AT(E, i, j) = e;
            AT(F, i, j) = f;
            AT(H, i, j) = h;
        }
    }
    /* traceback */
    int nr = 0, i = M - 1, j = N - 1, state = 0; /* 0 H, 1 F, 2 E */
    while (i >= 0 || j >= 0) {
        if (i < 0) { rev[nr++] = 'I'; --j; continue; }
        if (j < 0) { rev[nr++] = 'D'; --i; continue; }
        if (state == 0) {
            const int tc = tb_code(t[t_start + i]), qc = tb_code(q[q_start + j]);
            const int32_t s = (tc == qc && tc != 4) ? match : mismatch;
            if (AT(H, i, j) == AT(H, i - 1, j - 1) + s) {
                rev[nr++] = 'M';
                --i; --j;
            } else if (AT(H, i, j) == AT(F, i, j)) {
                state = 1;
            } else {
                state = 2;
            }
        } else if (state == 1) {
            rev[nr++] = 'D';
            const int32_t fv = AT(F, i, j);
            const int op = fv == AT(H, i - 1, j) - alpha, ex = fv == AT(F, i - 1, j) - beta;
            if (op && ex) {  /* both optimal: the smaller continuation (i >= 1 here: F(-1,j) = -inf) */
                const int tc = tb_code(t[t_start + i - 1]), qc = tb_code(q[q_start + j]);
                const int32_t s = (tc == qc && tc != 4) ? match : mismatch;
                const int32_t hv = AT(H, i - 1, j);
                const int next_i = !(hv == AT(H, i - 2, j - 1) + s) && !(hv == AT(F, i - 1, j));
                state = next_i ? 1 : 0;
            } else {
                state = op ? 0 : 1;
            }
            --i;
        } else {
            rev[nr++] = 'I';
            state = AT(E, i, j) == AT(H, i, j - 1) - alpha ? 0 : 2;
            --j;
        }
    }
    /* forward run-length encoding */
    int no = 0;
    for (int k = nr - 1; k >= 0;) {
        const char c = rev[k];
        int len = 0;
        while (k >= 0 && rev[k] == c) { ++len; --k; }
        if (no >= cap) { st = TB_ECAP; break; }
        ops[no++] = ((uint32_t)len << 4) | (uint32_t)(c == 'M' ? 0 : c == 'I' ? 1 : 2);
    }
    out[0] = st == TB_OK ? no : -1;
    out[1] = AT(H, M - 1, N - 1);
#undef AT
    free(H); free(E); free(F); free(rev);
    return st;
}
