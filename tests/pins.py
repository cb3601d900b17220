"""Independent formulations used to PIN the oracle (tests only; nothing here is imported by the
oracle or by the product).  Each is a different mathematical route to the same quantity:

* ``brute_local`` / ``brute_extend`` — enumerate every alignment path explicitly (exponential;
  tiny inputs only).  Gap cost g(k) = alpha + (k-1) beta per maximal run of one gap type; an
  insertion run followed by a deletion run is two gaps (SURVEY §8(c) "a gap may open after any
  column").  LOCAL: paths start with a match/mismatch column anywhere, value = path score, cell
  value = max(0, best path ending there) (Eq. 1 "0" term = empty alignment).  EXTEND:
  paths start at the anchor (-1,-1) with total h0 and are killed the moment the running total
  drops to <= 0 (SURVEY §8(c) brute-force definition).
* ``wsb_local`` / ``wsb_extend`` — the cubic Waterman-Smith-Beyer recurrence with an explicit
  general gap cost g(k) (no E/F auxiliary states at all).
* ``kadane_gapfree`` — when alpha > match*min(m,n) no gap can ever help, and H on every
  diagonal is Kadane's maximum-suffix recurrence H = max(0, H_prev + S).

All return (score, q_end, t_end) with the tie rule of SPEC S:205/S:256 (max score, then smallest
target index i, then smallest query index j) and the zero/anchor conventions of SURVEY §8(b).
"""
from __future__ import annotations

import sys

NEG = -(1 << 40)


def subst(a: str, b: str, match: int, mismatch: int) -> int:
    a, b = a.upper().replace("U", "T"), b.upper().replace("U", "T")
    return match if (a == b and a != "N") else mismatch


def _pick(cells: dict, floor: int, floor_pos: tuple[int, int]):
    """cells: {(i, j): value}; returns (score, q_end, t_end) by the tie rule."""
    best, bi, bj = floor, floor_pos[0], floor_pos[1]
    for (i, j) in sorted(cells):
        if cells[(i, j)] > best:
            best, bi, bj = cells[(i, j)], i, j
    return best, bj, bi


def _inband(i, j, band):
    return band is None or abs(i - j) <= band


def brute_local(q: str, t: str, match=1, mismatch=-4, alpha=7, beta=1, band=None):
    """band: None, or w >= 0 — paths may only visit cells with |i - j| <= w (NEXT-2)."""
    n, m = len(q), len(t)
    best: dict = {}
    sys.setrecursionlimit(10000)

    def rec(i, j, total, last):
        if not _inband(i, j, band):
            return
        key = (i, j)
        if total > best.get(key, NEG):
            best[key] = total
        if i + 1 < m and j + 1 < n:
            rec(i + 1, j + 1, total + subst(t[i + 1], q[j + 1], match, mismatch), "M")
        if j + 1 < n:
            rec(i, j + 1, total - (beta if last == "I" else alpha), "I")
        if i + 1 < m:
            rec(i + 1, j, total - (beta if last == "D" else alpha), "D")

    for i in range(m):
        for j in range(n):
            rec(i, j, subst(t[i], q[j], match, mismatch), "M")
    cells = {k: max(0, v) for k, v in best.items()}
    for i in range(m):
        for j in range(n):
            cells.setdefault((i, j), 0)
    return _pick(cells, 0, (0, 0))


def brute_extend(q: str, t: str, match=1, mismatch=-4, alpha=7, beta=1, h0=10, band=None):
    n, m = len(q), len(t)
    best: dict = {}

    def rec(i, j, total, last):
        if i >= 0 and j >= 0 and not _inband(i, j, band):
            return
        if i >= 0 and j >= 0 and total > best.get((i, j), NEG):
            best[(i, j)] = total
        if i + 1 < m and j + 1 < n:
            nt = total + subst(t[i + 1], q[j + 1], match, mismatch)
            if nt > 0:
                rec(i + 1, j + 1, nt, "M")
        if j + 1 < n:
            nt = total - (beta if last == "I" else alpha)
            if nt > 0:
                rec(i, j + 1, nt, "I")
        if i + 1 < m:
            nt = total - (beta if last == "D" else alpha)
            if nt > 0:
                rec(i + 1, j, nt, "D")

    rec(-1, -1, h0, None)
    return _pick(best, h0, (-1, -1))


def _g(k, alpha, beta):
    return alpha + (k - 1) * beta


def wsb_local(q: str, t: str, match=1, mismatch=-4, alpha=7, beta=1, band=None):
    n, m = len(q), len(t)
    H = [[0] * (n + 1) for _ in range(m + 1)]  # H[i+1][j+1]
    for i in range(m):
        for j in range(n):
            if not _inband(i, j, band):
                continue  # outside the band: H stays 0
            v = max(0, H[i][j] + subst(t[i], q[j], match, mismatch))
            for k in range(1, j + 2):
                v = max(v, H[i + 1][j + 1 - k] - _g(k, alpha, beta))
            for k in range(1, i + 2):
                v = max(v, H[i + 1 - k][j + 1] - _g(k, alpha, beta))
            H[i + 1][j + 1] = v
    cells = {(i, j): H[i + 1][j + 1] for i in range(m) for j in range(n)}
    return _pick(cells, 0, (0, 0))


def wsb_extend(q: str, t: str, match=1, mismatch=-4, alpha=7, beta=1, h0=10, band=None):
    n, m = len(q), len(t)
    H = [[0] * (n + 1) for _ in range(m + 1)]
    H[0][0] = h0
    for j in range(n):
        H[0][j + 1] = max(0, h0 - _g(j + 1, alpha, beta))
    for i in range(m):
        H[i + 1][0] = max(0, h0 - _g(i + 1, alpha, beta))
    for i in range(m):
        for j in range(n):
            if not _inband(i, j, band):
                continue
            hd = H[i][j]
            v = hd + subst(t[i], q[j], match, mismatch) if hd > 0 else 0
            v = max(0, v)
            for k in range(1, j + 2):
                src = H[i + 1][j + 1 - k]
                if src > 0:
                    v = max(v, src - _g(k, alpha, beta))
            for k in range(1, i + 2):
                src = H[i + 1 - k][j + 1]
                if src > 0:
                    v = max(v, src - _g(k, alpha, beta))
            H[i + 1][j + 1] = v
    cells = {(i, j): H[i + 1][j + 1] for i in range(m) for j in range(n)}
    return _pick(cells, h0, (-1, -1))


def kadane_gapfree(q: str, t: str, match=1, mismatch=-4):
    """LOCAL result when gaps can never help (alpha > match*min(m,n)): per diagonal Kadane."""
    n, m = len(q), len(t)
    cells = {}
    for d in range(-(m - 1), n):  # d = j - i
        run = 0
        i0 = max(0, -d)
        for i in range(i0, m):
            j = i + d
            if j >= n:
                break
            run = max(0, run + subst(t[i], q[j], match, mismatch))
            cells[(i, j)] = run
    return _pick(cells, 0, (0, 0))


# ---- start coordinates (LOCAL, reading 15) ---------------------
# The start of the reported alignment is the FIRST aligned column (t_start, q_start) of an optimal
# alignment ending at the reported end cell; among several, the largest t_start, then the largest
# q_start.  score 0: (0, 0).  Two routes, neither using a reversed DP:


def brute_local_start(q: str, t: str, match=1, mismatch=-4, alpha=7, beta=1):
    """(score, q_end, t_end, q_start, t_start) by explicit path enumeration (tiny inputs)."""
    score, qe, te = brute_local(q, t, match, mismatch, alpha, beta)
    if score == 0:
        return 0, qe, te, 0, 0
    n, m = len(q), len(t)
    starts = []

    def rec(i, j, total, last, s):
        if (i, j) == (te, qe) and last == "M" and total == score:
            starts.append(s)
        if i + 1 < m and j + 1 < n:
            rec(i + 1, j + 1, total + subst(t[i + 1], q[j + 1], match, mismatch), "M", s)
        if j + 1 < n:
            rec(i, j + 1, total - (beta if last == "I" else alpha), "I", s)
        if i + 1 < m:
            rec(i + 1, j, total - (beta if last == "D" else alpha), "D", s)

    for i in range(te + 1):
        for j in range(qe + 1):
            rec(i, j, subst(t[i], q[j], match, mismatch), "M", (i, j))
    ts, qs = max(starts)
    return score, qe, te, qs, ts


def anchored_global(q: str, t: str, qs, ts, qe, te, match=1, mismatch=-4, alpha=7, beta=1):
    """Best value of an alignment of t[ts..te] with q[qs..qe] whose first and last columns are
    aligned pairs (t_ts~q_qs, t_te~q_qe); cubic WSB form with an explicit gap cost, no E/F."""
    a, b = t[ts:te + 1], q[qs:qe + 1]
    m, n = len(a), len(b)
    # V / I / D[i][j]: best value of a path from (0,0)[M] ending at (i,j) with last column an
    # aligned pair / an insertion run / a deletion run (a run may follow a run of the other type)
    V = [[NEG] * n for _ in range(m)]
    I = [[NEG] * n for _ in range(m)]
    D = [[NEG] * n for _ in range(m)]
    V[0][0] = subst(a[0], b[0], match, mismatch)
    for i in range(m):
        for j in range(n):
            if i > 0 and j > 0:
                prev = max(V[i - 1][j - 1], I[i - 1][j - 1], D[i - 1][j - 1])
                if prev > NEG:
                    V[i][j] = prev + subst(a[i], b[j], match, mismatch)
            for k in range(1, j + 1):
                src = max(V[i][j - k], D[i][j - k])
                if src > NEG:
                    I[i][j] = max(I[i][j], src - _g(k, alpha, beta))
            for k in range(1, i + 1):
                src = max(V[i - k][j], I[i - k][j])
                if src > NEG:
                    D[i][j] = max(D[i][j], src - _g(k, alpha, beta))
    return V[m - 1][n - 1]


def anchored_local_start(q: str, t: str, match=1, mismatch=-4, alpha=7, beta=1):
    """Same quantity by scanning candidate starts from the largest (t_start, q_start) down and
    taking the first whose anchored alignment to the end cell reaches the score (WSB route)."""
    score, qe, te = wsb_local(q, t, match, mismatch, alpha, beta)
    if score == 0:
        return 0, qe, te, 0, 0
    for ts in range(te, -1, -1):
        for qs in range(qe, -1, -1):
            if anchored_global(q, t, qs, ts, qe, te, match, mismatch, alpha, beta) == score:
                return score, qe, te, qs, ts
    raise AssertionError("no start reaches the score")
