"""Pins of the BWA-MEM-compatible extension oracle (oracle/ksw.c; DESIGN.md
reading 17) against things other than itself:

* brute force: every alignment path from the seed anchor, enumerated op by op with BWA-MEM's rules
  (gaps open only right after a match/mismatch step or at the anchor, an insertion run never turns
  into a deletion run, separate insertion/deletion costs, N scores -1, a path dies when its running
  score reaches 0) gives the H table of every computed cell (flags = KSW_NO_TRIM);
* closed forms: identical strings, a band of width 0, an all-mismatch pair;
* a hand-derived z-drop case (an N run of known cost between two exact matches).
"""
import itertools

import numpy as np
import pytest

import oracle


def brute_table(q, t, h0, a, b, o_del, e_del, o_ins, e_ins, w):
    """Best live-path score ending at each cell (0 if no live path), paths enumerated one op at a
    time.  (i, j) = last consumed target / query index; mode A = anchor, D = after a match or
    mismatch step, I = inside an insertion run (query bases), X = inside a deletion run."""
    n, m = len(q), len(t)

    def S(i, j):
        if t[i] == "N" or q[j] == "N":
            return -1
        return a if t[i] == q[j] else -b

    best = np.zeros((m, n), np.int64)
    stack = [(-1, -1, "A", h0)]
    while stack:
        i, j, mode, sc = stack.pop()
        if i >= 0 and j >= 0:
            best[i, j] = max(best[i, j], sc)
        # match / mismatch step (needs a live cell: sc > 0 always holds for kept paths)
        if i + 1 < m and j + 1 < n and abs((i + 1) - (j + 1)) <= w:
            ns = sc + S(i + 1, j + 1)
            if ns > 0:
                stack.append((i + 1, j + 1, "D", ns))
        # insertion: opened right after a D step or at the anchor (row -1), extended inside a run
        if j + 1 < n and mode in ("A", "D", "I") and (i < 0 or abs(i - (j + 1)) <= w):
            ns = sc - (e_ins if mode == "I" else o_ins + e_ins)
            if ns > 0:
                stack.append((i, j + 1, "I", ns))
        # deletion: opened right after a D step or at the anchor (column -1), extended inside a run
        if i + 1 < m and mode in ("A", "D", "X") and (j < 0 or abs((i + 1) - j) <= w):
            ns = sc - (e_del if mode == "X" else o_del + e_del)
            if ns > 0:
                stack.append((i + 1, j, "X", ns))
    return best


def bookkeeping(B, h0, n, end_bonus, w):
    """The row-scan rules of ksw_extend2 applied to a full table (no z-drop, no trimming): the row
    maximum with its LAST column, the first row that strictly beats the running maximum, the
    end-to-end score of column n-1 (rows whose band reaches it) with its LAST row, stop after an
    all-zero row."""
    mx, mi, mjx, gscore, gi, off = h0, -1, -1, -1, -1, 0
    for i in range(B.shape[0]):
        row = B[i]
        mrow = int(row.max())
        mj = int(np.nonzero(row == mrow)[0][-1]) if mrow > 0 else -1
        h_last = int(row[n - 1])
        if i + w + 1 >= n and h_last >= gscore:
            gscore, gi = h_last, i
        if mrow == 0:
            break
        if mrow > mx:
            mx, mi, mjx = mrow, i, mj
            off = max(off, abs(mj - i))
    clip = 1 if (gscore <= 0 or gscore <= mx - end_bonus) else 0
    return dict(score=mx, qle=mjx + 1, tle=mi + 1, gtle=gi + 1, gscore=gscore, max_off=off, clip=clip)


def _random_case(rng, alphabet="ACGTN"):
    n, m = int(rng.integers(1, 6)), int(rng.integers(1, 6))
    q = "".join(rng.choice(list(alphabet), n))
    t = "".join(rng.choice(list(alphabet), m))
    p = dict(a=int(rng.integers(1, 4)), b=int(rng.integers(1, 5)), o_del=int(rng.integers(0, 7)),
             e_del=int(rng.integers(1, 4)), o_ins=int(rng.integers(0, 7)), e_ins=int(rng.integers(1, 4)),
             w=int(rng.integers(0, 7)), end_bonus=100, zdrop=0)
    return q, t, int(rng.integers(1, 16)), p


def test_table_equals_brute_force():
    """The DP values of every computed cell equal the best live path (2,000 random tiny cases:
    separate insertion/deletion costs, bands, N, seeds of 1..15)."""
    rng = np.random.default_rng(17)
    for _ in range(2000):
        q, t, h0, p = _random_case(rng)
        r = oracle.ksw_extend(q, t, h0, flags=oracle.KSW_NO_TRIM, table=True, **p)
        B = brute_table(q, t, h0, p["a"], p["b"], p["o_del"], p["e_del"], p["o_ins"], p["e_ins"], p["w"])
        H = r["H"]
        done = H >= 0
        assert np.array_equal(H[done], B[done]), (q, t, h0, p, H, B)
        # every in-band cell of every row up to the stop row was computed
        for i in range(len(t)):
            row = done[i]
            if not row.any():
                break
            lo, hi = max(0, i - p["w"]), min(len(q), i + p["w"] + 1)
            assert row[lo:hi].all() and not row[:lo].any() and not row[hi:].any(), (q, t, p, H)


def test_outputs_equal_brute_force_bookkeeping():
    rng = np.random.default_rng(29)
    for _ in range(2000):
        q, t, h0, p = _random_case(rng)
        r = oracle.ksw_extend(q, t, h0, flags=oracle.KSW_NO_TRIM, **p)
        B = brute_table(q, t, h0, p["a"], p["b"], p["o_del"], p["e_del"], p["o_ins"], p["e_ins"], p["w"])
        exp = bookkeeping(B, h0, len(q), p["end_bonus"], p["w"])
        assert {k: r[k] for k in exp} == exp, (q, t, h0, p, r, exp)


def test_exhaustive_len_1_to_3_bwa_scores():
    """All ACGT pairs of lengths 1..3 with BWA-MEM's scores and h0 in {1, 3, 8}: brute force."""
    strs = ["".join(s) for L in (1, 2, 3) for s in itertools.product("ACGT", repeat=L)]
    p = dict(oracle.KSW_BWA, end_bonus=100, zdrop=0)
    for q in strs:
        for t in strs:
            for h0 in (1, 3, 8):
                r = oracle.ksw_extend(q, t, h0, flags=oracle.KSW_NO_TRIM, **p)
                B = brute_table(q, t, h0, 1, 4, 6, 1, 6, 1, p["w"])
                exp = bookkeeping(B, h0, len(q), p["end_bonus"], p["w"])
                assert {k: r[k] for k in exp} == exp, (q, t, h0, r, exp)


def test_trimming_never_raises_the_score():
    """The beg/end row trimming only drops cells: score (trimmed) <= score (band only)."""
    rng = np.random.default_rng(3)
    for _ in range(500):
        L = int(rng.integers(5, 60))
        q = "".join(rng.choice(list("ACGT"), L))
        t = "".join(ch if rng.random() > 0.15 else rng.choice(list("ACGTN")) for ch in q)
        if rng.random() < 0.5:
            k = int(rng.integers(1, L))
            t = t[:k] + "".join(rng.choice(list("ACGT"), int(rng.integers(1, 6)))) + t[k:]
        h0 = int(rng.integers(1, 30))
        a = oracle.ksw_extend(q, t, h0)["score"]
        b = oracle.ksw_extend(q, t, h0, flags=oracle.KSW_NO_TRIM)["score"]
        assert h0 <= a <= b


@pytest.mark.parametrize("L", [1, 2, 7, 64, 150, 333])
def test_identical_closed_form(L):
    """q == t (no N): every base matches -> score = gscore = h0 + L*a at qle = tle = gtle = L; the
    end-to-end result is kept (clip 0), max_off 0.  BWA-MEM defaults incl. z-drop and trimming."""
    rng = np.random.default_rng(L)
    s = "".join(rng.choice(list("ACGT"), L))
    for h0 in (1, 19, 50):
        r = oracle.ksw_extend(s, s, h0)
        assert r == dict(score=h0 + L, qle=L, tle=L, gtle=L, gscore=h0 + L, max_off=0, clip=0), (L, h0, r)


def test_band_zero_blocks_gaps():
    """w = 0 keeps only the diagonal.  q = X GGGG S, t = X GGG S with X = ACGTACGTAA and S a 12-mer
    without two equal neighbours: on the diagonal the 13 bases X GGG match and every later cell
    compares S[k] with S[k+1] (a mismatch), so the band-0 extension keeps 20 + 13 at (13, 13); the
    default band crosses the extra G with one insertion (o_ins + e_ins = 7) and matches S:
    20 + 13 - 7 + 12 = 38 at (qle, tle) = (26, 25), which is also the end-to-end score."""
    S = "ACGTACGTACGT"
    q = "ACGTACGTAA" + "GGGG" + S
    t = "ACGTACGTAA" + "GGG" + S
    r = oracle.ksw_extend(q, t, 20, w=0, zdrop=0)
    assert r["score"] == 20 + 13 and (r["qle"], r["tle"]) == (13, 13)
    wide = oracle.ksw_extend(q, t, 20, zdrop=0)
    assert (wide["score"], wide["qle"], wide["tle"]) == (38, 26, 25)
    assert (wide["gscore"], wide["gtle"], wide["clip"]) == (38, 25, 0)


def test_all_mismatch_keeps_the_seed():
    r = oracle.ksw_extend("AAAA", "CCCC", 3)
    assert (r["score"], r["qle"], r["tle"]) == (3, 0, 0) and r["clip"] == 1


def test_zdrop_hand_derived():
    """X (50 exact bases), 110 N vs N (each -1), Y (200 exact bases), h0 = 120.  The best cell of
    row 49+k inside the N run is the diagonal one, 170 - k at column 49+k (any gap costs >= 7 more),
    so the z-drop test at that row is 170 - (170 - k) - 0 > zdrop, i.e. k > 100: the extension stops
    at row 150 and keeps the maximum 170 at (50, 50).  Without z-drop it reaches the end:
    170 - 110 + 200 = 260 at (360, 360), and the end-to-end result is kept (260 > 260 - 5)."""
    rng = np.random.default_rng(8)
    X = "".join(rng.choice(list("ACGT"), 50))
    Y = "".join(rng.choice(list("ACGT"), 200))
    s = X + "N" * 110 + Y
    r = oracle.ksw_extend(s, s, 120)
    assert r == dict(score=170, qle=50, tle=50, gtle=0, gscore=-1, max_off=0, clip=1), r
    r = oracle.ksw_extend(s, s, 120, zdrop=0)
    assert r == dict(score=260, qle=360, tle=360, gtle=360, gscore=260, max_off=0, clip=0), r
    # the drop peaks at k = 110 (the last N row): zdrop 110 never fires, zdrop 109 fires there
    assert oracle.ksw_extend(s, s, 120, zdrop=110)["score"] == 260
    assert oracle.ksw_extend(s, s, 120, zdrop=109)["score"] == 170
