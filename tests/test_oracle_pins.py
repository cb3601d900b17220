"""Pin the CPU oracle to things other than itself (CPU-only; runs under -m "not gpu").

Pins used (each chosen so a dropped term, a wrong sign/index or a transposed operand fails one):
  * SPEC.md worked examples (tests/golden/spec_examples.tsv, each row cited);
  * SURVEY Appendix A rows, re-derived here by brute force (tests/pins.py);
  * exhaustive brute-force path enumeration on all pairs of length <= 3 over ACGT (LOCAL) and on
    random tiny pairs for both modes and random schemes;
  * the cubic Waterman-Smith-Beyer recurrence (general gap cost, no E/F states) up to ~24 bp;
  * closed forms: identical strings, homopolymers, all-mismatch, gap-free Kadane regime;
  * invariants: 0 <= score <= match*min(m,n), swap symmetry, prefix monotonicity, N behaviour;
  * the two-row form equals the full-matrix definition.
"""
import itertools
import random

import pytest

import oracle
from conftest import load_tsv
from pins import brute_extend, brute_local, kadane_gapfree, wsb_extend, wsb_local

MODES = {"LOCAL": oracle.LOCAL, "EXTEND": oracle.EXTEND}


def orc(q, t, match=1, mismatch=-4, alpha=7, beta=1, mode=oracle.LOCAL, h0=0, rows=False):
    return oracle.align(q, t, match, mismatch, alpha, beta, mode, h0, rows=rows)


@pytest.mark.parametrize("row", load_tsv("spec_examples.tsv"), ids=lambda r: f"{r['q']}-{r['t']}")
def test_spec_examples(row):
    got = orc(row["q"], row["t"], row["match"], row["mismatch"], row["alpha"], row["beta"], MODES[row["mode"]],
              row["h0"])
    assert got == row["expect"], row["note"]


@pytest.mark.parametrize("row", load_tsv("survey_appendix_a.tsv"), ids=lambda r: f"{r['mode']}-{r['q']}-{r['t']}")
def test_appendix_a_with_brute_force(row):
    sc = dict(match=row["match"], mismatch=row["mismatch"], alpha=row["alpha"], beta=row["beta"])
    if row["mode"] == "LOCAL":
        ref = wsb_local(row["q"], row["t"], **sc)
        if len(row["q"]) * len(row["t"]) <= 64:
            assert brute_local(row["q"], row["t"], **sc) == ref
    else:
        ref = wsb_extend(row["q"], row["t"], h0=row["h0"], **sc)
        assert brute_extend(row["q"], row["t"], h0=row["h0"], **sc) == ref
    assert ref == row["expect"], "independent formulations disagree with the survey's value"
    assert orc(row["q"], row["t"], mode=MODES[row["mode"]], h0=row["h0"], **sc) == ref


def test_cell_update_worked_example_via_tables():
    """h_diag=4, h_left=3, e_left=2, h_up=0, f_up=0, s=+2, alpha=5, beta=1 -> e=1, f=0, h=6.
    Realised inside a table: the oracle's E/F/H at one cell must follow Eqs. 1-3 from its neighbours."""
    H, E, F, _ = oracle.tables("ACGTAC", "ACTTAC", match=2, mismatch=-1, alpha=5, beta=1)
    m, n = H.shape[0] - 1, H.shape[1] - 1
    q, t = "ACGTAC", "ACTTAC"
    for i in range(m):
        for j in range(n):
            e = max(0, H[i + 1, j] - 5, E[i + 1, j] - 1)
            f = max(0, H[i, j + 1] - 5, F[i, j + 1] - 1)
            s = 2 if q[j] == t[i] else -1
            assert E[i + 1, j + 1] == e and F[i + 1, j + 1] == f
            assert H[i + 1, j + 1] == max(0, e, f, H[i, j] + s)


def test_exhaustive_len_le_3_local_brute_force():
    """All 7,056 pairs of ACGT strings of length 1..3, alpha=2 beta=1 so gaps matter."""
    strs = ["".join(p) for L in (1, 2, 3) for p in itertools.product("ACGT", repeat=L)]
    bad = 0
    for q in strs:
        for t in strs:
            if orc(q, t, 1, -4, 2, 1) != brute_local(q, t, 1, -4, 2, 1):
                bad += 1
    assert bad == 0


def _rand_scheme(rng):
    beta = rng.randint(1, 3)
    return dict(match=rng.randint(1, 4), mismatch=rng.randint(-6, -1), alpha=rng.randint(beta, 8), beta=beta)


def _rand_seq(rng, lo, hi, alphabet="ACGT"):
    return "".join(rng.choice(alphabet) for _ in range(rng.randint(lo, hi)))


def test_random_tiny_brute_force_both_modes():
    rng = random.Random(20230123)
    for _ in range(400):
        sc = _rand_scheme(rng)
        q, t = _rand_seq(rng, 1, 5, "ACGTN"), _rand_seq(rng, 1, 5, "ACGTN")
        assert orc(q, t, **sc) == brute_local(q, t, **sc), (q, t, sc)
        h0 = rng.randint(1, 12)
        assert orc(q, t, mode=oracle.EXTEND, h0=h0, **sc) == brute_extend(q, t, h0=h0, **sc), (q, t, sc, h0)


def test_random_wsb_both_modes():
    rng = random.Random(7)
    for _ in range(150):
        sc = _rand_scheme(rng)
        q, t = _rand_seq(rng, 1, 24), _rand_seq(rng, 1, 24)
        if rng.random() < 0.5:  # related sequences so long gapped alignments occur
            t = "".join(c for c in q if rng.random() > 0.15) + _rand_seq(rng, 0, 4)
            t = t or "A"
        assert orc(q, t, **sc) == wsb_local(q, t, **sc), (q, t, sc)
        h0 = rng.randint(1, 30)
        assert orc(q, t, mode=oracle.EXTEND, h0=h0, **sc) == wsb_extend(q, t, h0=h0, **sc), (q, t, sc, h0)


@pytest.mark.parametrize("L", [1, 2, 7, 8, 9, 63, 150, 300])
def test_identical_strings_closed_form(L):
    rng = random.Random(L)
    s = _rand_seq(rng, L, L)
    for match in (1, 3):
        assert orc(s, s, match, -4, 7, 1) == (L * match, L - 1, L - 1)
        assert orc(s, s, match, -4, 7, 1, mode=oracle.EXTEND, h0=11) == (11 + L * match, L - 1, L - 1)


@pytest.mark.parametrize("n,m", [(1, 1), (4, 6), (6, 4), (8, 8), (20, 33)])
def test_homopolymer_closed_form(n, m):
    """H(i,j) = (min(i,j)+1)*match for identical homopolymers; max at (k-1,k-1), k = min(m,n)."""
    H, _, _, res = oracle.tables("A" * n, "A" * m, match=2, mismatch=-4, alpha=7, beta=1)
    for i in range(m):
        for j in range(n):
            assert H[i + 1, j + 1] == (min(i, j) + 1) * 2
    k = min(m, n)
    assert res == (2 * k, k - 1, k - 1)


def test_all_mismatch():
    assert orc("AAAAAAA", "CCCGGGTTT") == (0, 0, 0)
    assert orc("AAAAAAA", "CCCGGGTTT", mode=oracle.EXTEND, h0=9) == (9, -1, -1)


def test_gapfree_kadane_regime():
    rng = random.Random(11)
    for _ in range(200):
        q, t = _rand_seq(rng, 1, 40), _rand_seq(rng, 1, 40)
        match, mismatch = rng.randint(1, 3), rng.randint(-5, -1)
        alpha = match * min(len(q), len(t)) + 1
        assert orc(q, t, match, mismatch, alpha, 1) == kadane_gapfree(q, t, match, mismatch), (q, t)


def test_invariants_symmetry_bounds_prefix():
    rng = random.Random(5)
    for _ in range(200):
        sc = _rand_scheme(rng)
        q, t = _rand_seq(rng, 1, 60, "ACGTN"), _rand_seq(rng, 1, 60, "ACGTN")
        s, qe, te = orc(q, t, **sc)
        assert 0 <= s <= sc["match"] * min(len(q), len(t))
        s2, qe2, te2 = orc(t, q, **sc)
        assert s2 == s  # SPEC S:394 symmetry (coordinates swap only for a unique argmax)
        # prefix monotonicity: appending bases never lowers the score
        assert orc(q + _rand_seq(rng, 1, 5), t, **sc)[0] >= s
        assert orc(q, t + _rand_seq(rng, 1, 5), **sc)[0] >= s
        # EXTEND score >= h0 and coordinates in range
        h0 = rng.randint(1, 40)
        e, eq, et = orc(q, t, mode=oracle.EXTEND, h0=h0, **sc)
        assert e >= h0 and ((eq, et) == (-1, -1) if e == h0 else (0 <= eq < len(q) and 0 <= et < len(t)))


def test_lowercase_and_u():
    assert orc("acgu", "ACGT") == orc("ACGT", "ACGT") == (4, 3, 3)


def test_errors():
    with pytest.raises(ValueError):
        orc("ACGX", "ACGT")
    with pytest.raises(ValueError):
        orc("", "ACGT")
    with pytest.raises(ValueError):
        orc("ACGT", "ACGT", mode=oracle.EXTEND, h0=0)


def test_rows_form_equals_full_definition():
    rng = random.Random(3)
    for _ in range(300):
        sc = _rand_scheme(rng)
        q, t = _rand_seq(rng, 1, 300, "ACGTN"), _rand_seq(rng, 1, 300, "ACGTN")
        h0 = rng.randint(1, 50)
        for mode in (oracle.LOCAL, oracle.EXTEND):
            assert orc(q, t, mode=mode, h0=h0, **sc) == orc(q, t, mode=mode, h0=h0, rows=True, **sc)


def test_batch_driver_matches_single_calls():
    import synth

    b = synth.generate(1, 200, seed=99, p_n=0.01)
    for mode in (oracle.LOCAL, oracle.EXTEND):
        s, qe, te, st, _ = oracle.align_batch(b, mode=mode, threads=3)
        assert (st == 0).all()
        for k in range(0, 200, 17):
            q, t = b.pair(k)
            assert (s[k], qe[k], te[k]) == orc(q, t, mode=mode, h0=int(b.h0[k]))
