"""Pin the oracle's START coordinates (LOCAL, reading 15) to routes
other than its reverse DP (CPU-only).

Definition pinned: the start is the first aligned column (t_start, q_start) of an optimal alignment
ending at the reported end cell; among several, the largest t_start, then the largest q_start;
(0, 0) when the score is 0.  Routes: explicit path enumeration (tests/pins.py brute_local_start),
and a scan of candidate starts with an anchored cubic WSB recurrence (anchored_local_start) —
neither reverses anything.  Closed forms: identical strings start at (0, 0); a core planted between
N flanks (N never matches) starts and ends exactly at the core.
"""
import itertools
import random

import pytest

import oracle
import synth
from pins import anchored_global, anchored_local_start, brute_local_start


def _rand_scheme(rng):
    beta = rng.randint(1, 3)
    return dict(match=rng.randint(1, 4), mismatch=rng.randint(-6, -1), alpha=rng.randint(beta, 8), beta=beta)


def _rand_seq(rng, lo, hi, alphabet="ACGT"):
    return "".join(rng.choice(alphabet) for _ in range(rng.randint(lo, hi)))


def test_start_exhaustive_len_le_3_brute_force():
    """All 7,056 ACGT pairs of length 1..3, alpha=2 beta=1 (gaps and ties matter)."""
    strs = ["".join(p) for L in (1, 2, 3) for p in itertools.product("ACGT", repeat=L)]
    bad = [(q, t) for q in strs for t in strs
           if oracle.start(q, t, 1, -4, 2, 1) != brute_local_start(q, t, 1, -4, 2, 1)]
    assert not bad, bad[:5]


def test_start_random_tiny_brute_force():
    rng = random.Random(20231017)
    for _ in range(400):
        sc = _rand_scheme(rng)
        q, t = _rand_seq(rng, 1, 6, "ACGTN"), _rand_seq(rng, 1, 6, "ACGTN")
        assert oracle.start(q, t, **sc) == brute_local_start(q, t, **sc), (q, t, sc)


def test_start_random_anchored_wsb():
    rng = random.Random(99)
    for _ in range(60):
        sc = _rand_scheme(rng)
        q = _rand_seq(rng, 4, 14)
        t = "".join(c for c in q if rng.random() > 0.15) + _rand_seq(rng, 0, 3)
        t = _rand_seq(rng, 0, 3) + (t or "A")
        assert oracle.start(q, t, **sc) == anchored_local_start(q, t, **sc), (q, t, sc)


@pytest.mark.parametrize("L", [1, 8, 31, 150])
def test_start_identical_strings(L):
    s = "".join(random.Random(L).choice("ACGT") for _ in range(L))
    assert oracle.start(s, s) == (L, L - 1, L - 1, 0, 0)


@pytest.mark.parametrize("seed", range(6))
def test_start_planted_core_between_n_flanks(seed):
    rng = random.Random(seed)
    core = _rand_seq(rng, 5, 60)
    a, b, c, d = (rng.randint(0, 30) for _ in range(4))
    q, t = "N" * a + core + "N" * b, "N" * c + core + "N" * d
    L = len(core)
    assert oracle.start(q, t) == (L, a + L - 1, c + L - 1, a, c)


def test_start_zero_score_and_swap_symmetry():
    assert oracle.start("AAAA", "TTTT") == (0, 0, 0, 0, 0)
    assert oracle.start("NNNN", "NNNN") == (0, 0, 0, 0, 0)
    rng = random.Random(5)
    for _ in range(200):
        q, t = _rand_seq(rng, 1, 40), _rand_seq(rng, 1, 40)
        s, qe, te, qs, ts = oracle.start(q, t)
        assert 0 <= qs <= qe and 0 <= ts <= te
        if s > 0:  # the aligned substrings reach the score with both ends anchored
            assert anchored_global(q, t, qs, ts, qe, te) == s


def test_start_batch_matches_single_calls():
    b = synth.generate(1, 60, seed=3, p_n=0.01)
    out = oracle.start_batch(b)
    assert (out[5] == 0).all()
    for k in range(b.n):
        q, t = b.pair(k)
        assert tuple(int(x[k]) for x in out[:5]) == oracle.start(q, t)
    # forward part equals the plain oracle
    s, qe, te, st, _ = oracle.align_batch(b)
    assert (s == out[0]).all() and (qe == out[1]).all() and (te == out[2]).all()
