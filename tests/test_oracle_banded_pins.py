"""Pin the oracle's BANDED mode (reading 16) to routes other than
itself (CPU-only).  Definition: only cells with |i - j| <= w are in the table; the rest read as 0
like out-of-table cells.  Routes: path enumeration restricted to in-band cells and the cubic WSB
recurrence with out-of-band cells at 0 (tests/pins.py); special cases: w >= max(m, n) is the plain
(pinned) oracle; w = 0 keeps only the main diagonal (LOCAL: Kadane's maximum-suffix recurrence;
EXTEND: the anchored diagonal walk, killed at <= 0); invariant: the score never decreases with w.
"""
import random

import numpy as np
import pytest

import oracle
import synth
from pins import brute_extend, brute_local, subst, wsb_extend, wsb_local


def _rand_scheme(rng):
    beta = rng.randint(1, 3)
    return dict(match=rng.randint(1, 4), mismatch=rng.randint(-6, -1), alpha=rng.randint(beta, 8), beta=beta)


def _rand_seq(rng, lo, hi, alphabet="ACGT"):
    return "".join(rng.choice(alphabet) for _ in range(rng.randint(lo, hi)))


def test_banded_random_tiny_brute_force_both_modes():
    rng = random.Random(1728)
    for _ in range(400):
        sc = _rand_scheme(rng)
        q, t = _rand_seq(rng, 1, 6, "ACGTN"), _rand_seq(rng, 1, 6, "ACGTN")
        w, h0 = rng.randint(0, 4), rng.randint(1, 12)
        assert oracle.align_banded(q, t, w, **sc) == brute_local(q, t, band=w, **sc), (q, t, w, sc)
        assert oracle.align_banded(q, t, w, mode=oracle.EXTEND, h0=h0, **sc) == \
            brute_extend(q, t, h0=h0, band=w, **sc), (q, t, w, sc, h0)


def test_banded_wsb_both_modes():
    rng = random.Random(1735)
    for _ in range(120):
        sc = _rand_scheme(rng)
        q = _rand_seq(rng, 1, 24)
        t = "".join(c for c in q if rng.random() > 0.15) + _rand_seq(rng, 0, 4) or "A"
        w, h0 = rng.randint(0, 8), rng.randint(1, 30)
        assert oracle.align_banded(q, t, w, **sc) == wsb_local(q, t, band=w, **sc), (q, t, w, sc)
        assert oracle.align_banded(q, t, w, mode=oracle.EXTEND, h0=h0, **sc) == \
            wsb_extend(q, t, h0=h0, band=w, **sc), (q, t, w, sc, h0)


def test_wide_band_is_the_unbanded_oracle():
    rng = random.Random(3)
    for _ in range(200):
        q, t = _rand_seq(rng, 1, 60), _rand_seq(rng, 1, 60)
        w = max(len(q), len(t)) + rng.randint(0, 3)
        assert oracle.align_banded(q, t, w) == oracle.align(q, t)
        assert oracle.align_banded(q, t, w, mode=oracle.EXTEND, h0=9) == oracle.align(q, t, mode=oracle.EXTEND, h0=9)


def test_zero_band_is_the_main_diagonal():
    rng = random.Random(4)
    for _ in range(200):
        q, t = _rand_seq(rng, 1, 40), _rand_seq(rng, 1, 40)
        L = min(len(q), len(t))
        # LOCAL: Kadane on the main diagonal, first maximum
        run, best, bi = 0, 0, 0
        for i in range(L):
            run = max(0, run + subst(t[i], q[i], 1, -4))
            if run > best:
                best, bi = run, i
        assert oracle.align_banded(q, t, 0) == (best, bi, bi)
        # EXTEND: the anchored walk, killed once the running total drops to <= 0
        h0 = rng.randint(1, 10)
        run, best, bi = h0, h0, -1
        for i in range(L):
            run += subst(t[i], q[i], 1, -4)
            if run <= 0:
                break
            if run > best:
                best, bi = run, i
        assert oracle.align_banded(q, t, 0, mode=oracle.EXTEND, h0=h0) == (best, bi, bi)


def test_score_monotone_in_band():
    rng = random.Random(5)
    for _ in range(60):
        q = _rand_seq(rng, 10, 80)
        t = "".join(c for c in q if rng.random() > 0.1) + _rand_seq(rng, 0, 10)
        prev = -1
        for w in range(0, 20, 3):
            s = oracle.align_banded(q, t, w)[0]
            assert s >= prev
            prev = s


def test_banded_batch_matches_single_calls():
    b = synth.generate(1, 80, seed=8, p_n=0.01)
    w = np.random.default_rng(1).integers(0, 40, b.n).astype(np.int32)
    for mode in (oracle.LOCAL, oracle.EXTEND):
        s, qe, te, st = oracle.banded_batch(b, w, mode=mode)
        assert (st == 0).all()
        for k in range(b.n):
            q, t = b.pair(k)
            assert (s[k], qe[k], te[k]) == oracle.align_banded(q, t, int(w[k]), mode=mode, h0=int(b.h0[k]))
    with pytest.raises(ValueError):
        oracle.align_banded("ACGT", "ACGT", -1)
