"""Pins of the CIGAR traceback oracle (oracle/traceback.c; reading 18):

* brute force: every alignment of two short substrings, enumerated as an op string (M, I, D) and
  scored with the affine scheme (each maximal gap run costs alpha + beta*(len-1)); the oracle's
  score must be the optimum and its op string the smallest optimal one read from the end with
  M < D < I (the reading's choice);
* consistency on realistic pairs: for LOCAL results (oracle ends, oracle starts), the traceback of
  t[t_start..t_end] x q[q_start..q_end] scores exactly the local score, and an independent CIGAR
  scorer (walking the ops over the sequences) agrees; the ops consume exactly the two substrings;
* closed forms: identical strings -> one M run; an insertion in a homopolymer is left-aligned.
"""
import itertools

import numpy as np
import pytest

import oracle
import synth

RANK = {"M": 0, "D": 1, "I": 2}


def score_ops(ops, t, q, match, mismatch, alpha, beta):
    """Independent scorer: walk an op string over t (rows) and q (columns)."""
    i = j = 0
    sc = 0
    prev = None
    for op in ops:
        if op == "M":
            sc += match if (t[i] == q[j] and t[i] != "N") else mismatch
            i += 1
            j += 1
        elif op == "D":
            sc -= beta if prev == "D" else alpha
            i += 1
        else:
            sc -= beta if prev == "I" else alpha
            j += 1
        prev = op
    assert i == len(t) and j == len(q)
    return sc


def all_alignments(m, n):
    """Every op string over {M, D, I} consuming m target and n query bases."""
    out = []

    def rec(i, j, acc):
        if i == m and j == n:
            out.append("".join(acc))
            return
        if i < m and j < n:
            acc.append("M"); rec(i + 1, j + 1, acc); acc.pop()
        if i < m:
            acc.append("D"); rec(i + 1, j, acc); acc.pop()
        if j < n:
            acc.append("I"); rec(i, j + 1, acc); acc.pop()

    rec(0, 0, [])
    return out


def expand(cigar):
    out, num = [], ""
    for ch in cigar:
        if ch.isdigit():
            num += ch
        else:
            out.append(ch * int(num))
            num = ""
    return "".join(out)


def test_brute_force_optimal_and_smallest():
    rng = np.random.default_rng(18)
    cache = {}
    for _ in range(1500):
        m, n = int(rng.integers(1, 6)), int(rng.integers(1, 6))
        t = "".join(rng.choice(list("ACGTN"), m))
        q = "".join(rng.choice(list("ACGTN"), n))
        beta = int(rng.integers(1, 4))
        sc = (int(rng.integers(1, 4)), int(rng.integers(-5, 0)), int(rng.integers(beta, 8)), beta)
        cig, gs = oracle.traceback(q, t, 0, m - 1, 0, n - 1, *sc)
        alns = cache.setdefault((m, n), all_alignments(m, n))
        scores = [score_ops(a, t, q, *sc) for a in alns]
        best = max(scores)
        assert gs == best, (q, t, sc)
        opt = [a for a, s in zip(alns, scores) if s == best]
        want = min(opt, key=lambda a: [RANK[c] for c in reversed(a)])
        assert expand(cig) == want, (q, t, sc, cig, want, opt)


def test_local_results_consistency():
    """Config-1-like pairs: LOCAL end (oracle), start (oracle), traceback score == local score."""
    b = synth.generate(1, 300, seed=4)
    for k in range(b.n):
        q, t = (x.decode() for x in b.pair(k))
        s, qe, te, qs, ts = oracle.start(q, t, 1, -4, 7, 1)
        if s == 0:
            continue
        cig, gs = oracle.traceback(q, t, ts, te, qs, qe, 1, -4, 7, 1)
        ops = expand(cig)
        assert gs == s
        assert score_ops(ops, t[ts:te + 1], q[qs:qe + 1], 1, -4, 7, 1) == s
        assert ops[0] == "M" and ops[-1] == "M"  # a local alignment starts and ends on a match


@pytest.mark.parametrize("L", [1, 5, 150])
def test_identical_is_one_run(L):
    rng = np.random.default_rng(L)
    s = "".join(rng.choice(list("ACGT"), L))
    assert oracle.traceback(s, s, 0, L - 1, 0, L - 1) == (f"{L}M", L)


def test_homopolymer_insertion_left_aligned():
    q, t = "ACGTTTTACG", "ACGTTTACG"
    assert oracle.traceback(q, t, 0, len(t) - 1, 0, len(q) - 1, 1, -4, 2, 1) == ("3M1I6M", 9 - 2)
    assert oracle.traceback(t, q, 0, len(q) - 1, 0, len(t) - 1, 1, -4, 2, 1) == ("3M1D6M", 9 - 2)
