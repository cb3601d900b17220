"""Generator contract: determinism, slicing, shapes per config."""
import numpy as np

import oracle
import synth


def test_deterministic_and_sliceable():
    a = synth.generate(3, 500, seed=42)
    b = synth.generate(3, 500, seed=42)
    assert np.array_equal(a.q_ascii, b.q_ascii) and np.array_equal(a.t_ascii, b.t_ascii)
    assert np.array_equal(a.h0, b.h0)
    # per-pair streams: pairs 200..299 generated alone are identical to the slice
    c = synth.generate(3, 100, seed=42, first=200, n_total=500)
    for k in range(100):
        assert c.pair(k) == a.pair(200 + k)
    assert synth.generate(3, 50, seed=43).pair(0) != a.pair(0)


def test_config_shapes():
    q, t, h0 = synth.shapes(2, 5000)
    assert (q == 150).all() and (t == 250).all()
    assert h0.min() >= 19 and h0.max() <= 50
    q, t, _ = synth.shapes(1, 5000)
    assert (q == 150).all() and t.min() >= 140 and t.max() <= 260
    q, t, _ = synth.shapes(3, 20000)
    assert q.min() >= 100 and q.max() <= 999 and (t >= q - 10).all()
    # log-uniform: about half the mass below the geometric mean sqrt(100*1000) = 316
    assert 0.45 < (q < 316).mean() < 0.55
    q, t, _ = synth.shapes(4, 2000)
    assert q.min() >= 1000 and q.max() <= 10000
    q, t, _ = synth.shapes(5, 100000)
    assert q.min() >= 25 and q.max() <= 10000
    assert 0.85 < (q < 275).mean() < 0.95


def test_alphabet_and_n_injection():
    b = synth.generate(1, 300)
    assert set(np.unique(b.q_ascii).tolist()) <= set(b"ACGT")
    bn = synth.generate(1, 300, p_n=0.01)
    frac = (bn.q_ascii == ord("N")).mean()
    assert 0.004 < frac < 0.02


def test_alignability():
    """SPEC S:444-446 / acceptance 8 analogue: simulated config-2 reads align with high score."""
    b = synth.generate(2, 400, seed=1)
    s, _, _, st, _ = oracle.align_batch(b, threads=4)
    assert (st == 0).all()
    assert (s >= 100).mean() > 0.97
