"""GPU parity at the precision-routing boundaries and in the regimes round 1 left untested.

The int16x2 kernels are exact only under the routing bound of SURVEY §8(c) reading 8 / DESIGN.md §4
(LOCAL: match*min(m,n) + match <= 32767; EXTEND: lambda*(h0 + match*min(m,n)) + match <= 32767,
lambda = 2^k >= match + 1) and only for calls whose match/mismatch fit int8 (their substitution rows
are int8 bytes).  The FAST int32 kernels pack D*9 + column keys and need lambda*B + match < 2^27
(schedule.cu).  Each test sits exactly on one side of one bound, asserts the bin the scheduler chose
(through Options.bin_counts) and compares every output with the oracle (bit-exact).
Bins: int32 FAST 0..5 (log2 G), QN2 6, int32 wide 7, int16x2 8..13, QN 14 (common.cuh).
"""
import numpy as np
import pytest

import oracle
import synth

from test_gpu_parity import assert_same, gpu_align, oracle_align

pytestmark = pytest.mark.gpu

I32_BINS = list(range(0, 6)) + [7]
I16_BINS = list(range(8, 15)) + [6]


@pytest.fixture(scope="module")
def sb():
    import torch

    import build_native

    build_native.build_saloba()
    import paper_2301_09310_b200 as sb

    torch.cuda.init()
    return sb


def run_bins(sb, b, sc, mode):
    import torch

    bins = torch.zeros(16, dtype=torch.int32, device="cuda")
    got = gpu_align(sb, b, sc, mode, sb.Options(bin_counts=bins))
    assert got[3] == -1
    return got, bins.cpu().tolist()


def mutated(rng, s, p):
    out = list(s)
    for i in range(len(out)):
        if rng.random() < p:
            out[i] = "ACGT"[(("ACGT".index(out[i])) + int(rng.integers(1, 4))) % 4]
    return "".join(out)


# ---- scores that do not fit int8 never take the int16x2 kernels ----------------
@pytest.mark.parametrize("mode", [oracle.LOCAL, oracle.EXTEND])
@pytest.mark.parametrize("scheme", [(200, -4, 7, 1), (1, -200, 7, 1), (128, -3, 9, 2), (3, -129, 5, 2)])
def test_scores_beyond_int8_route_int32(sb, mode, scheme):
    sc = sb.Scoring(*scheme)
    b = synth.random_pairs(600, 60, 140, seed=300 + scheme[0] - scheme[1], p_mut=0.08, alphabet=b"ACGTACGTACGTN")
    got, bc = run_bins(sb, b, sc, mode)
    assert sum(bc[b_] for b_ in I16_BINS) == 0, bc
    assert_same(got, oracle_align(b, sc, mode), b, f"int8-overflow scheme {scheme} mode={mode}")


@pytest.mark.parametrize("mode", [oracle.LOCAL, oracle.EXTEND])
def test_int8_limit_scores_stay_int16(sb, mode):
    """match 127 / mismatch -128 are the largest int8 scores: still the int16x2 path, still exact."""
    sc = sb.Scoring(127, -128, 127, 1)
    rng = np.random.default_rng(5)
    pairs = []
    for _ in range(400):
        L = int(rng.integers(20, 120))
        q = "".join(rng.choice(list("ACGT"), L))
        pairs.append((q, mutated(rng, q, 0.1)))
    b = synth.from_pairs(pairs, rng.integers(1, 60, len(pairs)).astype(np.int32))
    got, bc = run_bins(sb, b, sc, mode)
    if mode == oracle.LOCAL:  # EXTEND: lambda = 128 puts every pair beyond the int16 bound
        assert sum(bc[b_] for b_ in I16_BINS) == b.n, bc
    assert_same(got, oracle_align(b, sc, mode), b, f"int8 limit mode={mode}")


# ---- LOCAL int16x2 bound: match*L + match = 32767 (int16x2) vs 32774 (int32) ----------------------
@pytest.mark.parametrize("L,expect_i16", [(4680, True), (4681, False)])
def test_local_bound_edge(sb, L, expect_i16):
    """match 7: 7*4680 + 7 = 32767 exactly (the largest int16x2 pair); 4681 bp is one past it."""
    sc = sb.Scoring(7, -4, 7, 1)
    rng = np.random.default_rng(L)
    q = "".join(rng.choice(list("ACGT"), L))
    pairs = [(q, q), (q, mutated(rng, q, 0.01)), (mutated(rng, q, 0.02), q), (q[::-1], q)]
    b = synth.from_pairs(pairs, np.full(len(pairs), 3, np.int32))
    got, bc = run_bins(sb, b, sc, oracle.LOCAL)
    n16 = sum(bc[b_] for b_ in I16_BINS)
    assert (n16 == len(pairs)) if expect_i16 else (n16 == 0), bc
    # identical pair: closed form (7L at (L-1, L-1)); everything against the oracle
    assert (got[0][0], got[1][0], got[2][0]) == (7 * L, L - 1, L - 1)
    assert_same(got, oracle_align(b, sc, oracle.LOCAL), b, f"LOCAL bound L={L}")


# ---- EXTEND int16x2 bound: lambda*(h0 + match*L) + match = 32767 vs 32769 / 32771 -----------------
@pytest.mark.parametrize("match,L,h0,expect_i16", [(1, 1000, 15383, True), (1, 1000, 15384, False),
                                                   (3, 2000, 2191, True), (3, 2000, 2192, False)])
def test_extend_bound_edge(sb, match, L, h0, expect_i16):
    """match 1 (lambda 2): 2*(15383 + 1000) + 1 = 32767; match 3 (lambda 4): 4*(2191 + 6000) + 3 = 32767."""
    sc = sb.Scoring(match, -4, 7, 1)
    rng = np.random.default_rng(L + h0)
    q = "".join(rng.choice(list("ACGT"), L))
    pairs = [(q, q), (q, mutated(rng, q, 0.02)), ("T" * 5 + q[5:], q), (q[: L // 2], q)]
    # the last pair has min(m, n) = L/2, so it is comfortably inside the bound either way
    b = synth.from_pairs(pairs, np.full(len(pairs), h0, np.int32))
    got, bc = run_bins(sb, b, sc, oracle.EXTEND)
    n16 = sum(bc[b_] for b_ in I16_BINS)
    assert (n16 == len(pairs)) if expect_i16 else (n16 == 1), bc
    assert (got[0][0], got[1][0], got[2][0]) == (h0 + match * L, L - 1, L - 1)
    assert_same(got, oracle_align(b, sc, oracle.EXTEND), b, f"EXTEND bound match={match} h0={h0}")


# ---- FAST int32 bound: lambda*B + match < 2^27 (FAST bins) vs >= 2^27 (wide bin 7) -----------------
@pytest.mark.parametrize("h0,wide", [(67108763, False), (67108764, True)])
def test_fast_int32_key_bound(sb, h0, wide):
    """match 1, 100 bp: 2*(h0 + 100) + 1 = 134217727 (< 2^27, FAST) / 134217729 (>= 2^27, wide bin)."""
    sc = sb.Scoring(1, -4, 7, 1)
    rng = np.random.default_rng(h0)
    q = "".join(rng.choice(list("ACGT"), 100))
    pairs = [(q, q), (q, mutated(rng, q, 0.05)), (mutated(rng, q, 0.1), q[3:] + "ACG")]
    b = synth.from_pairs(pairs, np.full(len(pairs), h0, np.int32))
    got, bc = run_bins(sb, b, sc, oracle.EXTEND)
    assert sum(bc[b_] for b_ in I16_BINS) == 0, bc
    if wide:
        assert bc[7] == len(pairs), bc  # min(m, n) = 100 for all three pairs
    else:
        assert bc[7] == 0 and sum(bc[0:6]) == len(pairs), bc
    assert (got[0][0], got[1][0], got[2][0]) == (h0 + 100, 99, 99)
    assert_same(got, oracle_align(b, sc, oracle.EXTEND), b, f"FAST int32 bound h0={h0}")


# ---- EXTEND on long reads (int16x2 with lambda*H ~ 2e4), configs 3 and 5 --------------------------
def _sampled(sb, cfg, n, mode, sample, n_longest=20, seed=None):
    b = synth.generate(cfg, n, seed=seed)
    got, bc = run_bins(sb, b, sb.BWA_MEM, mode)
    rng = np.random.default_rng(1000 + cfg)
    idx = np.sort(rng.choice(b.n, min(sample, b.n), replace=False))
    longest = np.argsort(b.qlen.astype(np.int64) * b.tlen)[-n_longest:]
    idx = np.unique(np.concatenate([idx, longest]))
    sub = b.subset(idx)
    assert_same(tuple(x[idx] for x in got[:3]), oracle_align(sub, sb.BWA_MEM, mode), sub,
                f"config{cfg} n={n} mode={mode}")
    return b, got, bc


def test_extend_config4_int16(sb):
    """Config-4 shapes in EXTEND route to the int16x2 long bin (lambda*(h0 + 10 kbp) ~ 2e4 < 32767)."""
    b, got, bc = _sampled(sb, 4, 3000, oracle.EXTEND, sample=40, n_longest=6)
    assert sum(bc[b_] for b_ in I16_BINS) == b.n, bc


def test_extend_config3_sampled(sb):
    _sampled(sb, 3, None, oracle.EXTEND, sample=3000)


def test_extend_config5_sampled(sb):
    _sampled(sb, 5, 300_000, oracle.EXTEND, sample=3000)


# ---- every pair of configs 2 and 3 (SURVEY §4 / BASELINE.md §3: full comparison for configs 1-3) ---
@pytest.mark.parametrize("mode", [oracle.LOCAL, oracle.EXTEND])
def test_config2_every_pair(sb, mode):
    b = synth.generate(2)
    got = gpu_align(sb, b, sb.BWA_MEM, mode)
    assert got[3] == -1
    assert_same(got, oracle_align(b, sb.BWA_MEM, mode), b, f"config2 full mode={mode}")


def test_config3_every_pair(sb):
    b = synth.generate(3)
    got = gpu_align(sb, b, sb.BWA_MEM, oracle.LOCAL)
    assert got[3] == -1
    assert_same(got, oracle_align(b, sb.BWA_MEM, oracle.LOCAL), b, "config3 full")
