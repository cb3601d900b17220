"""GPU parity of the cooperative long-pair kernel (dp_coop_kernel, DESIGN.md §4 A3 coop).

A long bin of few pairs (fewer than two waves of one-warp duos) runs on the cooperative kernel:
the warps of a block share each pair-duo, one 512-row chunk each, with the running maximum kept
in chunk order and pass 2 overlapping the next duo (§III-A load imbalance).
Bar: bit-exact score and end coordinates against the oracle, and bit-identical to the one-warp
long-bin kernel on the same batch (SALOBA_COOP_PAIRS=0 turns the cooperative kernel off).
"""
import os

import numpy as np
import pytest

import oracle
import synth
from test_gpu_parity import MODES, assert_same, gpu_align, oracle_align, sb  # noqa: F401

pytestmark = pytest.mark.gpu

COOP = 6  # long_group value of the cooperative kernel (saloba.h)


def run(sb, b, mode, fmt=4, coop=True):
    import torch

    lg = torch.zeros(1, dtype=torch.int32, device="cuda")
    bins = torch.zeros(16, dtype=torch.int32, device="cuda")
    old = os.environ.pop("SALOBA_COOP_PAIRS", None)
    if not coop:
        os.environ["SALOBA_COOP_PAIRS"] = "0"
    try:
        got = gpu_align(sb, b, sb.BWA_MEM, mode, sb.Options(bin_counts=bins, long_group=lg), fmt=fmt)
    finally:
        os.environ.pop("SALOBA_COOP_PAIRS", None)
        if old is not None:
            os.environ["SALOBA_COOP_PAIRS"] = old
    assert got[3] == -1
    return got, int(bins[13].item()), int(lg.item())


@pytest.mark.parametrize("mode", MODES)
def test_config4_every_pair(sb, mode):
    """Config-4 shapes (1-10 kbp, 15% errors): every pair against the oracle."""
    b = synth.generate(4, 240, seed=41 + mode)
    if mode == oracle.EXTEND:
        b.h0[:] = np.random.default_rng(5).integers(1, 60, b.n).astype(np.int32)
    got, n_long, lg = run(sb, b, mode)
    assert n_long > 0 and lg == COOP
    assert_same(got, oracle_align(b, sb.BWA_MEM, mode), b, f"coop config4 mode={mode}")


@pytest.mark.parametrize("mode", MODES)
def test_identical_to_one_warp_kernel(sb, mode):
    b = synth.generate(4, 900, seed=7)
    a, _, lg_a = run(sb, b, mode, coop=True)
    c, _, lg_c = run(sb, b, mode, coop=False)
    assert lg_a == COOP and lg_c in (4, 5)
    for x, y in zip(a[:3], c[:3]):
        assert np.array_equal(x, y)


def test_odd_count_pack2_and_mixed_shapes(sb):
    """Odd pair count (a dummy half), 2-bit packing, queries just over the long threshold
    (2048 bp), targets of one chunk (< 512 rows) and of many chunks in the same bin."""
    rng = np.random.default_rng(3)
    pairs = []
    acgt = np.frombuffer(b"ACGT", np.uint8)

    def rand_seq(n):
        return rng.choice(acgt, n).tobytes()

    for k in range(77):
        qlen = int(rng.choice([2048, 2049, 2100, 3000, 5000]))
        q = rand_seq(qlen)
        kind = k % 3
        if kind == 0:
            t = q[:300]                                   # one chunk, long query
        elif kind == 1:
            t = rand_seq(200) + q + rand_seq(100)
        else:
            mut = bytearray(q)
            for i in rng.choice(qlen, qlen // 20, replace=False):
                mut[i] = int(rng.choice(acgt))
            t = bytes(mut[: int(rng.integers(600, qlen))])
        pairs.append((q, t))
    b = synth.from_pairs(pairs, np.zeros(len(pairs), np.int32))
    for fmt in (4, 2):
        got, n_long, lg = run(sb, b, oracle.LOCAL, fmt=fmt)
        assert n_long >= b.n - 8 and lg == COOP  # (a few short-target pairs may take another bin)
        assert_same(got, oracle_align(b, sb.BWA_MEM, oracle.LOCAL), b, f"coop mixed fmt={fmt}")


def test_extend_floor_and_closed_form(sb):
    """EXTEND pairs whose best is the seed score h0 (no chunk improves: ends -1, -1), next to
    identical long pairs (closed form: len x match at the last cell)."""
    rng = np.random.default_rng(9)
    pairs, h0 = [], []
    for k in range(40):
        n = int(rng.integers(2100, 4000))
        q = rng.choice(np.frombuffer(b"ACGT", np.uint8), n).tobytes()
        if k % 2:
            pairs.append((q, q))
            h0.append(5)
        else:
            pairs.append((b"A" * n, b"C" * n))  # every cell a mismatch: nothing beats the seed score
            h0.append(100)
    b = synth.from_pairs(pairs, np.asarray(h0, np.int32))
    got, _, lg = run(sb, b, oracle.EXTEND)
    assert lg == COOP
    ref = oracle_align(b, sb.BWA_MEM, oracle.EXTEND)
    assert_same(got, ref, b, "coop extend floor")
    for k in range(1, b.n, 2):
        n = len(pairs[k][0])
        assert (got[0][k], got[1][k], got[2][k]) == (5 + n, n - 1, n - 1)
