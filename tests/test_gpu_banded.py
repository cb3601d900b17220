"""GPU parity of the banded DP (saloba_align_banded) vs the oracle's banded
definition (oracle.banded_batch, pinned in test_oracle_banded_pins.py): bit-exact score and ends,
through the C ABI, both modes, every subwarp size, band edges inside and across 8x8 blocks."""
import itertools

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
MODES = [oracle.LOCAL, oracle.EXTEND]


@pytest.fixture(scope="module")
def sb():
    import torch

    import build_native

    build_native.build_saloba()
    import paper_2301_09310_b200 as sb

    torch.cuda.init()
    return sb


def gpu_banded(sb, batch, w, scoring=None, mode=0, options=None, fmt=4):
    import torch

    scoring = scoring or sb.BWA_MEM
    d = "cuda"
    qa, qo = torch.from_numpy(batch.q_ascii).to(d), torch.from_numpy(batch.q_off).to(d)
    ta, to = torch.from_numpy(batch.t_ascii).to(d), torch.from_numpy(batch.t_off).to(d)
    qw, qwo, ql, _ = sb.pack(qa, qo, fmt)
    tw, two, tl, _ = sb.pack(ta, to, fmt)
    h0 = torch.from_numpy(batch.h0).to(d) if mode == sb.EXTEND else None
    wd = torch.from_numpy(np.ascontiguousarray(w, np.int32)).to(d)
    s, qe, te, st = sb.align_banded(qw, qwo[:-1], ql, tw, two[:-1], tl, wd, h0, scoring, mode, fmt, options=options)
    torch.cuda.synchronize()
    return s.cpu().numpy(), qe.cpu().numpy(), te.cpu().numpy(), int(st.item())


def oracle_banded(batch, w, sc, mode):
    s, qe, te, st = oracle.banded_batch(batch, w, sc.match, sc.mismatch, sc.gap_open, sc.gap_extend, mode)
    assert (st == 0).all(), np.unique(st)
    return s, qe, te


def assert_same(got, ref, batch, w, label):
    bad = np.nonzero((got[0] != ref[0]) | (got[1] != ref[1]) | (got[2] != ref[2]))[0]
    if len(bad):
        k = int(bad[0])
        q, t = batch.pair(k)
        raise AssertionError(f"{label}: {len(bad)} mismatches; first k={k} w={w[k]} gpu=({got[0][k]},{got[1][k]},"
                             f"{got[2][k]}) oracle=({ref[0][k]},{ref[1][k]},{ref[2][k]}) q={q[:60]!r} t={t[:60]!r}")


@pytest.mark.parametrize("mode", MODES)
def test_banded_exhaustive_len_1_to_4(sb, mode):
    strs = ["".join(p) for L in (1, 2, 3, 4) for p in itertools.product("ACGT", repeat=L)]
    pairs = [(q, t) for q in strs for t in strs]
    b = synth.from_pairs(pairs, np.full(len(pairs), 3, np.int32))
    w = np.arange(len(pairs), dtype=np.int32) % 4  # bands 0..3
    sc = sb.Scoring(1, -4, 2, 1)
    got = gpu_banded(sb, b, w, sc, mode)
    assert got[3] == -1
    assert_same(got, oracle_banded(b, w, sc, mode), b, w, f"exhaustive mode={mode}")


@pytest.mark.parametrize("mode", MODES)
def test_banded_random_schemes_and_bands(sb, mode):
    rng = np.random.default_rng(1728 + mode)
    for r in range(8):
        beta = int(rng.integers(1, 4))
        sc = sb.Scoring(int(rng.integers(1, 5)), int(rng.integers(-6, 0)), int(rng.integers(beta, 9)), beta)
        b = synth.random_pairs(900, 1, 512, seed=300 + r, p_mut=0.1 if r % 2 else 0.0)
        w = rng.integers(0, 80, b.n).astype(np.int32)
        got = gpu_banded(sb, b, w, sc, mode)
        assert got[3] == -1
        assert_same(got, oracle_banded(b, w, sc, mode), b, w, f"random r={r} {sc}")


@pytest.mark.parametrize("G", [1, 2, 4, 8, 16, 32])
def test_banded_across_group_size(sb, G):
    """The exact int32 banded kernel at every G (force_path=1; int16x2-eligible banded pairs otherwise
    take the int16x2 G = 1 BAND kernel, tested in test_gpu_banded_i16.py)."""
    b = synth.random_pairs(800, 1, 600, seed=79, p_mut=0.08)
    w = np.random.default_rng(G).integers(0, 120, b.n).astype(np.int32)
    for mode in MODES:
        got = gpu_banded(sb, b, w, sb.BWA_MEM, mode, sb.Options(force_group=G, force_path=1))
        assert_same(got, oracle_banded(b, w, sb.BWA_MEM, mode), b, w, f"G={G} mode={mode}")


def test_wide_band_equals_unbanded_path(sb):
    import torch

    b = synth.generate(3, 3000, seed=12)
    w = np.full(b.n, 100000, np.int32)
    for mode in MODES:
        got = gpu_banded(sb, b, w, sb.BWA_MEM, mode)
        d = "cuda"
        s, qe, te, st, _, _ = sb.align(torch.from_numpy(b.q_ascii).to(d), torch.from_numpy(b.q_off).to(d),
                                       torch.from_numpy(b.t_ascii).to(d), torch.from_numpy(b.t_off).to(d),
                                       torch.from_numpy(b.h0).to(d) if mode else None, sb.BWA_MEM, mode)
        torch.cuda.synchronize()
        assert np.array_equal(got[0], s.cpu().numpy()) and np.array_equal(got[1], qe.cpu().numpy())
        assert np.array_equal(got[2], te.cpu().numpy())


def test_banded_n_rich_pack2_and_invalid(sb):
    b = synth.random_pairs(1500, 1, 200, seed=6, alphabet=b"ACGTNN", p_mut=0.05)
    w = np.random.default_rng(2).integers(0, 30, b.n).astype(np.int32)
    for mode in MODES:
        assert_same(gpu_banded(sb, b, w, sb.BWA_MEM, mode), oracle_banded(b, w, sb.BWA_MEM, mode), b, w, "N-rich")
    b2 = synth.random_pairs(1500, 1, 300, seed=33, p_mut=0.1)
    w2 = np.random.default_rng(3).integers(0, 50, b2.n).astype(np.int32)
    assert_same(gpu_banded(sb, b2, w2, fmt=2), oracle_banded(b2, w2, sb.BWA_MEM, 0), b2, w2, "pack2")
    b3 = synth.from_pairs([("ACGT", "ACGT"), ("ACGT", "ACGT"), ("AC", "AC")])
    got = gpu_banded(sb, b3, np.array([0, -1, 5], np.int32))
    assert got[3] == 1 and got[0].tolist() == [4, -1, 2]


@pytest.mark.parametrize("mode", MODES)
def test_banded_long_reads_sampled(sb, mode):
    """config-4 shaped pairs (1-10 kbp, 15% errors) with BWA-MEM's default band w = 100."""
    b = synth.generate(4, 600, seed=4)
    w = np.full(b.n, 100, np.int32)
    got = gpu_banded(sb, b, w, sb.BWA_MEM, mode)
    assert got[3] == -1
    cells = (b.qlen.astype(np.int64) + 1) * (b.tlen + 1)
    rng = np.random.default_rng(5)
    cand = np.nonzero(cells < (1 << 26))[0]
    idx = np.sort(rng.choice(cand, min(40, len(cand)), replace=False))
    sub = b.subset(idx)
    ref = oracle_banded(sub, w[idx], sb.BWA_MEM, mode)
    assert_same(tuple(x[idx] for x in got[:3]), ref, sub, w[idx], f"config4 banded mode={mode}")


def test_banded_extend_large_h0_band_left_edge(sb):
    """EXTEND with large h0 and bands whose left edge falls exactly on a block boundary: the first
    in-band cell of a strip must see an out-of-band (zero) left neighbour, not the H(i,-1)
    boundary of column -1 (a stale-boundary bug would show up here)."""
    rng = np.random.default_rng(88)
    b = synth.random_pairs(3000, 20, 120, seed=88, p_mut=0.05)
    b.h0[:] = rng.integers(40, 120, b.n).astype(np.int32)
    w = rng.choice(np.array([0, 1, 8, 9, 16, 24], np.int32), b.n)
    for G in (None, 2, 8):
        opt = sb.Options(force_group=G, force_path=1) if G else None
        got = gpu_banded(sb, b, w, sb.BWA_MEM, sb.EXTEND, opt)
        assert_same(got, oracle_banded(b, w, sb.BWA_MEM, oracle.EXTEND), b, w, f"left edge G={G}")
