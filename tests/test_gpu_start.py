"""GPU parity of the start coordinates (LOCAL, saloba_locate_start) vs the
oracle's start (oracle.start_batch, pinned in test_oracle_start_pins.py): bit-exact score, ends and
starts, through the C ABI, on the same seeded inputs as the forward parity tests."""
import itertools

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import torch

    import build_native

    build_native.build_saloba()
    import paper_2301_09310_b200 as sb

    torch.cuda.init()
    return sb


def gpu_start(sb, batch, scoring=None, options=None, fmt=4):
    """pack -> align_batch (LOCAL) -> locate_start; returns 5 numpy arrays + the two statuses."""
    import torch

    scoring = scoring or sb.BWA_MEM
    d = "cuda"
    qa, qo = torch.from_numpy(batch.q_ascii).to(d), torch.from_numpy(batch.q_off).to(d)
    ta, to = torch.from_numpy(batch.t_ascii).to(d), torch.from_numpy(batch.t_off).to(d)
    qw, qwo, ql, _ = sb.pack(qa, qo, fmt)
    tw, two, tl, _ = sb.pack(ta, to, fmt)
    s, qe, te, st = sb.align_batch(qw, qwo[:-1], ql, tw, two[:-1], tl, None, scoring, sb.LOCAL, fmt, options=options)
    qs, ts, st2 = sb.locate_start(qw, qwo[:-1], tw, two[:-1], s, qe, te, scoring, fmt, options=options)
    torch.cuda.synchronize()
    out = tuple(x.cpu().numpy() for x in (s, qe, te, qs, ts))
    return out, int(st.item()), int(st2.item())


def oracle_start(batch, sc):
    out = oracle.start_batch(batch, sc.match, sc.mismatch, sc.gap_open, sc.gap_extend)
    assert (out[5] == 0).all()
    return out[:5]


def assert_same(got, ref, batch, label):
    names = ("score", "q_end", "t_end", "q_start", "t_start")
    bad = np.zeros(len(got[0]), bool)
    for g, r in zip(got, ref):
        bad |= g != r
    idx = np.nonzero(bad)[0]
    if len(idx):
        k = int(idx[0])
        q, t = batch.pair(k)
        raise AssertionError(f"{label}: {len(idx)} mismatches; first k={k} gpu={[int(g[k]) for g in got]} "
                             f"oracle={[int(r[k]) for r in ref]} ({names}) q={q[:80]!r} t={t[:80]!r}")


def test_start_exhaustive_len_1_to_4(sb):
    strs = ["".join(p) for L in (1, 2, 3, 4) for p in itertools.product("ACGT", repeat=L)]
    b = synth.from_pairs([(q, t) for q in strs for t in strs])
    sc = sb.Scoring(1, -4, 2, 1)
    got, st, st2 = gpu_start(sb, b, sc)
    assert st == -1 and st2 == -1
    assert_same(got, oracle_start(b, sc), b, "exhaustive")


def test_start_randomized_schemes(sb):
    rng = np.random.default_rng(31)
    for r in range(8):
        beta = int(rng.integers(1, 4))
        sc = sb.Scoring(int(rng.integers(1, 5)), int(rng.integers(-6, 0)), int(rng.integers(beta, 9)), beta)
        b = synth.random_pairs(900, 1, 512, seed=700 + r, p_mut=0.1 if r % 2 else 0.0)
        got, st, st2 = gpu_start(sb, b, sc)
        assert st == -1 and st2 == -1
        assert_same(got, oracle_start(b, sc), b, f"random r={r} {sc}")


def test_start_n_rich_and_config1(sb):
    b = synth.random_pairs(2000, 1, 200, seed=5, alphabet=b"ACGTNN", p_mut=0.05)
    got, _, st2 = gpu_start(sb, b)
    assert st2 == -1
    assert_same(got, oracle_start(b, sb.BWA_MEM), b, "N-rich")
    for bb in (synth.generate(1), synth.generate(1, seed=11, p_n=0.005)):
        got, _, st2 = gpu_start(sb, bb)
        assert st2 == -1
        assert_same(got, oracle_start(bb, sb.BWA_MEM), bb, "config1")


@pytest.mark.parametrize("G", [1, 4, 32])
def test_start_across_group_size_and_paths(sb, G):
    b = synth.random_pairs(1200, 1, 400, seed=78, p_mut=0.08)
    ref = oracle_start(b, sb.BWA_MEM)
    got, _, st2 = gpu_start(sb, b, options=sb.Options(force_group=G))
    assert st2 == -1
    assert_same(got, ref, b, f"G={G}")
    got, _, _ = gpu_start(sb, b, options=sb.Options(force_group=G, force_path=1))
    assert_same(got, ref, b, f"G={G} int32")


def test_start_pack2_and_edges(sb):
    b = synth.random_pairs(1500, 1, 300, seed=32, p_mut=0.1)
    got, _, _ = gpu_start(sb, b, fmt=2)
    assert_same(got, oracle_start(b, sb.BWA_MEM), b, "pack2")
    pairs = [("A", "A"), ("A", "C"), ("N", "N"), ("AAAA", "TTTT"), ("ACGTACGT", "ACGTACGT"),
             ("ACGTACGTA", "ACGTACGT"), ("A" * 257, "A" * 255), ("ACGT" * 64, "TGCA" * 64),
             ("NNNN" + "ACGTTGCAAC" * 3 + "NN", "NNNNNNN" + "ACGTTGCAAC" * 3)]
    b = synth.from_pairs(pairs)
    got, _, st2 = gpu_start(sb, b)
    assert st2 == -1
    assert_same(got, oracle_start(b, sb.BWA_MEM), b, "edges")
    assert (int(got[3][-1]), int(got[4][-1])) == (4, 7)  # planted core between N flanks


def test_start_invalid_pairs(sb):
    b = synth.from_pairs([("ACGT", "ACGT"), ("", "ACGT"), ("AC", "AC")])
    got, st, st2 = gpu_start(sb, b)
    assert st == 1 and st2 == -1
    assert got[3].tolist() == [0, -2, 0] and got[4].tolist() == [0, -2, 0]


@pytest.mark.parametrize("cfg,n,sample", [(2, None, 3000), (3, 100_000, 1500), (4, 1000, 30)])
def test_start_full_size_sampled(sb, cfg, n, sample):
    b = synth.generate(cfg, n)
    got, st, st2 = gpu_start(sb, b)
    assert st == -1 and st2 == -1
    rng = np.random.default_rng(cfg + 40)
    idx = np.sort(rng.choice(b.n, min(sample, b.n), replace=False))
    idx = np.unique(np.concatenate([idx, np.argsort(b.qlen.astype(np.int64) * b.tlen)[-10:]]))
    sub = b.subset(idx)
    assert_same(tuple(x[idx] for x in got), oracle_start(sub, sb.BWA_MEM), sub, f"config{cfg} start sample")
