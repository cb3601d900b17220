"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bar: bit-exact score, q_end and t_end (integer path).  Inputs are seeded: tiny
exhaustive sets, randomized pairs with randomized schemes, every BASELINE config (full config 1;
full-size configs 2-5 in the bench's launch configuration, compared on deterministic samples),
and the edge cases (empty batch, 1-base pairs, N-rich pairs, invalid data, 2-bit packing).
"""
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


def to_dev(batch):
    import torch

    d = "cuda"
    return (torch.from_numpy(batch.q_ascii).to(d), torch.from_numpy(batch.q_off).to(d),
            torch.from_numpy(batch.t_ascii).to(d), torch.from_numpy(batch.t_off).to(d),
            torch.from_numpy(batch.h0).to(d))


def gpu_align(sb, batch, scoring=None, mode=0, options=None, fmt=4):
    import torch

    scoring = scoring or sb.BWA_MEM
    qa, qo, ta, to, h0 = to_dev(batch)
    s, qe, te, st, qst, tst = sb.align(qa, qo, ta, to, h0 if mode == sb.EXTEND else None, scoring, mode, fmt,
                                       options=options)
    torch.cuda.synchronize()
    return s.cpu().numpy(), qe.cpu().numpy(), te.cpu().numpy(), int(st.item()), int(qst.item()), int(tst.item())


def oracle_align(batch, scoring, mode, threads=None):
    s, qe, te, st, _ = oracle.align_batch(batch, scoring.match, scoring.mismatch, scoring.gap_open,
                                          scoring.gap_extend, mode, threads=threads)
    assert (st == 0).all()
    return s, qe, te


def assert_same(got, ref, batch, label):
    s, qe, te = got[:3]
    rs, rq, rt = ref
    bad = np.nonzero((s != rs) | (qe != rq) | (te != rt))[0]
    if len(bad):
        k = int(bad[0])
        q, t = batch.pair(k)
        raise AssertionError(f"{label}: {len(bad)} mismatches; first k={k} gpu=({s[k]},{qe[k]},{te[k]}) "
                             f"oracle=({rs[k]},{rq[k]},{rt[k]}) q={q[:80]!r} t={t[:80]!r} h0={batch.h0[k]}")


# ---- A1 pack ---------------------------------------------------------------------------------
def test_pack_spec_examples(sb):
    import torch

    b = synth.from_pairs([("ACGTN", "AAAAAAAA"), ("ACGTACGT", "acgtacgtu"), ("A" * 9, "N")])
    qa, qo, ta, to, _ = to_dev(b)
    w, wo, ln, st = sb.pack(qa, qo)
    torch.cuda.synchronize()
    w = w.cpu().numpy().view(np.uint32)
    wo = wo.cpu().numpy()
    assert int(st.item()) == -1
    assert w[wo[0]] == 0xFFF43210  # S:50 "ACGTN" -> codes 0,1,2,3,4 then padding 15
    assert w[wo[1]] == 0x32103210
    assert w[wo[2]] == 0 and w[wo[2] + 1] == 0xFFFFFFF0  # 9 bases -> 2 words, 7 padding nibbles
    assert ln.cpu().tolist() == [5, 8, 9]
    w2, wo2, _, st2 = sb.pack(ta, to)
    torch.cuda.synchronize()
    w2 = w2.cpu().numpy().view(np.uint32)
    wo2 = wo2.cpu().numpy()
    assert w2[wo2[0]] == 0x00000000
    assert w2[wo2[1]] == 0x32103210 and w2[wo2[1] + 1] == 0xFFFFFFF3  # lowercase + U -> T
    assert w2[wo2[2]] == 0xFFFFFFF4


def test_pack_random_vs_host_packer(sb):
    import torch

    rng = np.random.default_rng(0)
    b = synth.random_pairs(3000, 1, 300, seed=1, alphabet=b"ACGTNacgtnUu")
    qa, qo, _, _, _ = to_dev(b)
    for fmt in (4,):
        w, wo, ln, st = sb.pack(qa, qo, fmt)
        torch.cuda.synchronize()
        w = w.cpu().numpy().view(np.uint32)
        wo = wo.cpu().numpy()
        code = np.full(256, 255, np.uint8)
        for ch, c in zip(b"ACGTUNacgtun", [0, 1, 2, 3, 3, 4, 0, 1, 2, 3, 3, 4]):
            code[ch] = c
        for k in rng.choice(b.n, 300, replace=False):
            q = np.frombuffer(b.pair(int(k))[0], np.uint8)
            cs = code[q]
            nw = (len(cs) + 7) // 8
            exp = np.full(nw * 8, 15, np.uint32)
            exp[:len(cs)] = cs
            expw = (exp.reshape(nw, 8) << (4 * np.arange(8, dtype=np.uint32))).sum(1).astype(np.uint32)
            assert np.array_equal(w[wo[k]:wo[k] + nw], expw)
    del rng


def _host_pack(ascii, off, fmt):
    """Plain numpy packer (A1 layout): sequence s at word off[s]//B + s, codes LSB-first,
    padding 15 (4-bit) / 0 (2-bit)."""
    B = 8 if fmt == 4 else 16
    code = np.full(256, 255, np.uint8)
    for ch, c in zip(b"ACGTUacgtu", [0, 1, 2, 3, 3, 0, 1, 2, 3, 3]):
        code[ch] = c
    if fmt == 4:
        code[ord("N")] = code[ord("n")] = 4
    out = {}
    for s in range(len(off) - 1):
        cs = code[ascii[off[s]:off[s + 1]]].astype(np.uint32)
        nw = (len(cs) + B - 1) // B
        exp = np.full(nw * B, 15 if fmt == 4 else 0, np.uint32)
        exp[:len(cs)] = cs
        bits = 4 if fmt == 4 else 2
        out[int(off[s] // B + s)] = (exp.reshape(nw, B) << (bits * np.arange(B, dtype=np.uint32))).sum(1).astype(np.uint32)
    return out


@pytest.mark.parametrize("fmt", [4, 2])
@pytest.mark.parametrize("shift", [0, 3, 13])
def test_pack_every_sequence_any_alignment(sb, fmt, shift):
    """Every word of every sequence against a host packer: lengths 0-40 (more sequence ends than
    lanes in a 512-byte window), 100-300 and 2-9 kbp, the ASCII buffer starting at an address that
    is not 16-byte aligned, and offsets that do not start at 0 (a slice of a larger batch)."""
    import torch

    rng = np.random.default_rng(fmt * 10 + shift)
    alpha = np.frombuffer(b"ACGTacgtUu" + (b"Nn" if fmt == 4 else b""), np.uint8)
    lens = np.concatenate([rng.integers(0, 41, 3000), rng.integers(100, 301, 1500), rng.integers(2000, 9000, 20)])
    rng.shuffle(lens)
    lead = 37  # bytes before the first sequence
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64) + lead
    ascii = rng.choice(alpha, int(off[-1])).astype(np.uint8)
    buf = torch.zeros(len(ascii) + 64, dtype=torch.uint8, device="cuda")
    dev = buf[shift:shift + len(ascii)]
    dev.copy_(torch.from_numpy(ascii))
    w, wo, ln, st = sb.pack(dev, torch.from_numpy(off).cuda(), fmt)
    torch.cuda.synchronize()
    assert int(st.item()) == -1
    w = w.cpu().numpy().view(np.uint32)
    wo = wo.cpu().numpy()
    assert ln.cpu().tolist() == lens.tolist()
    exp = _host_pack(ascii, off, fmt)
    for s in range(len(lens)):
        e = exp[int(wo[s])]
        assert np.array_equal(w[wo[s]:wo[s] + len(e)], e), (s, lens[s])


def test_pack_invalid_base_reported(sb):
    import torch

    b = synth.from_pairs([("ACGT", "ACGT"), ("ACXT", "ACGT"), ("AC-T", "ACGT")])
    qa, qo, _, _, _ = to_dev(b)
    _, _, _, st = sb.pack(qa, qo)
    torch.cuda.synchronize()
    assert int(st.item()) == 6  # first invalid byte: 'X' at global byte 4+2
    b2 = synth.from_pairs([("ACGN", "ACGT")])
    qa, qo, _, _, _ = to_dev(b2)
    _, _, _, st = sb.pack(qa, qo, sb.PACK2)  # N is not representable in 2 bits
    torch.cuda.synchronize()
    assert int(st.item()) == 3


# ---- A2-A4 DP parity -------------------------------------------------------------------------
@pytest.mark.parametrize("mode", MODES)
def test_exhaustive_len_1_to_4(sb, mode):
    """All 115,600 ordered pairs of ACGT strings of lengths 1..4 (SPEC acceptance 1)."""
    strs = ["".join(p) for L in (1, 2, 3, 4) for p in itertools.product("ACGT", repeat=L)]
    pairs = [(q, t) for q in strs for t in strs]
    b = synth.from_pairs(pairs, np.full(len(pairs), 3, np.int32))
    sc = sb.Scoring(1, -4, 2, 1)
    assert_same(gpu_align(sb, b, sc, mode), oracle_align(b, sc, mode), b, f"exhaustive mode={mode}")


@pytest.mark.parametrize("mode", MODES)
def test_randomized_schemes_1_to_512(sb, mode):
    """>= 10,000 random pairs of 1-512 bp, schemes from SPEC acceptance 2's ranges."""
    rng = np.random.default_rng(2023 + mode)
    for r in range(12):
        beta = int(rng.integers(1, 4))
        sc = sb.Scoring(int(rng.integers(1, 5)), int(rng.integers(-6, 0)), int(rng.integers(beta, 9)), beta)
        b = synth.random_pairs(900, 1, 512, seed=100 * r + mode, p_mut=0.1 if r % 2 else 0.0)
        assert_same(gpu_align(sb, b, sc, mode), oracle_align(b, sc, mode), b, f"random r={r} {sc}")


@pytest.mark.parametrize("mode", MODES)
def test_n_rich_pairs(sb, mode):
    b = synth.random_pairs(2000, 1, 200, seed=5, alphabet=b"ACGTNN", p_mut=0.05)
    sc = sb.BWA_MEM
    assert_same(gpu_align(sb, b, sc, mode), oracle_align(b, sc, mode), b, "N-rich")


@pytest.mark.parametrize("mode", MODES)
def test_config1_full(sb, mode):
    b = synth.generate(1)
    assert_same(gpu_align(sb, b, sb.BWA_MEM, mode), oracle_align(b, sb.BWA_MEM, mode), b, "config1")
    bn = synth.generate(1, seed=11, p_n=0.005)  # parity-only N set (§8(d))
    assert_same(gpu_align(sb, bn, sb.BWA_MEM, mode), oracle_align(bn, sb.BWA_MEM, mode), bn, "config1+N")


@pytest.mark.parametrize("G", [1, 2, 4, 8, 16, 32])
def test_bit_identical_across_group_size(sb, G):
    b = synth.random_pairs(1500, 1, 400, seed=77, p_mut=0.08)
    ref = oracle_align(b, sb.BWA_MEM, oracle.LOCAL)
    assert_same(gpu_align(sb, b, sb.BWA_MEM, 0, sb.Options(force_group=G)), ref, b, f"G={G}")
    ref = oracle_align(b, sb.BWA_MEM, oracle.EXTEND)
    assert_same(gpu_align(sb, b, sb.BWA_MEM, 1, sb.Options(force_group=G)), ref, b, f"G={G} extend")


def test_order_and_path_invariance(sb):
    b = synth.generate(3, 3000, seed=9)
    base = gpu_align(sb, b, sb.BWA_MEM, 0)
    for opt in (sb.Options(keep_order=1), sb.Options(force_path=1), sb.Options(force_path=2)):
        got = gpu_align(sb, b, sb.BWA_MEM, 0, opt)
        assert all(np.array_equal(x, y) for x, y in zip(base[:3], got[:3])), opt
    # permuting the batch permutes the results
    perm = np.random.default_rng(0).permutation(b.n)
    bp = b.subset(perm)
    got = gpu_align(sb, bp, sb.BWA_MEM, 0)
    assert all(np.array_equal(x[perm], y) for x, y in zip(base[:3], got[:3]))


@pytest.mark.parametrize("mode", MODES)
def test_pack2_path(sb, mode):
    b = synth.random_pairs(1500, 1, 300, seed=31, p_mut=0.1)
    ref = oracle_align(b, sb.BWA_MEM, mode)
    assert_same(gpu_align(sb, b, sb.BWA_MEM, mode, fmt=2), ref, b, "pack2")


def test_edge_cases(sb):
    import torch

    # empty batch
    b = synth.from_pairs([])
    qa, qo, ta, to, h0 = to_dev(b)
    s, qe, te, st, _, _ = sb.align(qa, qo, ta, to)
    torch.cuda.synchronize()
    assert s.numel() == 0 and int(st.item()) == -1
    # single bases, exact multiples of 8, one-off lengths
    pairs = [("A", "A"), ("A", "C"), ("N", "N"), ("ACGTACGT", "ACGTACGT"), ("ACGTACGTA", "ACGTACGT"),
             ("A" * 257, "A" * 255), ("ACGT" * 64, "TGCA" * 64)]
    b = synth.from_pairs(pairs, np.array([1, 5, 9, 3, 2, 40, 7], np.int32))
    for mode in MODES:
        assert_same(gpu_align(sb, b, sb.BWA_MEM, mode), oracle_align(b, sb.BWA_MEM, mode), b, "edge")


def test_invalid_pairs_reported(sb):
    import torch

    b = synth.from_pairs([("ACGT", "ACGT"), ("", "ACGT"), ("ACGT", ""), ("AC", "AC")],
                         np.array([5, 5, 5, 0], np.int32))
    qa, qo, ta, to, h0 = to_dev(b)
    s, qe, te, st, _, _ = sb.align(qa, qo, ta, to)
    torch.cuda.synchronize()
    assert int(st.item()) == 1
    assert s.cpu().tolist() == [4, -1, -1, 2]
    assert qe.cpu().tolist()[1:3] == [-2, -2]
    s, qe, te, st, _, _ = sb.align(qa, qo, ta, to, h0, mode=sb.EXTEND)  # h0 = 0 is invalid for pair 3
    torch.cuda.synchronize()
    assert int(st.item()) == 1 and s.cpu().tolist() == [9, -1, -1, -1]


def test_large_scores_int32_envelope(sb):
    """match 1024 x 3000 bp identical reads: scores ~3e6 exceed int16, int32 path exact."""
    rng = np.random.default_rng(4)
    q = "".join(rng.choice(list("ACGT"), 3000))
    t = q[:1000] + "GATTACA" + q[1000:]
    b = synth.from_pairs([(q, t), (q, q)], np.array([100000, 7], np.int32))
    sc = sb.Scoring(1024, -1024, 1024, 1)
    for mode in MODES:
        assert_same(gpu_align(sb, b, sc, mode), oracle_align(b, sc, mode), b, "big")


# ---- full-size configs in the bench's launch configuration, sampled -----------------------------
def _sample_check(sb, cfg, n=None, sample=3000, mode=0, seed=None):
    b = synth.generate(cfg, n, seed=seed)
    got = gpu_align(sb, b, sb.BWA_MEM, mode)
    assert got[3] == -1
    rng = np.random.default_rng(cfg)
    idx = np.sort(rng.choice(b.n, min(sample, b.n), replace=False))
    # include the longest pairs too (they exercise the most chunks / spill rows)
    longest = np.argsort(b.qlen.astype(np.int64) * b.tlen)[-20:]
    idx = np.unique(np.concatenate([idx, longest]))
    sub = b.subset(idx)
    ref = oracle_align(sub, sb.BWA_MEM, mode)
    assert_same(tuple(x[idx] for x in got[:3]), ref, sub, f"config{cfg} sample")


@pytest.mark.parametrize("mode", MODES)
def test_config2_full_size_sampled(sb, mode):
    _sample_check(sb, 2, mode=mode)


def test_config3_full_size_sampled(sb):
    _sample_check(sb, 3, sample=2000)


def test_config4_sampled(sb):
    _sample_check(sb, 4, n=2000, sample=40)


@pytest.mark.parametrize("n_long", [2_000, 12_000, 40_000])
def test_long_bin_width_rule(sb, n_long):
    """The int16x2 long bin (DESIGN.md §4 A2) runs on the cooperative kernel below two waves of
    one-warp duos, at G=32 for a few waves of long pairs and at G=16 once it holds >= 4 waves of
    G=16 subwarps; every choice is checked on sampled outputs."""
    import torch

    b = synth.generate(4, n_long, seed=11)
    lg = torch.zeros(1, dtype=torch.int32, device="cuda")
    bins = torch.zeros(16, dtype=torch.int32, device="cuda")
    got = gpu_align(sb, b, sb.BWA_MEM, 0, sb.Options(bin_counts=bins, long_group=lg))
    assert got[3] == -1
    assert int(bins[13].item()) > 0
    assert int(lg.item()) == (4 if n_long >= 40_000 else 5 if n_long >= 12_000 else 6)
    rng = np.random.default_rng(n_long)
    idx = np.unique(np.concatenate([rng.choice(b.n, 24, replace=False),
                                    np.argsort(b.qlen.astype(np.int64) * b.tlen)[-4:]]))
    sub = b.subset(idx)
    assert_same(tuple(x[idx] for x in got[:3]), oracle_align(sub, sb.BWA_MEM, 0), sub, f"long bin n={n_long}")


def test_config5_sampled(sb):
    _sample_check(sb, 5, n=300_000, sample=3000)


def test_host_entry_point_matches_device_path(sb):
    b = synth.generate(3, 5000, seed=3)
    dev = gpu_align(sb, b, sb.BWA_MEM, 1)
    s, qe, te, st = sb.align_host(b, sb.BWA_MEM, sb.EXTEND)
    assert st == -1
    assert np.array_equal(s, dev[0]) and np.array_equal(qe, dev[1]) and np.array_equal(te, dev[2])


def test_host_context_reuse_offsets_and_errors(sb):
    b = synth.generate(1, 800, seed=21)
    dev = gpu_align(sb, b, sb.BWA_MEM, 0)
    ctx = sb.HostContext(1000, len(b.q_ascii) + 100, len(b.t_ascii) + 100, 300)
    for _ in range(2):  # reuse
        s, qe, te, st = sb.align_host(b, sb.BWA_MEM, sb.LOCAL, ctx=ctx)
        assert st == -1 and np.array_equal(s, dev[0]) and np.array_equal(qe, dev[1]) and np.array_equal(te, dev[2])
    # a sub-batch whose offsets do not start at 0 (pairs 100..399 of the same buffers)
    sub = synth.Batch(b.q_ascii, b.q_off[100:401], b.t_ascii, b.t_off[100:401], b.h0[100:400])
    s, qe, te, st = sb.align_host(sub, sb.BWA_MEM, sb.LOCAL, ctx=ctx)
    assert st == -1 and np.array_equal(s, dev[0][100:400]) and np.array_equal(te, dev[2][100:400])
    # an invalid base in pair 523 and an empty target in pair 611 -> status = 523
    bad = synth.from_pairs([b.pair(k) for k in range(b.n)], b.h0)
    bad.q_ascii[bad.q_off[523] + 5] = ord("X")
    s, qe, te, st = sb.align_host(bad, sb.BWA_MEM, sb.LOCAL, ctx=ctx)
    assert st == 523
    # capacity exceeded -> SalobaError(EWORKSPACE)
    big = synth.generate(1, 1200, seed=3)
    with pytest.raises(sb.SalobaError):
        sb.align_host(big, sb.BWA_MEM, sb.LOCAL, ctx=ctx)
    ctx.close()


@pytest.mark.parametrize("mode", MODES)
def test_query_n_bin(sb, mode):
    """Reads with N in the query run on the int16x2 G=1 QN variant (bin 14: an N column's
    substitution forced to mismatch), bit-exact vs the oracle; N in the target only needs no bin."""
    import torch

    b = synth.generate(2, 120_000, seed=41, p_n=0.002)  # enough pairs to fill the GPU at G = 1
    bins = torch.zeros(16, dtype=torch.int32, device="cuda")
    got = gpu_align(sb, b, sb.BWA_MEM, mode, sb.Options(bin_counts=bins))
    bc = bins.cpu().tolist()
    assert bc[14] > 10000 and bc[8] > 10000 and sum(bc[0:8]) == 0, bc
    assert_same(got, oracle_align(b, sb.BWA_MEM, mode), b, f"query-N bin mode={mode}")


def test_long_identical_pair_closed_form(sb):
    """Maximum-size direction: one 50 kbp identical pair (score beyond int16 -> int32 long bin,
    2.5e9 cells on one subwarp) against the closed form (L, L-1, L-1); EXTEND adds h0."""
    rng = np.random.default_rng(50)
    L = 50_000
    q = "".join(rng.choice(list("ACGT"), L))
    b = synth.from_pairs([(q, q), ("ACGT", "ACGT")], np.array([5, 5], np.int32))
    got = gpu_align(sb, b, sb.BWA_MEM, 0)
    assert got[3] == -1 and (got[0][0], got[1][0], got[2][0]) == (L, L - 1, L - 1)
    got = gpu_align(sb, b, sb.BWA_MEM, 1)
    assert got[3] == -1 and (got[0][0], got[1][0], got[2][0]) == (L + 5, L - 1, L - 1)


def test_length_beyond_envelope_is_invalid(sb):
    """Lengths > 2^20 (the S:151 int32 envelope) are invalid data: status = first such pair."""
    import torch

    big = "A" * ((1 << 20) + 1)
    b = synth.from_pairs([("ACGT", "ACGT"), ("ACGT", big), ("AC", "AC")])
    d = "cuda"
    qa, qo = torch.from_numpy(b.q_ascii).to(d), torch.from_numpy(b.q_off).to(d)
    ta, to = torch.from_numpy(b.t_ascii).to(d), torch.from_numpy(b.t_off).to(d)
    s, qe, te, st, qst, tst = sb.align(qa, qo, ta, to, max_qlen=64)
    torch.cuda.synchronize()
    assert int(st.item()) == 1 and s.cpu().tolist() == [4, -1, 2]


def test_small_batch_latency_floor(sb):
    """Batches too small to fill the GPU at G = 1 get a latency floor on G (api.cu): 1,000 pairs run
    at G = 32 (long bin), a full-size batch stays at G = 1; results identical either way."""
    import torch

    b = synth.generate(1)
    bins = torch.zeros(16, dtype=torch.int32, device="cuda")
    got = gpu_align(sb, b, sb.BWA_MEM, 0, sb.Options(bin_counts=bins))
    bc = bins.cpu().tolist()
    assert bc[13] == b.n, bc
    assert_same(got, oracle_align(b, sb.BWA_MEM, 0), b, "small batch")


@pytest.mark.parametrize("mode", MODES)
def test_query_n_bin_g2(sb, mode):
    """Mid-length reads with N in the query (config 3 shapes) take the QN variant at G = 2 (bin 6)."""
    import torch

    b = synth.generate(3, 150_000, seed=43, p_n=0.002)
    bins = torch.zeros(16, dtype=torch.int32, device="cuda")
    got = gpu_align(sb, b, sb.BWA_MEM, mode, sb.Options(bin_counts=bins))
    bc = bins.cpu().tolist()
    assert bc[6] > 1000 and bc[14] > 1000, bc
    rng = np.random.default_rng(43 + mode)
    idx = np.sort(rng.choice(b.n, 4000, replace=False))
    idx = np.unique(np.concatenate([idx, np.nonzero(b.qlen > 640)[0][:500]]))
    sub = b.subset(idx)
    assert_same(tuple(x[idx] for x in got[:3]), oracle_align(sub, sb.BWA_MEM, mode), sub, f"QN G=2 mode={mode}")


def test_pack_capacity_overflow_reported(sb):
    """saloba_pack with a words buffer one word short of the closed-form layout (total/8 + n words:
    sequence s ends at or before word byte_off[s+1]/8 + s + 1): nothing is written and the status is
    byte_off[n] (one past the last byte); exactly total/8 + n words packs normally."""
    import ctypes

    import torch

    b = synth.random_pairs(50, 5, 40, seed=3)
    qa, qo = torch.from_numpy(b.q_ascii).cuda(), torch.from_numpy(b.q_off).cuda()
    n = b.n
    need = len(b.q_ascii) // 8 + n
    assert sb.packed_words(len(b.q_ascii), n) == need + 1  # the advertised capacity keeps one spare word
    for cap, expect in ((need - 1, len(b.q_ascii)), (need, -1)):
        words = torch.full((need,), 0x7777, dtype=torch.int32, device="cuda")
        wo = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        st = torch.empty(1, dtype=torch.int64, device="cuda")
        rc = sb.lib().saloba_pack(ctypes.c_void_p(qa.data_ptr()), ctypes.c_void_p(qo.data_ptr()), n, 4,
                                  ctypes.c_void_p(words.data_ptr()), cap, ctypes.c_void_p(wo.data_ptr()), None,
                                  ctypes.c_void_p(st.data_ptr()), None)
        torch.cuda.synchronize()
        assert rc == 0 and int(st.item()) == expect
        if expect != -1:
            assert bool((words == 0x7777).all())


def test_host_stream_pipelined_batches(sb):
    """saloba_stream_*: three different batches in flight two at a time give the same results as
    the device path; an invalid base in the third batch is reported through its own status."""
    import ctypes

    import torch

    batches = [synth.generate(1, 700, seed=s) for s in (31, 32, 33)]
    bad = synth.from_pairs([batches[2].pair(k) for k in range(batches[2].n)], batches[2].h0)
    bad.q_ascii[bad.q_off[412] + 3] = ord("X")
    batches[2] = bad
    cap_q = max(len(b.q_ascii) for b in batches) + 64
    cap_t = max(len(b.t_ascii) for b in batches) + 64
    hs = sb.HostStream(800, cap_q, cap_t, 300)
    outs = [torch.empty((3, b.n), dtype=torch.int32, pin_memory=True).numpy() for b in batches]
    sts = [ctypes.c_int64(99) for _ in batches]
    for b, o, st in zip(batches, outs, sts):
        hs.submit(b, o, st, sb.BWA_MEM, sb.EXTEND)
    hs.wait()
    assert [st.value for st in sts] == [-1, -1, 412]
    for b, o in zip(batches[:2], outs[:2]):
        dev = gpu_align(sb, b, sb.BWA_MEM, 1)
        assert all(np.array_equal(o[i], dev[i]) for i in range(3))
    hs.close()
