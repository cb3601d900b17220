"""GPU parity of the BWA-MEM-compatible extension (saloba_ksw_extend) against the
pinned oracle (oracle/ksw.c): all seven outputs (score, qle, tle, gtle, gscore, max_off, clip)
compared element by element, bit-exact.  Inputs: random tiny pairs with random parameters (bands,
separate insertion/deletion costs, N), BWA-MEM defaults on configs 2 and 4 (sampled + longest for 4),
z-drop constructed cases, long queries (eh rows in global memory), PACK2, invalid data."""
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


def gpu_ksw(sb, b, params, fmt=4, max_qlen=None):
    import torch

    d = "cuda"
    t = [torch.from_numpy(x).to(d) for x in (b.q_ascii, b.q_off, b.t_ascii, b.t_off, b.h0)]
    out, st, qst, tst = sb.ksw_align(*t, params=params, fmt=fmt, max_qlen=max_qlen)
    torch.cuda.synchronize()
    assert int(qst.item()) == -1 and int(tst.item()) == -1
    return out.cpu().numpy(), int(st.item())


def oracle_ksw(b, params):
    kw = {k: getattr(params, k) for k in ("a", "b", "o_del", "e_del", "o_ins", "e_ins", "w", "end_bonus", "zdrop")}
    out, st = oracle.ksw_batch(b, **kw)
    assert (st == 0).all()
    return out


def assert_same(got, ref, b, label):
    bad = np.nonzero((got != ref).any(axis=0))[0]
    if len(bad):
        k = int(bad[0])
        q, t = b.pair(k)
        raise AssertionError(f"{label}: {len(bad)} mismatching pairs; first k={k} gpu={got[:, k].tolist()} "
                             f"oracle={ref[:, k].tolist()} fields={oracle.KSW_FIELDS} h0={b.h0[k]} "
                             f"q={q[:80]!r} t={t[:80]!r}")


def test_random_small_random_params(sb):
    rng = np.random.default_rng(101)
    for r in range(10):
        p = sb.KswParams(a=int(rng.integers(1, 4)), b=int(rng.integers(1, 6)), o_del=int(rng.integers(0, 9)),
                         e_del=int(rng.integers(1, 4)), o_ins=int(rng.integers(0, 9)), e_ins=int(rng.integers(1, 4)),
                         w=int(rng.integers(0, 40)), end_bonus=int(rng.integers(0, 10)),
                         zdrop=int(rng.choice([0, 5, 20, 100])))
        b = synth.random_pairs(1500, 1, 120, seed=500 + r, alphabet=b"ACGTACGTN", p_mut=0.1 if r % 2 else 0.0)
        b.h0[:] = rng.integers(1, 60, b.n)
        got, st = gpu_ksw(sb, b, p)
        assert st == -1
        assert_same(got, oracle_ksw(b, p), b, f"random r={r} {p}")


@pytest.mark.parametrize("cfg", [1, 2])
def test_bwa_defaults_config(sb, cfg):
    """BWA-MEM defaults (o 6, e 1, w 100, end_bonus 5, zdrop 100) on configs 1 and 2, every pair."""
    b = synth.generate(cfg, 200_000 if cfg == 2 else None)
    got, st = gpu_ksw(sb, b, sb.BWA_KSW)
    assert st == -1
    assert_same(got, oracle_ksw(b, sb.BWA_KSW), b, f"config{cfg}")


def test_bwa_defaults_config4_sampled(sb):
    """Long reads (1-10 kbp, 15% errors): eh rows in global memory; 400 pairs, every one compared."""
    b = synth.generate(4, 400, seed=44)
    got, st = gpu_ksw(sb, b, sb.BWA_KSW)
    assert st == -1
    assert_same(got, oracle_ksw(b, sb.BWA_KSW), b, "config4")


def test_zdrop_and_closed_forms(sb):
    """The hand-derived z-drop case of tests/test_oracle_ksw_pins.py and identical strings."""
    rng = np.random.default_rng(8)
    X = "".join(rng.choice(list("ACGT"), 50))
    Y = "".join(rng.choice(list("ACGT"), 200))
    s = X + "N" * 110 + Y
    idn = "".join(rng.choice(list("ACGT"), 150))
    b = synth.from_pairs([(s, s), (idn, idn), ("AAAA", "CCCC")], np.array([120, 19, 3], np.int32))
    got, st = gpu_ksw(sb, b, sb.BWA_KSW)
    assert st == -1
    assert got[:, 0].tolist() == [170, 50, 50, 0, -1, 0, 1]
    assert got[:, 1].tolist() == [169, 150, 150, 150, 169, 0, 0]
    assert got[:3, 2].tolist() == [3, 0, 0]
    got, _ = gpu_ksw(sb, b, sb.KswParams(zdrop=0))
    assert got[:, 0].tolist() == [260, 360, 360, 360, 260, 0, 0]


def test_long_queries_global_rows(sb):
    """Queries of 1,100-3,000 bp (> the shared-memory row capacity): per-warp rows in global memory."""
    b = synth.random_pairs(300, 1100, 3000, seed=77, p_mut=0.08)
    got, st = gpu_ksw(sb, b, sb.BWA_KSW)
    assert st == -1
    assert_same(got, oracle_ksw(b, sb.BWA_KSW), b, "long queries")


def test_pack2(sb):
    b = synth.random_pairs(2000, 1, 300, seed=9, p_mut=0.1)
    got, st = gpu_ksw(sb, b, sb.BWA_KSW, fmt=2)
    assert st == -1
    assert_same(got, oracle_ksw(b, sb.BWA_KSW), b, "pack2")


def test_invalid_pairs(sb):
    import torch

    b = synth.from_pairs([("ACGT", "ACGT"), ("", "ACGT"), ("ACGT", "ACGT")], np.array([5, 5, 0], np.int32))
    d = "cuda"
    t = [torch.from_numpy(x).to(d) for x in (b.q_ascii, b.q_off, b.t_ascii, b.t_off, b.h0)]
    out, st, _, _ = sb.ksw_align(*t)
    torch.cuda.synchronize()
    assert int(st.item()) == 1
    o = out.cpu().numpy()
    assert o[:, 0].tolist()[:3] == [9, 4, 4] and o[0, 1] == -1 and o[0, 2] == -1
