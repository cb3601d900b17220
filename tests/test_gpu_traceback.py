"""GPU parity of the CIGAR traceback (saloba_traceback) against the pinned
oracle (oracle/traceback.c), string for string, on the LOCAL results of the GPU path itself (ends
from saloba_align_batch, starts from saloba_locate_start — both already bit-exact to their oracles).
"""
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


def gpu_cigars(sb, b, scoring, cap=96, fmt=4, score_override=None):
    import torch

    d = "cuda"
    qa, qo = torch.from_numpy(b.q_ascii).to(d), torch.from_numpy(b.q_off).to(d)
    ta, to = torch.from_numpy(b.t_ascii).to(d), torch.from_numpy(b.t_off).to(d)
    qw, qwo, ql, _ = sb.pack(qa, qo, fmt)
    tw, two, tl, _ = sb.pack(ta, to, fmt)
    s, qe, te, st = sb.align_batch(qw, qwo[:-1], ql, tw, two[:-1], tl, None, scoring, sb.LOCAL, fmt)
    qs, ts, sst = sb.locate_start(qw, qwo[:-1], tw, two[:-1], s, qe, te, scoring, fmt)
    torch.cuda.synchronize()
    assert int(st.item()) == -1 and int(sst.item()) == -1
    if score_override is not None:
        s = score_override(s)
    cig, n_ops, tst = sb.traceback(qw, qwo[:-1], tw, two[:-1], s, qs, qe, ts, te, scoring, fmt, cigar_cap=cap)
    torch.cuda.synchronize()
    res = dict(score=s.cpu().numpy(), q_end=qe.cpu().numpy(), t_end=te.cpu().numpy(), q_start=qs.cpu().numpy(),
               t_start=ts.cpu().numpy())
    return sb.cigar_strings(cig, n_ops), int(tst.item()), res


def check(b, cigars, res, scoring, label):
    for k in range(b.n):
        if res["score"][k] == 0:
            assert cigars[k] == "", (label, k)
            continue
        q, t = (x.decode() for x in b.pair(k))
        want, gs = oracle.traceback(q, t, int(res["t_start"][k]), int(res["t_end"][k]), int(res["q_start"][k]),
                                    int(res["q_end"][k]), scoring.match, scoring.mismatch, scoring.gap_open,
                                    scoring.gap_extend)
        assert gs == res["score"][k], (label, k)
        assert cigars[k] == want, (label, k, cigars[k], want, q[:60], t[:60])


def test_config1_every_pair(sb):
    b = synth.generate(1)
    cig, st, res = gpu_cigars(sb, b, sb.BWA_MEM)
    assert st == -1
    check(b, cig, res, sb.BWA_MEM, "config1")


def test_config2_sample(sb):
    b = synth.generate(2, 20_000, seed=12)
    cig, st, res = gpu_cigars(sb, b, sb.BWA_MEM)
    assert st == -1
    check(b, cig, res, sb.BWA_MEM, "config2")


@pytest.mark.parametrize("r", range(6))
def test_random_schemes_with_n(sb, r):
    """Random pairs (1-200 bp, N included) under random schemes, alpha == beta included."""
    rng = np.random.default_rng(900 + r)
    beta = int(rng.integers(1, 4))
    alpha = beta if r % 3 == 0 else int(rng.integers(beta, 9))
    sc = sb.Scoring(int(rng.integers(1, 4)), int(rng.integers(-6, 0)), alpha, beta)
    b = synth.random_pairs(1500, 1, 200, seed=700 + r, alphabet=b"ACGTACGTN", p_mut=0.12)
    cig, st, res = gpu_cigars(sb, b, sc, cap=256)
    assert st == -1
    check(b, cig, res, sc, f"random r={r} {sc}")


def test_long_regions_workspace_path(sb):
    """Regions of 300-900 rows (beyond the 256-row shared-memory limit): per-warp workspace slots."""
    b = synth.random_pairs(40, 300, 900, seed=33, p_mut=0.06)
    cig, st, res = gpu_cigars(sb, b, sb.BWA_MEM, cap=512)
    assert st == -1
    assert (res["t_end"] - res["t_start"] + 1).max() > 256
    check(b, cig, res, sb.BWA_MEM, "long regions")


def test_inconsistent_score_and_overflow_reported(sb):
    b = synth.generate(1, 200, seed=3)

    def bump(s):
        s = s.clone()
        s[17] += 1  # a score the region cannot reach: reported, pair 17 is the first such
        return s

    _, st, res = gpu_cigars(sb, b, sb.BWA_MEM, score_override=bump)
    assert st == 17 or res["score"][17] == 0
    cig, st, res = gpu_cigars(sb, b, sb.BWA_MEM, cap=1)  # one element cannot hold an indel CIGAR
    multi = []
    for k in range(b.n):
        if res["score"][k] > 0:
            q, t = (x.decode() for x in b.pair(k))
            want, _ = oracle.traceback(q, t, int(res["t_start"][k]), int(res["t_end"][k]), int(res["q_start"][k]),
                                       int(res["q_end"][k]))
            if sum(ch.isalpha() for ch in want) > 1:
                multi.append(k)
    assert multi and st == multi[0] and all(cig[k] is None for k in multi)
