"""NEXT-4: the paper's structural laws reproduced as device counters of the int16x2
kernels (saloba_options.counters), exactly:

* step law (§IV-A, SPEC acceptance 3): a chunk of G strips takes Q + G - 1
  wavefront steps (Q + 31 at G = 32); the dedicated G = 1 kernel takes Q;
* lazy spill ("reduces the amount of intermediate data access to 1/32", SPEC acceptance 4
  and 9): chunk-bottom rows produced at G are 1/G of those an every-strip spill produces; the rows
  actually spilled are (chunks - 1) x Q blocks per work item;
* stored volume (Table II `tab:moti` P:549-568, "Stored 2N + N^2/4", SPEC acceptance 5): with
  16-row strips and 16-bit H and F, an N x N pair spills (N/16 - 1) x N x 4 bytes = N^2/4 - 4N.
Every run is also checked against the oracle."""
import numpy as np
import pytest

import oracle
import synth

from test_gpu_parity import assert_same, gpu_align, oracle_align

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import torch

    import build_native

    build_native.build_saloba()
    import paper_2301_09310_b200 as sb

    torch.cuda.init()
    return sb


def run_counted(sb, b, G, mode=0):
    import torch

    ctr = torch.zeros(8, dtype=torch.int64, device="cuda")
    bins = torch.zeros(16, dtype=torch.int32, device="cuda")
    got = gpu_align(sb, b, sb.BWA_MEM, mode, sb.Options(force_group=G, bin_counts=bins, counters=ctr))
    assert got[3] == -1
    assert_same(got, oracle_align(b, sb.BWA_MEM, mode), b, f"counted G={G}")
    bc = bins.cpu().tolist()
    assert sum(bc[8:14]) == b.n and bc[8 + int(np.log2(G))] == b.n, bc  # every pair on the int16x2 G bin
    return [int(x) for x in ctr.cpu().tolist()]


def same_shape_pairs(n, qlen, tlen, seed):
    rng = np.random.default_rng(seed)
    pairs = []
    for _ in range(n):
        q = "".join(rng.choice(list("ACGT"), qlen))
        t = "".join(rng.choice(list("ACGT"), tlen - qlen)) + q
        pairs.append((q, t))
    return synth.from_pairs(pairs, np.full(n, 20, np.int32))


@pytest.mark.parametrize("G", [1, 2, 4, 8, 16, 32])
def test_step_law(sb, G):
    """64 pairs of 200 x 300 bp (32 work items): Q = 25 blocks, 19 strips, ceil(19/G) chunks."""
    b = same_shape_pairs(64, 200, 300, seed=G)
    c = run_counted(sb, b, G)
    Q, strips = 25, 19
    chunks = -(-strips // G)
    items = 32
    assert c[7] == items
    assert c[0] == items * chunks
    assert c[1] == items * chunks * (Q if G == 1 else Q + G - 1)  # Q + 31 at G = 32
    assert c[6] == items * chunks * G
    assert c[2] == items * (chunks - 1) * Q
    if G > 1:
        assert c[1] * G - c[0] * Q * G == c[0] * (G - 1) * G  # utilisation Q / (Q + G - 1)


def test_lazy_spill_is_one_over_G(sb):
    """SPEC acceptance 4 on a 2048 x 2048 duo (two identical pairs) at G = 32: 128 strips of 16 rows,
    Q = 256 blocks, 4 chunks; chunk-bottom rows produced = 1/32 of the strips (the rows an eager,
    every-strip spill would produce), rows spilled = 3 boundaries x Q blocks, steps = 4 x (Q + 31)."""
    rng = np.random.default_rng(2048)
    q = "".join(rng.choice(list("ACGT"), 2048))
    b = synth.from_pairs([(q, q), (q, q)])
    c = run_counted(sb, b, 32)
    Q, strips = 256, 128
    assert c[6] == strips and c[0] * 32 == c[6]
    assert c[2] == (strips // 32 - 1) * Q
    assert c[1] == (strips // 32) * (Q + 31)


def test_spill_g1_vs_g32(sb):
    """The same 640 x 1024 duo at G = 1 (every strip spills: 63 boundaries) and G = 32 (2 chunks: 1
    boundary): spilled blocks 63 x 80 vs 1 x 80; rows produced 64 vs 2 = 1/32 (G = 1 takes queries
    up to 640 bp: its spill rows are sized for 80 blocks)."""
    rng = np.random.default_rng(640)
    q = "".join(rng.choice(list("ACGT"), 640))
    t = "".join(rng.choice(list("ACGT"), 384)) + q
    b = synth.from_pairs([(q, t), (q, t)])
    base, lazy = run_counted(sb, b, 1), run_counted(sb, b, 32)
    assert base[0] == 64 and lazy[0] == 2 and lazy[0] * 32 == base[0]
    assert base[2] == 63 * 80 and lazy[2] == 1 * 80


@pytest.mark.parametrize("N", [64, 256, 640])
def test_stored_volume_table2(sb, N):
    """G = 1 (queries up to 640 bp): spilled bytes per pair = (N/16 - 1) x N x 4 = N^2/4 - 4N (Table
    II's N^2/4 term)."""
    rng = np.random.default_rng(N)
    q = "".join(rng.choice(list("ACGT"), N))
    t = "".join(rng.choice(list("ACGT"), N))
    b = synth.from_pairs([(q, t), (t, q)])
    c = run_counted(sb, b, 1)
    stored_per_pair = c[2] * 64 // 2  # a 64-byte block holds 8 columns of (H, F) for both halves
    assert stored_per_pair == (N // 16 - 1) * N * 4 == N * N // 4 - 4 * N
