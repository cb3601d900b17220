"""GPU parity of the banded DP on the int16x2 G = 1 kernel (dp_g1.cu BAND variant; SURVEY §8(f) NEXT-2,
DESIGN.md reading 16): bit-exact to the banded oracle (pinned in test_oracle_banded_pins.py), with
the bin the scheduler chose asserted (bin 8 = int16x2 G = 1).  Covers band edges inside and across
8x8 blocks and 16-row strips, w = 0, bands past the table, different bands in the two halves of a
duo, EXTEND (boundary row and column unchanged by the band), PACK2, config 2 every pair with BWA-MEM's
w = 100, and config-4 long reads (whose band rows are indexed per strip)."""
import numpy as np
import pytest

import oracle
import synth

from test_gpu_banded import assert_same, gpu_banded, oracle_banded

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


def banded_bins(sb, b, w, mode, fmt=4):
    import torch

    bins = torch.zeros(16, dtype=torch.int32, device="cuda")
    # force_path = 2: the int16x2 band kernel even for batches too small to fill the GPU at G = 1
    got = gpu_banded(sb, b, w, sb.BWA_MEM, mode, sb.Options(force_path=2, bin_counts=bins), fmt=fmt)
    return got, bins.cpu().tolist()


@pytest.mark.parametrize("mode", MODES)
def test_random_bands(sb, mode):
    b = synth.random_pairs(3000, 1, 400, seed=61 + mode, p_mut=0.08)
    w = np.random.default_rng(7 + mode).choice(np.array([0, 1, 2, 7, 8, 9, 15, 16, 17, 31, 33, 64, 100, 5000], np.int32),
                                               b.n)
    got, bc = banded_bins(sb, b, w, mode)
    assert got[3] == -1 and bc[8] == b.n, bc
    assert_same(got, oracle_banded(b, w, sb.BWA_MEM, mode), b, w, f"i16 band mode={mode}")


def test_extend_large_h0_and_pack2(sb):
    rng = np.random.default_rng(91)
    b = synth.random_pairs(3000, 10, 200, seed=91, p_mut=0.05)
    b.h0[:] = rng.integers(1, 150, b.n).astype(np.int32)
    w = rng.integers(0, 40, b.n).astype(np.int32)
    got, bc = banded_bins(sb, b, w, sb.EXTEND)
    assert bc[8] == b.n, bc
    assert_same(got, oracle_banded(b, w, sb.BWA_MEM, oracle.EXTEND), b, w, "EXTEND h0")
    got, bc = banded_bins(sb, b, w, sb.LOCAL, fmt=2)
    assert bc[8] == b.n, bc
    assert_same(got, oracle_banded(b, w, sb.BWA_MEM, oracle.LOCAL), b, w, "pack2")


@pytest.mark.parametrize("mode", MODES)
def test_config2_every_pair_w100(sb, mode):
    b = synth.generate(2, 200_000, seed=2)
    w = np.full(b.n, 100, np.int32)
    got, bc = banded_bins(sb, b, w, mode)
    assert got[3] == -1 and bc[8] == b.n, bc
    assert_same(got, oracle_banded(b, w, sb.BWA_MEM, mode), b, w, f"config2 w=100 mode={mode}")


def test_config4_long_reads_w100(sb):
    """1-10 kbp reads: Q up to 1250 blocks, band rows of ~31 blocks indexed per strip."""
    b = synth.generate(4, 400, seed=14)
    w = np.full(b.n, 100, np.int32)
    got, bc = banded_bins(sb, b, w, sb.LOCAL)
    assert got[3] == -1 and bc[8] == b.n, bc
    rng = np.random.default_rng(14)
    cells = (b.qlen.astype(np.int64) + 1) * (b.tlen + 1)
    idx = np.sort(rng.choice(np.nonzero(cells < (1 << 26))[0], 60, replace=False))
    sub = b.subset(idx)
    assert_same(tuple(x[idx] for x in got[:3]), oracle_banded(sub, w[idx], sb.BWA_MEM, 0), sub, w[idx], "config4")


def test_wide_bands_take_int32(sb):
    """Bands whose rows would exceed the G = 1 kernel's 80-block spill rows go to the int32 kernel."""
    b = synth.random_pairs(500, 700, 900, seed=5, p_mut=0.05)
    w = np.full(b.n, 400, np.int32)
    got, bc = banded_bins(sb, b, w, sb.LOCAL)
    assert bc[8] == 0 and sum(bc[0:8]) == b.n, bc
    assert_same(got, oracle_banded(b, w, sb.BWA_MEM, 0), b, w, "wide band int32")


def test_small_batch_of_long_banded_reads_takes_int32(sb):
    """Without force_path, a batch too small to fill the GPU at one lane per pair keeps the int32
    banded kernel (G >= 2 spreads each pair over several lanes)."""
    import torch

    b = synth.generate(4, 300, seed=15)
    w = np.full(b.n, 100, np.int32)
    bins = torch.zeros(16, dtype=torch.int32, device="cuda")
    got = gpu_banded(sb, b, w, sb.BWA_MEM, sb.LOCAL, sb.Options(bin_counts=bins))
    bc = bins.cpu().tolist()
    assert got[3] == -1 and bc[8] == 0 and sum(bc[0:8]) == b.n, bc


def test_split_pass2_extend_halves_at_different_strips(sb):
    """Regression (round-2 stress): a duo whose halves win in different strips (here strip 5 and
    strip 0) runs pass 2 over the union of both band ranges, which starts before the first block the
    strip above the later half ever wrote.  Those top-row blocks are left of its band and must read
    as H = F = 0; read as stale memory they reached the other half through EXTEND's 32-bit
    lambda * hdiag product (scheme 3/-2/7/3, w = 40, seeds as tools/repro_band.py found them)."""
    import torch

    full = synth.generate(2, 20000, seed=7, p_n=0.002)
    full.h0[:] = np.random.default_rng(7).integers(1, 80, full.n).astype(np.int32)
    b = full.subset([18510, 18511])
    sc = sb.Scoring(3, -2, 7, 3)
    w = np.full(b.n, 40, np.int32)
    bins = torch.zeros(16, dtype=torch.int32, device="cuda")
    got = gpu_banded(sb, b, w, sc, sb.EXTEND, sb.Options(force_path=2, keep_order=1, bin_counts=bins))
    assert int(bins[8].item()) == 2
    assert_same(got, oracle_banded(b, w, sc, oracle.EXTEND), b, w, "split pass 2")
