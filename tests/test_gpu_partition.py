"""A5 on the GPU: saloba_partition vs the test reference of its assignment (bit-exact ranks), the
balance target of SURVEY §8(e) (max/mean modelled cost <= 1.02 on config 5, grouped order
included), and the multi-rank bench path (2 ranks sharing one GPU over gloo, balanced shards,
results gathered to rank 0)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import synth
from test_dist_gloo import snake_reference

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sb():
    import torch

    import build_native

    build_native.build_saloba()
    import paper_2301_09310_b200 as sb

    torch.cuda.init()
    return sb


@pytest.mark.parametrize("grouped", [False, True])
def test_partition_matches_reference_and_balances(sb, grouped):
    from paper_2301_09310_b200 import dist as sd

    ql, tl, _ = synth.shapes(5, 300_000, grouped=grouped)
    cost = sd.pair_cost(ql, tl)
    for world in (1, 2, 3, 4, 8):
        owner = sd.balanced_partition(ql, tl, world)
        assert np.array_equal(owner, snake_reference(ql, tl, world)), world
        assert sd.imbalance(cost, owner, world) <= 1.02
    assert sb.partition.__doc__


def test_partition_edge_cases(sb):
    import torch

    e = torch.empty(0, dtype=torch.int32, device="cuda")
    assert sb.partition(e, e, 4).numel() == 0
    q = torch.tensor([5, 5, 5], dtype=torch.int32, device="cuda")
    assert sb.partition(q, q, 8).cpu().tolist() == [0, 1, 2]  # equal costs keep input order
    with pytest.raises(sb.SalobaError):
        sb.partition(q, q, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_balanced_shards(sb):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--dist-backend", "gloo", "--config", "5", "--pairs", "20000", "--grouped", "--no-cpu-baseline",
           "--e2e-steps", "0", "--start-steps", "0"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert "length-balanced" in line["config"]["partition"]
    assert line["config"]["measured_rank_balance_max_over_mean"] >= 1.0


def _bench(args, nproc, timeout=900):
    if nproc > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", str(nproc),
               "--dist-backend", "gloo"]
    else:
        cmd = [sys.executable, "bench.py", "--gpus", "1"]
    cmd += ["--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "0", "--start-steps", "0",
            "--no-graph"] + args
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])


@pytest.mark.parametrize("partition", ["balanced", "equal"])
def test_sharded_results_reassembled_in_input_order(sb, tmp_path, partition):
    """A5 end to end: config 5 grouped (the worst case for an equal split),
    strong scaling, 2 ranks sharing one GPU over gloo.  Rank 0 gathers the shards and puts them back
    in input order with saloba_scatter_results inside the timed step; the reassembled results must be
    identical to a 1-rank run of the same global batch (S:292, S:496 results independent of
    sharding) and to the oracle on a sample (+ the longest pairs)."""
    import oracle
    from test_gpu_parity import assert_same, oracle_align

    n = 40_000
    common = ["--config", "5", "--pairs", str(n), "--grouped", "--strong", "--partition", partition]
    line2 = _bench(common + ["--dump-results", str(tmp_path / "r2.npy")], 2)
    line1 = _bench(common + ["--dump-results", str(tmp_path / "r1.npy")], 1)
    assert line2["scaling"] == "strong" and line2["config"]["pairs_total"] == n
    r2, r1 = np.load(tmp_path / "r2.npy"), np.load(tmp_path / "r1.npy")
    assert r2.shape == (3, n) and r1.shape == (3, n)
    assert np.array_equal(r2, r1)
    b = synth.generate(5, n, seed=5, grouped=True)
    rng = np.random.default_rng(55)
    idx = np.unique(np.concatenate([rng.choice(n, 2500, replace=False),
                                    np.argsort(b.qlen.astype(np.int64) * b.tlen)[-20:]]))
    sub = b.subset(idx)
    assert_same(tuple(r2[i][idx] for i in range(3)), oracle_align(sub, sb.BWA_MEM, oracle.LOCAL), sub,
                f"2-rank reassembled ({partition})")


def test_scatter_results_kernel(sb):
    """saloba_scatter_results alone: a random permutation split over 3 ranks with padding columns;
    an out-of-range index is reported through status and not written."""
    import torch

    rng = np.random.default_rng(3)
    n, world = 10_001, 3
    perm = rng.permutation(n).astype(np.int32)
    cuts = [0, 2_000, 7_500, n]
    stride = max(cuts[i + 1] - cuts[i] for i in range(world)) + 5
    index = np.full((world, stride), -1, np.int32)
    parts = np.full((world, 3, stride), -7, np.int32)
    truth = rng.integers(-5, 1000, (3, n)).astype(np.int32)
    for r in range(world):
        ix = perm[cuts[r]:cuts[r + 1]]
        index[r, :len(ix)] = ix
        parts[r, :, :len(ix)] = truth[:, ix]
    out, st = sb.scatter_results(torch.from_numpy(parts).cuda(), torch.from_numpy(index).cuda(), n)
    torch.cuda.synchronize()
    assert int(st.item()) == -1 and np.array_equal(out.cpu().numpy(), truth)
    index[1, 3] = n + 4  # inconsistent index: reported (flat slot 1*stride+3), column not written
    out, st = sb.scatter_results(torch.from_numpy(parts).cuda(), torch.from_numpy(index).cuda(), n)
    torch.cuda.synchronize()
    assert int(st.item()) == stride + 3
