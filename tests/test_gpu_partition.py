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
