"""A5 host logic at world size 2 over gloo (CPU): partition, per-rank compute, gather to rank 0,
reassembly in input order.  The per-rank compute here is the CPU oracle standing in for the GPU
(the test covers the sharding/gather logic, not the kernels)."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_2301_09310_b200 import dist as sd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def snake_reference(qlen, tlen, world):
    """Test reference of saloba_partition's assignment (include/saloba.h): stable sort by
    descending q*t + 2048, dealt 0..W-1, W-1..0, ...  (numpy; the product computes it on the GPU)."""
    cost = qlen.astype(np.int64) * tlen.astype(np.int64) + 2048
    order = np.argsort(-cost, kind="stable")
    k = np.arange(len(cost))
    rnd, pos = k // world, k % world
    owner = np.empty(len(cost), np.int32)
    owner[order] = np.where(rnd % 2 == 0, pos, world - 1 - pos)
    return owner


def test_partition_balance_and_coverage():
    import synth

    ql, tl, _ = synth.shapes(5, 200_000, grouped=True)  # worst case for an equal split
    cost = sd.pair_cost(ql, tl)
    for world in (2, 4, 8):
        owner = snake_reference(ql, tl, world)
        assert owner.min() == 0 and owner.max() == world - 1
        assert sd.imbalance(cost, owner, world) < 1.02
        eq = np.repeat(np.arange(world), [sd.shard_range(len(cost), world, r)[1] - sd.shard_range(len(cost), world, r)[0] for r in range(world)])
        assert sd.imbalance(cost, eq, world) > 1.3  # the equal split of a grouped batch is badly skewed


def test_shard_range_covers():
    for n in (0, 1, 7, 1000):
        for w in (1, 2, 3, 8):
            rs = [sd.shard_range(n, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import oracle
    import synth
    from paper_2301_09310_b200 import dist as sd

    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = synth.generate(3, 600, seed=5)
    owner = snake_reference(b.qlen, b.tlen, world)
    idx = [np.nonzero(owner == r)[0] for r in range(world)]
    mine = b.subset(idx[rank])
    s, qe, te, st, _ = oracle.align_batch(mine, threads=2)
    local = torch.from_numpy(np.stack([s, qe, te]).astype(np.int32))
    parts = sd.gather_results(local, [len(i) for i in idx])
    if rank == 0:
        full = sd.reassemble(parts, idx, b.n)
        ref = oracle.align_batch(b, threads=2)
        q.put(bool(np.array_equal(full, np.stack(ref[:3]))))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_to_rank0_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert ok
