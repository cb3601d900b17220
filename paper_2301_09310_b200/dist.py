"""A5: sharding pairs across the GPUs of one box and gathering results to rank 0 (
PAPER.md §VII-C P:1738-1743 "split the queries ... assigning them to multiple GPUs", fixing
imbalance "with dynamic assignment or preprocessing with approximate sorting").

Pairs are independent, so no collective touches the DP: every rank aligns its own shard with the
C-ABI library and the only exchange is one gather of 12 bytes per pair to rank 0.  Host-side
logic only (index arithmetic + torch.distributed calls); the alignment itself runs in the library.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_range(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous equal-count split (the paper's "split equally"): [start, end)."""
    return n_total * rank // world, n_total * (rank + 1) // world


def pair_cost(qlen: np.ndarray, tlen: np.ndarray, kappa: float = 2048.0) -> np.ndarray:
    """Modelled cost of a pair, for REPORTING balance (the partition itself runs on the GPU with
    the same model: saloba_partition): cells + a per-pair overhead kappa."""
    return qlen.astype(np.float64) * tlen.astype(np.float64) + kappa


def balanced_partition(qlen, tlen, world: int) -> np.ndarray:
    """Length-balanced rank per pair, computed on the current GPU by saloba_partition (cost sort +
    snake deal, include/saloba.h).  Deterministic, so every rank can compute it from the global
    lengths without a collective.  qlen / tlen: numpy or torch int32.  Returns int32 numpy."""
    from . import partition

    dev = torch.device("cuda", torch.cuda.current_device())
    q = torch.as_tensor(np.asarray(qlen, np.int32)).to(dev)
    t = torch.as_tensor(np.asarray(tlen, np.int32)).to(dev)
    return partition(q, t, world).cpu().numpy()


def imbalance(cost: np.ndarray, owner: np.ndarray, world: int) -> float:
    """max/mean of per-rank total cost."""
    per = np.bincount(owner, weights=cost, minlength=world)
    return float(per.max() / per.mean()) if per.mean() > 0 else 1.0


def gather_results(local: torch.Tensor, counts: list[int], dst: int = 0):
    """Gather each rank's (3, n_r) int32 results to `dst`.  Works on NCCL (cuda tensors) and gloo
    (cpu tensors).  Returns the list of per-rank tensors on dst, None elsewhere."""
    world = dist.get_world_size()
    rank = dist.get_rank()
    nmax = max(counts)
    buf = local
    if local.shape[1] != nmax:  # gather needs equal shapes: pad
        buf = torch.full((3, nmax), -9, dtype=local.dtype, device=local.device)
        buf[:, :local.shape[1]] = local
    bufs = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, bufs, dst=dst)
    if rank != dst:
        return None
    return [b[:, :c] for b, c in zip(bufs, counts)]


def reassemble(parts: list[torch.Tensor], index_of_rank: list[np.ndarray], n_total: int) -> np.ndarray:
    """Place each rank's results back at the input positions it owned -> (3, n_total) int32."""
    out = np.full((3, n_total), -9, np.int32)
    for part, idx in zip(parts, index_of_rank):
        out[:, idx] = part.cpu().numpy()
    return out
