"""Multi-GPU plumbing for the batch path.

P:131: "the total number of alignments is divided by the number of ranks ...
the data is then sent to each rank ... gathered back in the main process".
Here every rank holds all sequences (they are small), takes a cost-balanced
share of the pairs, runs nw_align_batch_dev on its share, and one NCCL
all-gather returns every rank's int32 scores (reading R18:
the result is independent of the partition).

Host logic only: the scores themselves come from the CUDA library.
"""
from __future__ import annotations

import numpy as np


def pair_costs(lengths: np.ndarray, pairs: np.ndarray) -> np.ndarray:
    """m * n cells of each (p, q) pair."""
    lengths = np.asarray(lengths, dtype=np.int64)
    return lengths[pairs[:, 0]] * lengths[pairs[:, 1]]


def partition_pairs(cost: np.ndarray, world: int) -> list[np.ndarray]:
    """Cost-balanced partition of pair indices over `world` ranks.

    Pairs sorted by cost (descending) are dealt in boustrophedon order
    (0..G-1, G-1..0, ...), which keeps every rank within one pair's cost of the
    others; each rank's indices are returned sorted (pair order)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = np.argsort(-np.asarray(cost), kind="stable")
    npairs = len(order)
    pos = np.arange(npairs)
    rnd, k = pos // world, pos % world
    rank_of = np.where(rnd % 2 == 0, k, world - 1 - k)
    return [np.sort(order[rank_of == r]) for r in range(world)]


def shard_capacity(npairs: int, world: int) -> int:
    """Largest shard size of partition_pairs (all-gather buffers are padded to it)."""
    return -(-npairs // world)


def gather_scores(local_scores, local_idx: np.ndarray, npairs: int, world: int, group=None):
    """All-gather every rank's shard scores and indices (torch tensors on the
    process group's device) and return the full int32 score vector in pair order."""
    import torch
    import torch.distributed as dist
    cap = shard_capacity(npairs, world)
    dev = local_scores.device
    sc = torch.zeros(cap, dtype=torch.int32, device=dev)
    ix = torch.full((cap,), -1, dtype=torch.int64, device=dev)
    n = len(local_idx)
    sc[:n] = local_scores[:n]
    ix[:n] = torch.as_tensor(local_idx, dtype=torch.int64, device=dev)
    all_sc = [torch.empty_like(sc) for _ in range(world)]
    all_ix = [torch.empty_like(ix) for _ in range(world)]
    dist.all_gather(all_sc, sc, group=group)
    dist.all_gather(all_ix, ix, group=group)
    full = torch.empty(npairs, dtype=torch.int32, device=dev)
    for s_, i_ in zip(all_sc, all_ix):
        keep = i_ >= 0
        full[i_[keep]] = s_[keep]
    return full


def cblock_score(ctx, d_a, d_b, sc, group=None, block_cols: int = 0) -> int:
    """Score of one giant pair with the column-block pipeline across the ranks of
    `group` (one process per GPU). Receive buffers are
    symmetric memory, so each rank writes its right boundary columns straight
    into the next rank's buffer over NVLink; one all-reduce returns H(m, n).
    Not exercised on more than one GPU in this round (tests cover the same
    kernel with ranks on concurrent streams of one GPU)."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm
    from . import nw as _nw
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    nbytes = _nw.nw_cblock_recv_bytes(d_a.numel())
    buf = symm.empty(nbytes, dtype=torch.uint8, device=d_a.device)
    hdl = symm.rendezvous(buf, group if group is not None else dist.group.WORLD)
    nxt = hdl.get_buffer((rank + 1) % world, [nbytes], torch.uint8)
    buf.zero_()
    torch.cuda.synchronize()
    dist.barrier(group)  # every receive buffer is zero before anyone writes
    part = torch.zeros(1, dtype=torch.int64, device=d_a.device)
    _nw.nw_score_only_cblock_rank_dev(ctx, d_a, d_b, sc, rank, world, block_cols, buf, nxt, part)
    dist.all_reduce(part, group=group)
    return int(part.item())
