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
