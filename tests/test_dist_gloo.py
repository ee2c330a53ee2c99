"""Multi-process (world_size 2, gloo, CPU) checks of the batch sharding and the
score gather (SURVEY.md §4 T4 host logic; S:362 result invariance across
partitions). The per-shard scores come from the oracle here because this box
has no GPU; on the GPU path they come from nw_align_batch_dev."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import nwgen
import oracle
from paper_2412_21103_b200 import dist as nwdist


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ss = nwgen.random_set(77, 24, 0, 300)
    pairs = nwgen.all_pairs(ss.nseq)
    cost = nwdist.pair_costs(ss.lengths(), pairs)
    shard = nwdist.partition_pairs(cost, world)[rank]
    local = oracle.batch_score(ss.residues, ss.offs, pairs[shard], nwgen.PAPER_DNA, nthreads=1)
    full = nwdist.gather_scores(torch.as_tensor(local.astype(np.int32)), shard, len(pairs), world)
    if rank == 0:
        np.save(out_path, full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_partition_covers_and_balances():
    rng = np.random.Generator(np.random.PCG64(4))
    cost = rng.integers(1, 4_000_000, size=10_001)
    for world in (1, 2, 3, 8):
        parts = nwdist.partition_pairs(cost, world)
        allidx = np.concatenate(parts)
        assert len(allidx) == len(cost) and len(np.unique(allidx)) == len(cost)
        loads = [cost[p].sum() for p in parts]
        assert max(loads) - min(loads) <= cost.max()
        assert max(len(p) for p in parts) <= nwdist.shard_capacity(len(cost), world)


def test_gather_two_ranks_matches_single(tmp_path):
    world, port = 2, _free_port()
    out = str(tmp_path / "full.npy")
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    got = np.load(out)
    ss = nwgen.random_set(77, 24, 0, 300)
    want = oracle.batch_score(ss.residues, ss.offs, nwgen.all_pairs(ss.nseq), nwgen.PAPER_DNA)
    assert got.tolist() == want.tolist()
