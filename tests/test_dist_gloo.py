"""Multi-process (gloo, CPU) checks of the dist context's host logic (
S:362 result invariance across partitions):
  - nw_batch_partition against its definition (brute force), explicit and implicit;
  - the NCCL id shared from rank 0 over a gloo group (the library's own id);
  - the gather protocol of nw_align_batch on a dist ctx, replayed with gloo: every
    rank aligns its range (here with the oracle: no GPU on this box) and in-place
    broadcasts of every rank's range rebuild the full result, equal to one call;
  - bench.py's own launcher (dist.launch) forks N ranks that see each other.
"""
from __future__ import annotations

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist

import nwgen
import oracle
from paper_2412_21103_b200 import dist as nwdist


def _bounds_by_definition(costs, world):
    """bounds[r] = first task whose cost prefix * world >= r * total."""
    total = int(np.sum(costs))
    pref = np.concatenate([[0], np.cumsum(costs, dtype=np.int64)])
    out = [0]
    for r in range(1, world):
        k = int(np.argmax(pref * world >= r * total)) if total else 0
        out.append(min(k, len(costs)))
    out.append(len(costs))
    return np.maximum.accumulate(np.array(out, dtype=np.int64))


def _rank_space(ss):
    """k_batch's implicit task order: p' < q' over the stable length-descending order."""
    lens = ss.lengths()
    perm = sorted(range(ss.nseq), key=lambda k: -lens[k])  # Python sort is stable
    tasks = [(perm[p], perm[q]) for p in range(ss.nseq) for q in range(p + 1, ss.nseq)]
    return perm, tasks


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partition_matches_definition(world):
    ss = nwgen.random_set(70 + world, 40, 0, 900)
    rng = np.random.Generator(np.random.PCG64(world))
    pairs = rng.integers(0, ss.nseq, size=(3001, 2)).astype(np.int32)
    lens = ss.lengths()
    costs = lens[pairs[:, 0]] * lens[pairs[:, 1]]
    b = nwdist.partition(ss.offs, pairs, world)
    assert b.tolist() == _bounds_by_definition(costs, world).tolist()
    loads = [costs[b[r]:b[r + 1]].sum() for r in range(world)]
    assert max(loads) - min(loads) <= 2 * costs.max()
    _, tasks = _rank_space(ss)
    tcost = np.array([lens[p] * lens[q] for p, q in tasks], dtype=np.int64)
    bi = nwdist.partition(ss.offs, None, world)
    assert bi.tolist() == _bounds_by_definition(tcost, world).tolist()


def test_partition_degenerate():
    offs = np.array([0, 0, 0, 5], dtype=np.int64)  # empty sequences: zero-cost tasks
    assert nwdist.partition(offs, None, 4).tolist()[-1] == 3
    assert nwdist.partition(np.array([0], dtype=np.int64), None, 3).tolist() == [0, 0, 0, 0]


def _gather_worker(implicit: bool, out_path: str):
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    uid = nwdist.share_unique_id()
    ids = [None] * world
    dist.all_gather_object(ids, uid)
    assert all(x == ids[0] for x in ids) and len(uid) == 128
    ss = nwgen.random_set(77, 24, 0, 300)
    sc = nwgen.PAPER_DNA
    if implicit:
        perm, tasks = _rank_space(ss)
        b = nwdist.partition(ss.offs, None, world)
        rs = torch.zeros(len(tasks), dtype=torch.int32)
        mine = np.array(tasks[b[rank]:b[rank + 1]], dtype=np.int32).reshape(-1, 2)
        if len(mine):
            rs[b[rank]:b[rank + 1]] = torch.from_numpy(
                oracle.batch_score(ss.residues, ss.offs, mine, sc, nthreads=1).astype(np.int32))
        for g in range(world):  # the library's grouped in-place broadcasts
            if b[g + 1] > b[g]:
                view = rs[b[g]:b[g + 1]].clone()
                dist.broadcast(view, src=g)
                rs[b[g]:b[g + 1]] = view
        full = np.zeros(len(tasks), dtype=np.int32)  # k_rs_scatter: rank space -> pair order
        n = ss.nseq
        for t, (x, y) in enumerate(tasks):
            p, q = min(x, y), max(x, y)
            full[p * n - p * (p + 1) // 2 + (q - p - 1)] = rs[t]
    else:
        pairs = nwgen.all_pairs(ss.nseq)[::-1].copy()
        b = nwdist.partition(ss.offs, pairs, world)
        sc_t = torch.zeros(len(pairs), dtype=torch.int32)
        lo, hi = b[rank], b[rank + 1]
        if hi > lo:
            sc_t[lo:hi] = torch.from_numpy(
                oracle.batch_score(ss.residues, ss.offs, pairs[lo:hi], sc, nthreads=1).astype(np.int32))
        for g in range(world):
            if b[g + 1] > b[g]:
                view = sc_t[b[g]:b[g + 1]].clone()
                dist.broadcast(view, src=g)
                sc_t[b[g]:b[g + 1]] = view
        full = sc_t.numpy()
    if rank == 0:
        np.save(out_path, full)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("implicit", [True, False])
def test_gather_protocol_two_ranks(tmp_path, implicit):
    out = str(tmp_path / "full.npy")
    nwdist.launch(2, _gather_worker, (implicit, out))
    got = np.load(out)
    ss = nwgen.random_set(77, 24, 0, 300)
    pairs = nwgen.all_pairs(ss.nseq)
    if not implicit:
        pairs = pairs[::-1].copy()
    want = oracle.batch_score(ss.residues, ss.offs, pairs, nwgen.PAPER_DNA)
    assert got.tolist() == want.tolist()


def _hello(out_dir: str):
    dist.init_process_group("gloo")
    r, w = dist.get_rank(), dist.get_world_size()
    t = torch.tensor([r + 1])
    dist.all_reduce(t)
    with open(os.path.join(out_dir, f"rank{r}"), "w") as f:
        f.write(f"{r} {w} {int(t)} {os.environ['LOCAL_RANK']}")
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [2, 3])
def test_launcher_forks_ranks(tmp_path, n):
    nwdist.launch(n, _hello, (str(tmp_path),))
    got = sorted(open(os.path.join(tmp_path, f"rank{r}")).read() for r in range(n))
    assert got == sorted(f"{r} {n} {n * (n + 1) // 2} {r}" for r in range(n))
