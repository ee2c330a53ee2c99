"""The dist context on one GPU.

- world = 1 through a real NCCL communicator (nw_dist_unique_id + nw_ctx_set_dist):
  the partition, the compact rank-space scores, the in-place broadcasts and the
  rank-space -> pair-order scatter all run; results equal the plain context's and
  the oracle's.
- Partition invariance for G in {1, 2, 3, 8}: the same code path with the test option
  dist_virtual_world/rank, G sequential calls (one per rank) into the same output
  buffers; the merged result must equal the single call and the oracle.
"""
import numpy as np
import pytest

import nwgen
import oracle
import paper_2412_21103_b200 as nwb

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = nwb.Context(0)
    yield c
    c.close()


def _dev_inputs(torch, ss, pairs):
    d_seqs = torch.from_numpy(ss.residues).cuda()
    d_offs = torch.from_numpy(ss.offs).cuda()
    d_pairs = None if pairs is None else torch.from_numpy(np.ascontiguousarray(pairs)).cuda()
    return d_seqs, d_offs, d_pairs


def _run(ctx, torch, ss, pairs, sc, flags, bufs=None):
    npairs = ss.nseq * (ss.nseq - 1) // 2 if pairs is None else len(pairs)
    d_seqs, d_offs, d_pairs = _dev_inputs(torch, ss, pairs)
    oo = nwb.nw_batch_ops_offsets(ss.offs, pairs)
    if bufs is None:
        bufs = (torch.full((npairs,), -7, dtype=torch.int32, device="cuda"),
                torch.from_numpy(oo).cuda(),
                torch.zeros(int(oo[-1]) + 1, dtype=torch.uint8, device="cuda"),
                torch.zeros(max(npairs, 1), dtype=torch.int32, device="cuda"))
    d_sc, d_oo, d_ops, d_len = bufs
    tb = flags == nwb.NW_TRACEBACK
    nwb.nw_align_batch_dev(ctx, d_seqs, d_offs, ss.offs, d_pairs, pairs, npairs, sc, flags, d_sc,
                           d_oo if tb else None, d_ops if tb else None, d_len if tb else None)
    ctx.sync()
    return bufs, oo


def _results(bufs, oo, tb):
    scores = bufs[0].cpu().numpy()
    if not tb:
        return scores, None
    paths = nwb.batch_paths(bufs[2].cpu().numpy(), oo, bufs[3].cpu().numpy())
    return scores, [p.tolist() for p in paths]


CASES = [("implicit", 0), ("explicit", 0), ("explicit", 1), ("implicit", 1)]


def _case(kind, seed=5):
    ss = nwgen.random_set(300 + seed, 60, 0, 700)
    rng = np.random.Generator(np.random.PCG64(seed))
    pairs = None if kind == "implicit" else rng.integers(0, ss.nseq, size=(900, 2)).astype(np.int32)
    return ss, pairs


def _oracle(ss, pairs, sc, tb, sample=None):
    allp = nwgen.all_pairs(ss.nseq) if pairs is None else pairs
    want = oracle.batch_score(ss.residues, ss.offs, allp, sc)
    paths = None
    if tb:
        idx = range(len(allp)) if sample is None else [k for k in sample if k < len(allp)]
        paths = {k: oracle.align(ss.seq(allp[k][0]), ss.seq(allp[k][1]), sc)[1].tolist() for k in idx}
    return want, paths


@pytest.mark.parametrize("kind,tb", CASES)
def test_world1_nccl_communicator(kind, tb):
    import torch
    sc = nwgen.PAPER_DNA
    ss, pairs = _case(kind)
    c = nwb.Context(0)
    c.set_dist(0, 1, nwb.nw_dist_unique_id())
    assert c.dist_info() == (0, 1)
    flags = nwb.NW_TRACEBACK if tb else nwb.NW_SCORE_ONLY
    bufs, oo = _run(c, torch, ss, pairs, sc, flags)
    scores, paths = _results(bufs, oo, tb)
    want, wpaths = _oracle(ss, pairs, sc, tb, sample=range(0, 1800, 7))
    assert scores.tolist() == want.tolist()
    if tb:
        for k, p in wpaths.items():
            assert paths[k] == p, k
    # the host entry point on the dist ctx
    r = nwb.nw_align_batch(c, ss.residues, ss.offs, pairs, sc, flags)
    assert (r[0] if tb else r).tolist() == want.tolist()
    c.close()


@pytest.mark.parametrize("kind,tb", CASES)
@pytest.mark.parametrize("G", [1, 2, 3, 8])
def test_partition_invariance_virtual_ranks(ctx, opts, kind, tb, G):
    """G ranks replayed on one GPU: rank r of G aligns only its range; after all G
    calls the outputs equal the oracle's (reading R18)."""
    import torch
    sc = nwgen.Scoring(tie=(2, 3, 1)) if tb else nwgen.PAPER_DNA
    ss, pairs = _case(kind, seed=G)
    flags = nwb.NW_TRACEBACK if tb else nwb.NW_SCORE_ONLY
    opts(ctx, "dist_virtual_world", G)
    bufs = None
    for r in range(G):
        ctx.set_option("dist_virtual_rank", r)
        bufs, oo = _run(ctx, torch, ss, pairs, sc, flags, bufs)
    ctx.set_option("dist_virtual_rank", 0)
    scores, paths = _results(bufs, oo, tb)
    want, wpaths = _oracle(ss, pairs, sc, tb, sample=range(0, 1700, 11))
    assert scores.tolist() == want.tolist()
    if tb:
        for k, p in wpaths.items():
            assert paths[k] == p, k


def test_c3_partition_ranges_fullsize(ctx, opts):
    """C3 at full size in 8 virtual ranks (the SCALE run's partition): merged scores
    equal a single call's (whose digest test_gpu_fullsize checks against the oracle)."""
    import torch
    ss = nwgen.config_c3()
    sc = nwgen.PAPER_DNA
    single, _ = _run(ctx, torch, ss, None, sc, nwb.NW_SCORE_ONLY)
    opts(ctx, "dist_virtual_world", 8)
    bufs = None
    for r in range(8):
        ctx.set_option("dist_virtual_rank", r)
        bufs, _ = _run(ctx, torch, ss, None, sc, nwb.NW_SCORE_ONLY, bufs)
    ctx.set_option("dist_virtual_rank", 0)
    assert torch.equal(bufs[0], single[0])


@pytest.mark.parametrize("G", [2, 3])
def test_partition_invariance_host_entry(ctx, opts, G):
    """The host entry point (nw_align_batch) on the same replayed G-rank partition,
    explicit pairs with traceback, into caller-owned output buffers."""
    sc = nwgen.PAPER_DNA
    ss, pairs = _case("explicit", seed=10 + G)
    oo = nwb.nw_batch_ops_offsets(ss.offs, pairs)
    out = (np.full(len(pairs), -7, np.int32), np.zeros(int(oo[-1]) + 1, np.uint8),
           np.zeros(len(pairs) + 1, np.int64), np.zeros(len(pairs), np.int32))
    opts(ctx, "dist_virtual_world", G)
    for r in range(G):
        ctx.set_option("dist_virtual_rank", r)
        scores, ops, ops_off, ops_len = nwb.nw_align_batch(ctx, ss.residues, ss.offs, pairs, sc,
                                                           nwb.NW_TRACEBACK, out=out)
    ctx.set_option("dist_virtual_rank", 0)
    want = oracle.batch_score(ss.residues, ss.offs, pairs, sc)
    assert scores.tolist() == want.tolist()
    paths = nwb.batch_paths(ops, ops_off, ops_len)
    for k in range(0, len(pairs), 13):
        assert paths[k].tolist() == oracle.align(ss.seq(pairs[k][0]), ss.seq(pairs[k][1]), sc)[1].tolist()


def test_set_dist_validates(ctx):
    uid = nwb.nw_dist_unique_id()
    for rank, world in [(-1, 1), (1, 1), (0, 0)]:
        with pytest.raises(nwb.NWError) as e:
            ctx.set_dist(rank, world, uid)
        assert e.value.status == nwb.NW_E_INVAL
    assert ctx.dist_info() == (0, 1)
