"""GPU parity of the checkpointed traceback (nw_align_pair_linear, SURVEY.md §8(f)
NEXT #3): with budgets that force many segments, score and op
string identical to the oracle (and so to the one-shot traceback)."""
from __future__ import annotations

import numpy as np
import pytest

import nwgen
import oracle
import paper_2412_21103_b200 as nwb

pytestmark = pytest.mark.gpu

ORDERS = [(1, 2, 3), (1, 3, 2), (2, 1, 3), (2, 3, 1), (3, 1, 2), (3, 2, 1)]


@pytest.fixture(scope="module")
def ctx():
    c = nwb.Context(0)
    yield c
    c.close()


def _check(ctx, a, b, sc, budget):
    ws, wops = oracle.align(a, b, sc)
    gs, gops = nwb.nw_align_pair_linear(ctx, a, b, sc, budget)
    assert gs == ws, (len(a), len(b), budget)
    assert gops.tolist() == wops.tolist(), (len(a), len(b), budget, sc.tie)


@pytest.mark.parametrize("m,n,budget", [(3000, 2500, 20_000), (3000, 2500, 70_000),
                                        (1000, 4000, 5_000), (5000, 300, 2_000),
                                        (2048, 2048, 1), (777, 1300, 0)])
def test_segment_splits(ctx, m, n, budget):
    """budget 1: one strip of the checkpoint pass per segment; 0: default (one shot)."""
    a, b = nwgen.random_pair(m + 7 * n, m, n)
    _check(ctx, a, b, nwgen.PAPER_DNA, budget)


@pytest.mark.parametrize("tie", ORDERS)
def test_tie_orders_protein_and_ties(ctx, tie):
    a, b = nwgen.random_pair(3, 1500, 1400, nwgen.PROTEIN)
    sc = nwgen.Scoring(match=0, mismatch=0, gap=-5, alphabet=nwgen.PROTEIN, subst=nwgen.BLOSUM62,
                       tie=tie)
    _check(ctx, a, b, sc, 30_000)
    a, b = b"ACGTTGCA" * 300, b"ACGTTGCAA" * 250  # periodic: many co-optimal paths
    _check(ctx, a, b, nwgen.Scoring(tie=tie), 25_000)


def test_paths_hitting_the_borders(ctx):
    """Paths that reach column 0 or row 0 early (long leading gaps)."""
    a = b"A" * 4000 + b"CGT"
    b = b"CGT"
    _check(ctx, a, b, nwgen.PAPER_DNA, 500)
    _check(ctx, b, a, nwgen.PAPER_DNA, 500)
    a2, b2 = nwgen.random_pair(9, 2000, 60)
    _check(ctx, a2, b2, nwgen.PAPER_DNA, 200)


def test_c2_with_small_budget(ctx):
    """configs[1] (20k x 20k) in ~8 segments vs the oracle."""
    a, b = nwgen.config_c2()
    _check(ctx, a, b, nwgen.PAPER_DNA, 13_000_000)


def test_c5_scale_closed_forms(ctx):
    """1M x 1M with a 24 GB direction budget (several segments): a = b gives
    1,000,000 diagonal moves, and the random C5 pair's path consumes both
    sequences and its column sum equals the score-only H(m, n)."""
    a, b = nwgen.config_c5()
    s, ops = nwb.nw_align_pair_linear(ctx, a, a, nwgen.PAPER_DNA, 24 << 30)
    assert s == len(a) and len(ops) == len(a) and int(ops.max()) == 1
    s2 = nwb.nw_score_only(ctx, a, b, nwgen.PAPER_DNA)
    s, ops = nwb.nw_align_pair_linear(ctx, a, b, nwgen.PAPER_DNA, 24 << 30)
    assert s == s2
    ops = ops.astype(np.int64)
    assert (ops != 3).sum() == len(a) and (ops != 2).sum() == len(b)
    av = np.frombuffer(a, dtype=np.uint8)
    bv = np.frombuffer(b, dtype=np.uint8)
    i = np.cumsum(ops != 3) - 1
    j = np.cumsum(ops != 2) - 1
    d = ops == 1
    match = av[i[d]] == bv[j[d]]
    col = int(match.sum()) - int((~match).sum()) - int((ops != 1).sum())
    assert col == s


@pytest.mark.parametrize("m,n,budget", [(80_000, 400, 1), (80_000, 400, 2_000_000),
                                        (100_000, 1_500, 9_000_000)])
@pytest.mark.parametrize("int32", [False, True])
def test_tall_packed_checkpoint_pass(ctx, opts, m, n, budget, int32):
    """Tall pairs (>= 76,800 rows): the checkpoint pass runs the packed difference
    form, whose checkpoint rows carry V and are prefix-summed into H' for the
    refills (k_ckpt_prefix); NW_LINEAR_INT32 forces the int32 pass. Both must give
    the oracle's score and canonical path, many segments down to one strip each."""
    if int32:
        opts(ctx, "linear_int32", 1)
    a, b = nwgen.random_pair(m + n, m, n)
    for tie in [(1, 2, 3), (3, 2, 1)]:
        _check(ctx, a, b, nwgen.Scoring(tie=tie), budget)
