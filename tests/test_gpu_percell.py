"""GPU parity of the paper's per-cell kernel (ablation baseline, SURVEY.md §8(f)
NEXT #4): score and op string identical to the oracle."""
from __future__ import annotations

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


def _check(ctx, a, b, sc):
    ws, wops = oracle.align(a, b, sc)
    gs, gops = nwb.nw_align_pair_percell(ctx, a, b, sc)
    assert gs == ws and gops.tolist() == wops.tolist(), (len(a), len(b), sc.tie)


@pytest.mark.parametrize("m,n", [(1, 1), (1, 7), (7, 1), (31, 33), (100, 257), (513, 300),
                                 (1000, 1000)])
def test_sizes(ctx, m, n):
    a, b = nwgen.random_pair(m * 131 + n, m, n)
    _check(ctx, a, b, nwgen.PAPER_DNA)


@pytest.mark.parametrize("tie", ORDERS)
def test_tie_orders_and_protein(ctx, tie):
    a, b = nwgen.random_pair(5, 200, 180, nwgen.PROTEIN)
    sc = nwgen.Scoring(match=0, mismatch=0, gap=-5, alphabet=nwgen.PROTEIN, subst=nwgen.BLOSUM62,
                       tie=tie)
    _check(ctx, a, b, sc)
    a, b = b"ACACACGT" * 20, b"ACGTACAC" * 21  # low complexity: many ties
    _check(ctx, a, b, nwgen.Scoring(tie=tie))


def test_empty_and_worked_grid(ctx):
    for a, b in [(b"", b""), (b"ACG", b""), (b"", b"TT"), (b"GATTACA", b"GCATGCT")]:
        _check(ctx, a, b, nwgen.PAPER_DNA)


def test_c1_config(ctx):
    a, b = nwgen.config_c1()
    _check(ctx, a, b, nwgen.PAPER_DNA)
