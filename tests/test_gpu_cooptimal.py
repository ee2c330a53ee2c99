"""GPU parity of the co-optimal count and enumeration (nw_cooptimal, SURVEY.md
§8(f) NEXT #2) against oracle/cooptimal.py: counts equal (saturating at 2^64-1)
and the enumerated paths identical, in order."""
from __future__ import annotations

import itertools
from math import comb

import pytest

import nwgen
from oracle import brute, cooptimal
import paper_2412_21103_b200 as nwb

pytestmark = pytest.mark.gpu

ORDERS = [(1, 2, 3), (1, 3, 2), (2, 1, 3), (2, 3, 1), (3, 1, 2), (3, 2, 1)]
U64 = (1 << 64) - 1


@pytest.fixture(scope="module")
def ctx():
    c = nwb.Context(0)
    yield c
    c.close()


def _check(ctx, a, b, sc, cap):
    want_n = cooptimal.count(a, b, sc)
    got_n, sat, paths = nwb.nw_cooptimal(ctx, a, b, sc, cap)
    assert got_n == min(want_n, U64) and sat == (want_n >= U64), (len(a), len(b))
    if cap:
        want = cooptimal.enumerate_optimal(a, b, sc, cap)
        assert [p.tolist() for p in paths] == want, (len(a), len(b), sc.tie)


def test_exhaustive_small_all_orders(ctx):
    strs = list(brute.all_strings("AC", 3))
    for tie in ORDERS:
        sc = nwgen.Scoring(tie=tie)
        for a, b in itertools.product(strs, strs):
            _check(ctx, a, b, sc, 1000)


@pytest.mark.parametrize("m,n", [(1, 40), (33, 31), (64, 65), (100, 37), (150, 150)])
def test_random_dna(ctx, m, n):
    a, b = nwgen.random_pair(m * 3 + n, m, n)
    for tie in ORDERS[:3]:
        _check(ctx, a, b, nwgen.Scoring(tie=tie), 50)


def test_protein_and_low_complexity(ctx):
    a, b = nwgen.random_pair(4, 90, 80, nwgen.PROTEIN)
    _check(ctx, a, b, nwgen.PROTEIN_BLOSUM62, 40)
    _check(ctx, b"ACAC" * 20, b"CACA" * 21, nwgen.PAPER_DNA, 256)


def test_delannoy_and_saturation(ctx):
    """No matches, mismatch = 2g: count = D(m, n); D(40, 40) > 2^64 saturates."""
    sc = nwgen.Scoring(match=1, mismatch=-2, gap=-1)
    for m, n in [(5, 7), (25, 25), (30, 24)]:
        want = sum(comb(m, k) * comb(n, k) * 2 ** k for k in range(min(m, n) + 1))
        got, sat, _ = nwb.nw_cooptimal(ctx, b"A" * m, b"C" * n, sc)
        assert (got, sat) == (min(want, U64), want >= U64)
    got, sat, paths = nwb.nw_cooptimal(ctx, b"A" * 40, b"C" * 40, sc, 3)
    assert sat and got == U64 and len(paths) == 3


def test_c1_cap_256(ctx):
    """configs[0]: count vs the oracle and the first 256 paths; path 0 = canonical."""
    a, b = nwgen.config_c1()
    _check(ctx, a, b, nwgen.PAPER_DNA, 256)
    _, tb = nwb.nw_align_pair(ctx, a, b, nwgen.PAPER_DNA)
    canon = nwb.nw_traceback(ctx, tb)
    tb.free()
    _, _, paths = nwb.nw_cooptimal(ctx, a, b, nwgen.PAPER_DNA, 1)
    assert paths[0].tolist() == canon.tolist()
