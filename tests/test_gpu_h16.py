"""GPU parity of the packed H' single-pair sweep with a moving base (nw_fill_h16.cuh,
DESIGN.md §3.16) against the oracle: score-only pairs, bit-exact.

The sweep keeps H' - B in 16-bit halves and moves the per-strip base B every `reb`
8-step groups; the tests force it at every rows-per-lane setting, at the shortest
rebase period (1 group, the most rebases) and the default, with scorings whose
largest s - 2g puts the relative values close to 2^16, and check the fallback to the
difference form when no period fits. Reference: Eq. 1 (reading R1),
borders P:43-45.
"""
from __future__ import annotations

import pytest

import nwgen
import oracle
import paper_2412_21103_b200 as nwb

pytestmark = pytest.mark.gpu

KRS = [8, 12, 16, 18, 20, 22, 24, 26, 28, 30, 32]


@pytest.fixture(scope="module")
def ctx():
    c = nwb.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("reb", [1, 0])
@pytest.mark.parametrize("kr", KRS)
def test_h16_every_kr(ctx, opts, kr, reb):
    """Several strips with a ragged last one, a one-strip pair, very short rows and the
    1 x 1 grid, at every strip height, with the most frequent and the default rebase."""
    opts(ctx, "h16_kr", kr)
    opts(ctx, "h16_rebase", reb)
    for k, (m, n) in enumerate([(2500, 700), (32 * kr * 3 + 17, 333), (5, 900), (700, 5),
                                (1, 1), (64, 64)]):
        a, b = nwgen.random_pair(9300 + 41 * kr + k, m, n)
        for sc in (nwgen.PAPER_DNA, nwgen.Scoring(match=2, mismatch=-1, gap=-3)):
            assert nwb.nw_score_only(ctx, a, b, sc) == oracle.score(a, b, sc), (kr, reb, m, n)


@pytest.mark.parametrize("reb", [1, 4, 0])
def test_h16_tall_long_rebases(ctx, opts, reb):
    """A tall pair on the library's own tall-pair path (the default form) with long
    rows: the base moves thousands of times per strip."""
    opts(ctx, "h16_rebase", reb)
    a, b = nwgen.random_pair(9401, 90_000, 4_000)
    for sc in (nwgen.PAPER_DNA, nwgen.Scoring(match=3, mismatch=-2, gap=-2)):
        assert nwb.nw_score_only(ctx, a, b, sc) == oracle.score(a, b, sc), reb


@pytest.mark.parametrize("gap", [-1, -8, -15])
def test_h16_values_near_16_bits(ctx, opts, gap):
    """max(s - 2g) = 31 - 2 gap (match is capped at 31): at gap -15 (S = 61) only a
    2-group rebase period keeps S (32 KR + 8 reb + 160) <= 65535 at KR 28, so the
    relative values come within a few hundred of 2^16."""
    opts(ctx, "h16_kr", 28)
    sc = nwgen.Scoring(match=31, mismatch=2 * gap, gap=gap)
    for k, (m, n) in enumerate([(4000, 3000), (32 * 28 * 2 + 5, 2000)]):
        a, b = nwgen.random_pair(9500 - gap + k, m, n)
        assert nwb.nw_score_only(ctx, a, b, sc) == oracle.score(a, b, sc), (gap, m, n)
        a2 = b"A" * m  # all matches on the diagonal: the largest H' growth per column
        b2 = b"A" * n
        assert nwb.nw_score_only(ctx, a2, b2, sc) == oracle.score(a2, b2, sc), (gap, m, n)


def test_h16_falls_back_when_no_period_fits(ctx, opts):
    """S = 31 + 40 = 71 cannot keep a 28-row-per-lane strip in 16 bits: the library
    must fall back to the difference form, not overflow."""
    opts(ctx, "h16_kr", 28)
    sc = nwgen.Scoring(match=31, mismatch=-31, gap=-20)
    a, b = nwgen.random_pair(9601, 3000, 2500)
    assert nwb.nw_score_only(ctx, a, b, sc) == oracle.score(a, b, sc)
    a2 = b"A" * 3000
    assert nwb.nw_score_only(ctx, a2, a2, sc) == oracle.score(a2, a2, sc)


def test_h16_vs_difference_form_tall(ctx, opts):
    """The two packed tall-pair forms agree with each other and the oracle on a
    non-degenerate tall pair (~100 strips at the default rows per lane)."""
    a, b = nwgen.random_pair(9701, 100_000, 2_000)
    sc = nwgen.PAPER_DNA
    want = oracle.score(a, b, sc)
    assert nwb.nw_score_only(ctx, a, b, sc) == want
    opts(ctx, "pair_form", 1)
    assert nwb.nw_score_only(ctx, a, b, sc) == want


def test_h16_watchdog(ctx, opts):
    """A withheld boundary row makes the h16 sweep return NW_E_DEADLOCK, not hang."""
    opts(ctx, "h16_kr", 16)
    opts(ctx, "watchdog_polls", 20_000)
    opts(ctx, "test_withhold", 2)
    a, b = nwgen.random_pair(9801, 32 * 16 * 4, 900)
    with pytest.raises(nwb.NWError) as e:
        nwb.nw_score_only(ctx, a, b, nwgen.PAPER_DNA)
    assert e.value.status == nwb.NW_E_DEADLOCK


ORDERS = [(1, 2, 3), (1, 3, 2), (2, 1, 3), (2, 3, 1), (3, 1, 2), (3, 2, 1)]


@pytest.mark.parametrize("tie", ORDERS)
@pytest.mark.parametrize("kr", [0, 8])
def test_h16_direction_fill_traceback(ctx, opts, tie, kr):
    """pair_form 2: direction fills of DNA pairs in the packed H' form, flags re-phased
    into the int32 layout so the strip traceback reads them unchanged: score and op string
    vs the oracle for every tie order, several strips, ragged edges, a degenerate column."""
    opts(ctx, "pair_form", 2)
    opts(ctx, "rows_per_lane", kr)
    for k, (m, n) in enumerate([(1000, 1000), (700, 2300), (2600, 333), (129, 1), (5, 77)]):
        a, b = nwgen.random_pair(9900 + 7 * k + kr, m, n)
        for sc in (nwgen.Scoring(tie=tie), nwgen.Scoring(match=2, mismatch=-1, gap=-3, tie=tie)):
            want_score, want_ops = oracle.align(a, b, sc)
            got, tb = nwb.nw_align_pair(ctx, a, b, sc)
            ops = nwb.nw_traceback(ctx, tb)
            tb.free()
            assert got == want_score and ops.tolist() == want_ops.tolist(), (tie, kr, m, n)
