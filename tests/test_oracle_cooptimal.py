"""Pins of the co-optimal oracle (oracle/cooptimal.py) to things other than itself:
brute-force enumeration of every alignment (oracle/brute.py, no DP), the
Delannoy closed form, the SPEC examples and the canonical traceback."""
from __future__ import annotations

import itertools
import random
from math import comb

import nwgen
import oracle
from oracle import brute, cooptimal

ORDERS = [(1, 2, 3), (1, 3, 2), (2, 1, 3), (2, 3, 1), (3, 1, 2), (3, 2, 1)]


def _dfs_key(tie):
    rank = {code: r for r, code in enumerate(tie)}
    return lambda ops: [rank[o] for o in reversed(ops)]


def test_count_and_order_vs_brute_force_exhaustive():
    """Every {A,C} pair up to length 3 x 3, all six orders: the count is the size of
    the brute-force optimal set and the enumeration is that set in depth-first order
    (reversed op strings compared under pi)."""
    strs = list(brute.all_strings("AC", 3))
    for tie in ORDERS:
        sc = nwgen.Scoring(tie=tie)
        for a, b in itertools.product(strs, strs):
            _, opt = brute.optimum(a, b, sc)
            assert cooptimal.count(a, b, sc) == len(opt)
            want = sorted(opt, key=_dfs_key(tie))
            got = cooptimal.enumerate_optimal(a, b, sc, 10 ** 6)
            assert [tuple(x) for x in got] == want, (a, b, tie)


def test_vs_brute_force_random():
    rng = random.Random(5)
    for _ in range(150):
        a = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, 6))).encode()
        b = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, 6))).encode()
        tie = rng.choice(ORDERS)
        sc = nwgen.Scoring(tie=tie)
        _, opt = brute.optimum(a, b, sc)
        assert cooptimal.count(a, b, sc) == len(opt)
        cap = rng.randint(1, 5)
        got = cooptimal.enumerate_optimal(a, b, sc, cap)
        assert [tuple(x) for x in got] == sorted(opt, key=_dfs_key(tie))[:cap]


def test_delannoy_closed_form():
    """No matches and mismatch = 2g: every alignment scores (m+n)g, so the count is
    the Delannoy number D(m, n) = sum_k C(m,k) C(n,k) 2^k."""
    sc = nwgen.Scoring(match=1, mismatch=-2, gap=-1)
    for m, n in [(0, 0), (1, 1), (3, 3), (7, 7), (12, 9), (25, 31)]:
        want = sum(comb(m, k) * comb(n, k) * 2 ** k for k in range(min(m, n) + 1))
        assert cooptimal.count(b"A" * m, b"C" * n, sc) == want
    assert cooptimal.count(b"AAA", b"CCC", sc) == 63  # D(3,3)


def test_spec_examples():
    """("A","A") -> exactly one; ("AG","GA") -> the brute-force set;
    cap = 1 -> the canonical traceback (P:90 tie order)."""
    sc = nwgen.PAPER_DNA
    assert cooptimal.enumerate_optimal(b"A", b"A", sc, 256) == [[1]]
    _, opt = brute.optimum(b"AG", b"GA", sc)
    got = cooptimal.enumerate_optimal(b"AG", b"GA", sc, 256)
    assert sorted(tuple(x) for x in got) == sorted(opt)
    rng = random.Random(9)
    for tie in ORDERS:
        sc = nwgen.Scoring(tie=tie)
        for _ in range(20):
            a = "".join(rng.choice("ACGT") for _ in range(rng.randint(1, 30))).encode()
            b = "".join(rng.choice("ACGT") for _ in range(rng.randint(1, 30))).encode()
            _, ops = oracle.align(a, b, sc)
            assert cooptimal.enumerate_optimal(a, b, sc, 1) == [ops.tolist()]


def test_worked_grid_three_optima():
    """GATTACA / GCATGCU has exactly 3 optimal alignments."""
    sc = nwgen.Scoring(alphabet="ACGTU")
    assert cooptimal.count(b"GATTACA", b"GCATGCU", sc) == 3
    rows = [oracle.render(b"GATTACA", b"GCATGCU", ops)
            for ops in cooptimal.enumerate_optimal(b"GATTACA", b"GCATGCU", sc, 10)]
    assert sorted(rows) == sorted([("G-ATTACA", "GCA-TGCU"), ("G-ATTACA", "GCAT-GCU"),
                                   ("G-ATTACA", "GCATG-CU")])


def test_mirror_counts():
    """Transposing the pair (U <-> L) keeps the count."""
    rng = random.Random(2)
    for _ in range(30):
        a = "".join(rng.choice("AC") for _ in range(rng.randint(0, 12))).encode()
        b = "".join(rng.choice("AC") for _ in range(rng.randint(0, 12))).encode()
        assert cooptimal.count(a, b, nwgen.PAPER_DNA) == cooptimal.count(b, a, nwgen.PAPER_DNA)
