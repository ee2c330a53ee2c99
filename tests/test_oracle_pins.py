"""Pins of the CPU oracle to things other than itself.

Each test checks oracle/ against a value the paper (or a cited worked example)
prints, brute-force enumeration of every alignment (oracle/brute.py, no DP), a
closed form, an independent textbook routine (tests/pins.py), or an invariant
-- chosen so that a dropped term, wrong sign, wrong index or transposed operand
in the oracle fails at least one of them.
"""
from __future__ import annotations

import itertools
import os
import random

import numpy as np
import pytest

import nwgen
import oracle
from oracle import brute
from pins import myers_edit_distance

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
ORDERS = {"DUL": (1, 2, 3), "DLU": (1, 3, 2), "UDL": (2, 1, 3), "ULD": (2, 3, 1),
          "LDU": (3, 1, 2), "LUD": (3, 2, 1)}


def _sc(**kw):
    return nwgen.Scoring(**kw)


# ---------------------------------------------------------------- paper values

def test_border_p45():
    """P:43-45 (Sec. 2.2): H(0,0)=0, first row/column decrease by |g| per cell."""
    for line in open(os.path.join(GOLDEN, "border_p45.txt")):
        if line.startswith("#") or not line.strip():
            continue
        head, row0, col0 = line.split("|")
        m, n, g = map(int, head.split())
        H, T, _ = oracle.fill(b"A" * m, b"A" * n, _sc(gap=g))
        assert H[0, :].tolist() == [int(x) for x in row0.split()]
        assert H[:, 0].tolist() == [int(x) for x in col0.split()]
        # border codes (R7): row 0 horizontal, column 0 vertical, origin unset
        assert T[0, 0] == 0
        assert (T[0, 1:] == oracle.L).all() and (T[1:, 0] == oracle.U).all()


def _read_grid():
    d = {"H": [], "T": [], "canon": {}}
    for line in open(os.path.join(GOLDEN, "gattaca_gcatgcu.txt")):
        if line.startswith("#") or not line.strip():
            continue
        k, *rest = line.split()
        if k in ("H", "T"):
            d[k].append([int(x) for x in rest])
        elif k == "canon":
            d["canon"][rest[0]] = tuple(rest[1].split("/"))
        elif k == "optimal":
            d["optimal"] = {tuple(x.split("/")) for x in rest}
        else:
            d[k] = rest[0]
    return d


def test_worked_grid_matches_fixture():
    g = _read_grid()
    sc = _sc(alphabet=g["alphabet"])
    H, T, score = oracle.fill(g["a"].encode(), g["b"].encode(), sc)
    assert H.tolist() == g["H"]
    assert T.tolist() == g["T"]
    assert score == int(g["score"]) == 0  # S:90 / S:134


def test_worked_grid_every_cell_by_brute_force():
    """Every H(i,j) of the GATTACA/GCATGCU grid = max over all alignments of the
    prefixes (no DP); every T(i,j) = last op of the canonical optimal prefix
    alignment -- for all six tie orders."""
    g = _read_grid()
    a, b = g["a"].encode(), g["b"].encode()
    for name, tie in ORDERS.items():
        sc = _sc(alphabet=g["alphabet"], tie=tie)
        H, T, _ = oracle.fill(a, b, sc)
        for i in range(len(a) + 1):
            for j in range(len(b) + 1):
                if i == 0 and j == 0:
                    continue
                best, opt = brute.optimum(a[:i], b[:j], sc)
                assert H[i, j] == best, (name, i, j)
                assert T[i, j] == brute.canonical(opt, tie)[-1], (name, i, j)


def test_worked_grid_canonical_alignments_all_orders():
    g = _read_grid()
    a, b = g["a"].encode(), g["b"].encode()
    for name, want in g["canon"].items():
        sc = _sc(alphabet=g["alphabet"], tie=ORDERS[name])
        score, ops = oracle.align(a, b, sc)
        assert oracle.render(a, b, ops) == want
    _, opt = brute.optimum(a, b, _sc(alphabet=g["alphabet"]))
    assert {oracle.render(a, b, o) for o in opt} == g["optimal"]


def test_small_examples():
    for line in open(os.path.join(GOLDEN, "small_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        src, a, b, kind, score, aln = [x.strip() for x in line.split("|")]
        sc = nwgen.PROTEIN_BLOSUM62 if kind == "blosum62g5" else nwgen.PAPER_DNA
        s, ops = oracle.align(a.encode(), b.encode(), sc)
        assert s == int(score), src
        assert oracle.score(a.encode(), b.encode(), sc) == int(score), src
        if aln != "-":
            assert "/".join(oracle.render(a.encode(), b.encode(), ops)) == aln, src


def test_blosum62_table_sanity():
    B = nwgen.BLOSUM62
    assert (B == B.T).all()
    assert B.min() == -4 and B.max() == 11
    idx = {c: k for k, c in enumerate(nwgen.PROTEIN)}
    assert B[idx["W"], idx["W"]] == 11 and B[idx["C"], idx["C"]] == 9
    assert (np.diag(B) > 0).all()


# ---------------------------------------------------------------- brute force

def test_exhaustive_brute_force_AC_up_to_4():
    """SPEC S:496 (scaled): every pair over {A,C} with lengths <= 4, all 6 orders:
    score = brute-force optimum, traceback = canonical optimal alignment."""
    strings = list(brute.all_strings("AC", 4))
    for a, b in itertools.product(strings, strings):
        opt_cache = None
        for tie in ORDERS.values():
            sc = _sc(tie=tie)
            score, ops = oracle.align(a, b, sc)
            if opt_cache is None:
                opt_cache = brute.optimum(a, b, sc)
            best, opt = opt_cache
            assert score == best
            assert tuple(int(x) for x in ops) == brute.canonical(opt, tie), (a, b, tie)


def test_random_brute_force_dna_and_scores():
    rng = random.Random(1)
    for _ in range(150):
        a = bytes(rng.choice(b"ACGT") for _ in range(rng.randint(0, 6)))
        b = bytes(rng.choice(b"ACGT") for _ in range(rng.randint(0, 6)))
        mm = rng.choice([-1, -2, -3, 0])
        g = rng.choice([-1, -2, -3])
        tie = rng.choice(list(ORDERS.values()))
        sc = _sc(match=rng.choice([1, 2, 3]), mismatch=mm, gap=g, tie=tie)
        best, opt = brute.optimum(a, b, sc)
        score, ops = oracle.align(a, b, sc)
        assert score == best == oracle.score(a, b, sc)
        assert tuple(int(x) for x in ops) == brute.canonical(opt, tie)


def test_random_brute_force_protein_blosum62():
    rng = random.Random(2)
    for _ in range(60):
        a = bytes(rng.choice(nwgen.PROTEIN.encode()) for _ in range(rng.randint(0, 5)))
        b = bytes(rng.choice(nwgen.PROTEIN.encode()) for _ in range(rng.randint(0, 5)))
        tie = rng.choice(list(ORDERS.values()))
        sc = nwgen.Scoring(match=0, mismatch=0, gap=-5, alphabet=nwgen.PROTEIN,
                           subst=nwgen.BLOSUM62, tie=tie)
        best, opt = brute.optimum(a, b, sc)
        score, ops = oracle.align(a, b, sc)
        assert score == best
        assert tuple(int(x) for x in ops) == brute.canonical(opt, tie)


def test_delannoy_counts():
    assert brute.delannoy(3, 3) == 63 and brute.delannoy(7, 7) == 48639


# ---------------------------------------------------------------- closed forms

@pytest.mark.parametrize("m", [0, 1, 5, 50, 700])
def test_identical_sequences(m):
    a = nwgen.random_pair(7 + m, m, 0)[0]
    for tie in ORDERS.values():
        s, ops = oracle.align(a, a, _sc(tie=tie))
        assert s == m  # m * match
        assert (ops == oracle.D).all() and len(ops) == m


@pytest.mark.parametrize("m,n", [(7, 3), (3, 9), (40, 40), (1, 0), (0, 5), (300, 120)])
def test_disjoint_alphabets(m, n):
    """a = A^m, b = C^n: min(m,n)*max(mismatch, 2g) + |m-n|*g; under D>U>L the
    path is U^(m-n) D^n (m > n) or L^(n-m) D^m (m < n)."""
    a, b = b"A" * m, b"C" * n
    sc = _sc()
    s, ops = oracle.align(a, b, sc)
    assert s == min(m, n) * max(sc.mismatch, 2 * sc.gap) + abs(m - n) * sc.gap == -max(m, n)
    if m >= n:
        want = [oracle.U] * (m - n) + [oracle.D] * n
    else:
        want = [oracle.L] * (n - m) + [oracle.D] * m
    assert ops.tolist() == want


def test_edit_distance_scoring():
    """Scoring (0, -1, -1) gives -Levenshtein (independent Myers bit-vector)."""
    rng = np.random.Generator(np.random.PCG64(5))
    sc = _sc(match=0, mismatch=-1, gap=-1)
    for _ in range(60):
        a = nwgen.random_seq(rng, int(rng.integers(0, 300)))
        b = nwgen.random_seq(rng, int(rng.integers(0, 300)))
        assert oracle.score(a, b, sc) == -myers_edit_distance(a, b)


def test_empty_inputs():
    sc = _sc()
    assert oracle.align(b"", b"", sc)[0] == 0
    s, ops = oracle.align(b"", b"AA", sc)
    assert s == -2 and oracle.render(b"", b"AA", ops) == ("--", "AA")
    s, ops = oracle.align(b"ACG", b"", _sc(gap=-3))
    assert s == -9 and ops.tolist() == [oracle.U] * 3


# ---------------------------------------------------------------- invariants

def test_invariants_random():
    """Transpose, reverse, super-additivity, upper bound, validity, mirror."""
    rng = np.random.Generator(np.random.PCG64(11))
    mirror = {1: 1, 2: 3, 3: 2}
    for _ in range(80):
        m, n = int(rng.integers(0, 60)), int(rng.integers(0, 60))
        a, b = nwgen.random_seq(rng, m), nwgen.random_seq(rng, n)
        tie = list(ORDERS.values())[int(rng.integers(0, 6))]
        sc = _sc(tie=tie)
        H, T, s = oracle.fill(a, b, sc)
        Ht, _, st = oracle.fill(b, a, sc)
        assert (Ht == H.T).all() and s == st
        assert oracle.score(a[::-1], b[::-1], sc) == s
        k1, k2 = int(rng.integers(0, m + 1)), int(rng.integers(0, n + 1))
        assert s >= oracle.score(a[:k1], b[:k2], sc) + oracle.score(a[k1:], b[k2:], sc)
        assert s <= min(m, n) * sc.match + abs(m - n) * sc.gap
        ops = oracle.traceback(T)
        ga, gb = oracle.render(a, b, ops)
        assert oracle.column_score(ga, gb, sc) == s
        assert max(m, n) <= len(ops) <= m + n
        # mirror: trace(b, a, pi with U<->L) = row-swapped trace(a, b, pi)
        tie_m = tuple(mirror[x] for x in tie)
        _, ops_m = oracle.align(b, a, _sc(tie=tie_m))
        assert [mirror[int(x)] for x in ops_m] == ops.tolist()


def test_batch_matches_single_and_pair_count():
    ss = nwgen.random_set(3, 9, 0, 40)
    pairs = nwgen.all_pairs(ss.nseq)
    assert len(pairs) == 9 * 8 // 2
    out = oracle.batch_score(ss.residues, ss.offs, pairs, nwgen.PAPER_DNA, nthreads=3)
    for k, (p, q) in enumerate(pairs):
        assert out[k] == oracle.score(ss.seq(p), ss.seq(q), nwgen.PAPER_DNA)
        assert out[k] == oracle.score(ss.seq(q), ss.seq(p), nwgen.PAPER_DNA)


def test_alphabet_error_position():
    with pytest.raises(oracle.OracleError) as e:
        oracle.score(b"ACGT", b"ACNT", nwgen.PAPER_DNA)
    assert e.value.status == 2
