"""Pins of the center-star oracle (oracle/msa.py) to things other than itself.

SPEC.md S:263-301 examples (select_center, merge_alignments, msa), brute-force
optima (oracle/brute.py, no DP) for the center choice on tiny sets, and the
properties that define the union-gap merge: every row degaps to its input, all
rows have one length, no column is all gaps, each pairwise alignment survives
intact (projection onto rows (center, k) minus their common gap columns), the
width is the smallest that holds every alignment's center gapping, and the
result does not depend on the merge order.
"""
from __future__ import annotations

import random

import numpy as np
import pytest

import nwgen
import oracle
from oracle import brute, msa

ORDERS = [(1, 2, 3), (1, 3, 2), (2, 1, 3), (2, 3, 1), (3, 1, 2), (3, 2, 1)]


def _seqs(seed, n, lo, hi, alphabet="ACGT"):
    rng = random.Random(seed)
    return ["".join(rng.choice(alphabet) for _ in range(rng.randint(lo, hi))).encode()
            for _ in range(n)]


def _check_msa(seqs, center, rows, sc):
    n = len(seqs)
    assert len(rows) == n
    W = len(rows[0])
    assert all(len(r) == W for r in rows), "rows differ in length"
    for p in range(n):
        assert rows[p].replace("-", "").encode() == seqs[p], f"row {p} does not degap"
    for col in range(W):
        assert any(r[col] != "-" for r in rows), f"all-gap column {col}"
    # each pairwise alignment (center, k) is intact in the MSA
    cs = seqs[center]
    gc = [0] * (len(cs) + 1)  # union gapping: max over k of the gaps before center residue r
    for k in range(n):
        if k == center:
            continue
        _, ops = oracle.align(cs, seqs[k], sc)
        ca, ok = oracle.render(cs, seqs[k], ops)
        proj = [(x, y) for x, y in zip(rows[center], rows[k]) if not (x == "-" and y == "-")]
        assert "".join(x for x, _ in proj) == ca and "".join(y for _, y in proj) == ok, k
        r = run = 0
        for ch in ca:
            if ch == "-":
                run += 1
            else:
                gc[r] = max(gc[r], run); run = 0; r += 1
        gc[r] = max(gc[r], run)
    assert W == len(cs) + sum(gc), "MSA wider than the union gapping"


# ---------------------------------------------------------------- SPEC examples

def test_select_center_forced_argmax():
    """row sums [5, 9, 2] -> 1."""
    S = np.array([[0, 6, -1], [6, 0, 3], [-1, 3, 0]], dtype=np.int64)
    assert S.sum(axis=1).tolist() == [5, 9, 2]
    assert msa.select_center(S) == 1


def test_select_center_ties_lowest_index():
    """three identical sequences -> index 0; all-equal sums -> 0."""
    seqs = [b"ACGTAC"] * 3
    assert msa.select_center(msa.pair_score_matrix(seqs, nwgen.PAPER_DNA)) == 0
    assert msa.select_center(np.zeros((5, 5), dtype=np.int64)) == 0
    S = np.array([[0, 1, 2], [1, 0, 2], [2, 2, 0]])  # sums 3, 3, 4
    assert msa.select_center(S) == 2


def test_select_center_matches_brute_force():
    """the center equals an independently recomputed argmax of row sums,
    here from brute-force optima (every alignment enumerated, no DP)."""
    for seed in range(40):
        seqs = _seqs(seed, random.Random(seed).randint(2, 4), 0, 3, "AC")
        n = len(seqs)
        sums = [sum(brute.optimum(seqs[p], seqs[q], nwgen.PAPER_DNA)[0]
                    for q in range(n) if q != p) for p in range(n)]
        want = max(range(n), key=lambda p: (sums[p], -p))
        assert msa.select_center(msa.pair_score_matrix(seqs, nwgen.PAPER_DNA)) == want


def test_select_center_scale_invariant():
    """scaling all three scheme parameters by a positive integer keeps the center."""
    for seed in range(10):
        seqs = _seqs(100 + seed, 6, 5, 20)
        c1 = msa.select_center(msa.pair_score_matrix(seqs, nwgen.PAPER_DNA))
        c3 = msa.select_center(msa.pair_score_matrix(seqs, nwgen.Scoring(3, -3, -3)))
        assert c1 == c3


def test_msa_two_sequences_is_the_pairwise_alignment():
    """n = 2 -> the single pairwise alignment."""
    for a, b in [(b"GATTACA", b"GCATGCT"), (b"ACGT", b""), (b"AAC", b"CAAGT")]:
        c, rows = msa.msa([a, b], nwgen.PAPER_DNA)
        assert c == 0
        _, ops = oracle.align(a, b, nwgen.PAPER_DNA)
        assert tuple(rows) == oracle.render(a, b, ops)


def test_msa_identical_sequences_gap_free():
    """identical sequences -> identical gap-free rows."""
    c, rows = msa.msa([b"ACGTTGCA"] * 4, nwgen.PAPER_DNA)
    assert c == 0 and rows == ["ACGTTGCA"] * 4


def test_msa_spec_three_sequences():
    """{ACT, AT, ACGT}. Scores (+1/-1/-1): ACT/AT = 1, ACT/ACGT = 2,
    AT/ACGT = 0, so the center is ACT (sums 3, 1, 2). Only ACGT opens a center
    gap (between C and T), so the union center is AC-T; AT aligns A-T to ACT."""
    seqs = [b"ACT", b"AT", b"ACGT"]
    S = msa.pair_score_matrix(seqs, nwgen.PAPER_DNA)
    assert (S[0, 1], S[0, 2], S[1, 2]) == (1, 2, 0)
    c, rows = msa.msa(seqs, nwgen.PAPER_DNA)
    assert c == 0
    assert rows == ["AC-T", "A--T", "ACGT"]


# ---------------------------------------------------------------- merge properties

@pytest.mark.parametrize("alphabet,sc", [("ACGT", nwgen.PAPER_DNA),
                                          (nwgen.PROTEIN, nwgen.PROTEIN_BLOSUM62)])
def test_msa_invariants_random(alphabet, sc):
    """degapping, equal lengths, no all-gap column; plus each pairwise
    alignment intact and the minimal (union) width."""
    for seed in range(12):
        seqs = _seqs(1000 + seed, 2 + seed % 6, 0, 40, alphabet)
        c, rows = msa.msa(seqs, sc)
        _check_msa(seqs, c, rows, sc)


def test_msa_tie_orders():
    """The merge holds for every tie order (each order's canonical alignments)."""
    for tie in ORDERS:
        sc = nwgen.Scoring(tie=tie)
        seqs = _seqs(7, 6, 3, 25)
        c, rows = msa.msa(seqs, sc)
        _check_msa(seqs, c, rows, sc)


def test_merge_order_independent():
    """Merging the same alignments in reverse order gives the same rows."""
    for seed in range(10):
        seqs = _seqs(2000 + seed, 7, 1, 30)
        sc = nwgen.PAPER_DNA
        c = msa.select_center(msa.pair_score_matrix(seqs, sc))
        al = msa.align_all_to_center(seqs, c, sc)
        fwd = msa.merge_alignments(seqs[c], al, len(seqs), c)
        rev = msa.merge_alignments(seqs[c], al[::-1], len(seqs), c)
        assert fwd == rev


def test_merge_rejects_bad_center_row():
    """an alignment whose center row does not degap to the center is reported."""
    with pytest.raises(ValueError):
        msa.merge_alignments(b"ACT", [(1, "A-T", "AGT"), (2, "AC-", "ACG")], 3, 0)
