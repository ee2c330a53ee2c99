"""Center-star multiple alignment -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

SURVEY.md §8(f) NEXT #1. PAPER.md P:127-131 (Sec. 3.2): "the simple center star
multiple sequence alignment algorithm": compute the score of every pair (Eq. 2,
n(n-1)/2 alignments), take the sequence "most similar to the rest of the
sequences" as the center, "align all pairwise sequences with the center" and
"iteratively merge the alignments using the aligned center sequence as a
reference". SPEC.md S:263-301 states the operations (select_center,
align_all_to_center, merge_alignments, msa); the readings are DESIGN.md R20-R23:

  R20  similarity = the pairwise NW score with the same scoring; the center
       is argmax_p sum_{q != p} score(p, q), lowest index on ties.
  R21  alignment k pairs (center, k) with the center on the rows (a = center), the
       canonical traceback of the tie order (R6).
  R22  merge = "once a gap, always a gap": the alignments are merged one
       by one in increasing k; walking the current center row and alignment k's
       center row together, a gap column present in both takes k's residue, a
       gap column only in the MSA gives k a '-', and a gap only in alignment k
       inserts a new column (a '-' in every row merged so far).
  R23  rows are returned in input order; the center's row is the merged center.

Plain Python loops over strings; the pairwise scores and alignments come from
the scalar C oracle (oracle.score / oracle.align). Pins: tests/test_oracle_msa.py.
"""
from __future__ import annotations

import numpy as np

from . import align, render, score


def pair_score_matrix(seqs: list[bytes], sc) -> np.ndarray:
    """n x n symmetric int64 matrix of pairwise scores, diagonal 0."""
    n = len(seqs)
    S = np.zeros((n, n), dtype=np.int64)
    for p in range(n):
        for q in range(p + 1, n):
            S[p, q] = S[q, p] = score(seqs[p], seqs[q], sc)
    return S


def select_center(S: np.ndarray) -> int:
    """argmax over p of sum_{q != p} S[p, q]; lowest index on ties (R20)."""
    n = S.shape[0]
    best, best_sum = 0, None
    for p in range(n):
        tot = 0
        for q in range(n):
            if q != p:
                tot += int(S[p, q])
        if best_sum is None or tot > best_sum:
            best, best_sum = p, tot
    return best


def align_all_to_center(seqs: list[bytes], center: int, sc) -> list[tuple[int, str, str]]:
    """[(k, center_row, other_row)] for every k != center in increasing k (R21)."""
    out = []
    for k in range(len(seqs)):
        if k == center:
            continue
        _, ops = align(seqs[center], seqs[k], sc)
        ca, ok = render(seqs[center], seqs[k], ops)
        out.append((k, ca, ok))
    return out


def merge_alignments(center_seq: bytes, alignments: list[tuple[int, str, str]], n: int,
                     center: int) -> list[str]:
    """Union-gap merge of the pairwise alignments (R22); rows in input order."""
    if not alignments:
        return [center_seq.decode()]
    k0, c0, o0 = alignments[0]
    if c0.replace("-", "") != center_seq.decode():
        raise ValueError(f"alignment {k0}: center row does not degap to the center")
    mc = list(c0)                      # the merged center row
    rows: dict[int, list[str]] = {k0: list(o0)}
    for k, ck, ok in alignments[1:]:
        if ck.replace("-", "") != center_seq.decode():
            raise ValueError(f"alignment {k}: center row does not degap to the center")
        new_row: list[str] = []
        i = x = 0  # column in the MSA, column in alignment k
        while i < len(mc) or x < len(ck):
            m_gap = i < len(mc) and mc[i] == "-"
            k_gap = x < len(ck) and ck[x] == "-"
            if m_gap and k_gap:            # gap column in both: k's inserted residue
                new_row.append(ok[x]); i += 1; x += 1
            elif m_gap:                    # only the MSA has a gap here
                new_row.append("-"); i += 1
            elif k_gap:                    # only alignment k: a new column everywhere
                mc.insert(i, "-")
                for r in rows.values():
                    r.insert(i, "-")
                new_row.append(ok[x]); i += 1; x += 1
            else:                          # both at the same center residue
                new_row.append(ok[x]); i += 1; x += 1
        rows[k] = new_row
    out = []
    for p in range(n):
        out.append("".join(mc) if p == center else "".join(rows[p]))
    return out


def msa(seqs: list[bytes], sc) -> tuple[int, list[str]]:
    """(center, rows): the composition of S:294-297 (pairs -> center -> align -> merge)."""
    if len(seqs) < 2:
        raise ValueError("msa needs at least 2 sequences (S:295)")
    c = select_center(pair_score_matrix(seqs, sc))
    return c, merge_alignments(seqs[c], align_all_to_center(seqs, c, sc), len(seqs), c)
