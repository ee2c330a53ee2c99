"""Independent reference routines used to pin the oracle (test infrastructure).

Nothing here is the NW recurrence: these are textbook algorithms whose results
NW must reproduce in special cases (SURVEY.md §8(c) "Score closed forms").
"""
from __future__ import annotations


def myers_edit_distance(a: bytes, b: bytes) -> int:
    """Levenshtein distance by Myers' (1999) bit-vector algorithm (Hyyro's
    formulation) with Python big ints as the bit vectors -- a different algorithm
    from the DP: NW with scoring (0, -1, -1) must return -distance."""
    m = len(a)
    if m == 0:
        return len(b)
    peq = {}
    for i, c in enumerate(a):
        peq[c] = peq.get(c, 0) | (1 << i)
    mask = (1 << m) - 1
    high = 1 << (m - 1)
    pv, mv, score = mask, 0, m
    for c in b:
        eq = peq.get(c, 0)
        xv = eq | mv
        xh = (((eq & pv) + pv) ^ pv) | eq
        ph = mv | (~(xh | pv) & mask)
        mh = pv & xh
        if ph & high:
            score += 1
        elif mh & high:
            score -= 1
        ph = ((ph << 1) | 1) & mask
        mh = (mh << 1) & mask
        pv = mh | (~(xv | ph) & mask)
        mv = ph & xv
    return score


def levenshtein_rows(a: bytes, b: bytes) -> int:
    """Plain Wagner-Fischer, only for cross-checking myers_edit_distance."""
    prev = list(range(len(b) + 1))
    for i, x in enumerate(a, 1):
        cur = [i] + [0] * len(b)
        for j, y in enumerate(b, 1):
            cur[j] = min(prev[j] + 1, cur[j - 1] + 1, prev[j - 1] + (x != y))
        prev = cur
    return prev[-1]
