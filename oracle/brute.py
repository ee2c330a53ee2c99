"""Brute-force global alignment by enumeration -- TEST INFRASTRUCTURE ONLY.

The plain definition of what NW computes (SURVEY.md §8(c) "Score"): the
maximum, over every global alignment of a and b (columns (x, y), never both
gaps, degapping to a and b), of the column-score sum. No dynamic programming
is used here, so it pins the DP oracle from outside. The number of alignments
is the Delannoy number D(m, n) (63 at 3x3, 48,639 at 7x7): tiny inputs only.

Canonical alignment under a tie order pi (R6): the
optimal alignment whose op string read right-to-left is lexicographically
smallest when ops are ranked by their position in pi.
"""
from __future__ import annotations

import itertools

D, U, L = 1, 2, 3


def _sub(sc, x: int, y: int) -> int:
    if sc.subst is not None:
        return int(sc.subst[sc.alphabet.index(chr(x))][sc.alphabet.index(chr(y))])
    return sc.match if x == y else sc.mismatch


def alignments(m: int, n: int):
    """Every op string (tuple of 1/2/3) consuming m rows and n columns."""
    if m == 0 and n == 0:
        yield ()
        return
    if m > 0 and n > 0:
        for rest in alignments(m - 1, n - 1):
            yield rest + (D,)
    if m > 0:
        for rest in alignments(m - 1, n):
            yield rest + (U,)
    if n > 0:
        for rest in alignments(m, n - 1):
            yield rest + (L,)


def ops_score(a: bytes, b: bytes, ops, sc) -> int:
    i = j = 0
    total = 0
    for op in ops:
        if op == D:
            total += _sub(sc, a[i], b[j]); i += 1; j += 1
        elif op == U:
            total += sc.gap; i += 1
        else:
            total += sc.gap; j += 1
    return total


def optimum(a: bytes, b: bytes, sc):
    """(best score, list of every optimal op string)."""
    best, arg = None, []
    for ops in alignments(len(a), len(b)):
        s = ops_score(a, b, ops, sc)
        if best is None or s > best:
            best, arg = s, [ops]
        elif s == best:
            arg.append(ops)
    return best, arg


def canonical(opt_set, tie) -> tuple:
    rank = {code: r for r, code in enumerate(tie)}
    return min(opt_set, key=lambda ops: [rank[o] for o in reversed(ops)])


def delannoy(m: int, n: int) -> int:
    return sum(1 for _ in alignments(m, n))


def all_strings(alphabet: str, max_len: int):
    for ln in range(max_len + 1):
        for t in itertools.product(alphabet, repeat=ln):
            yield "".join(t).encode()
