"""Co-optimal alignments -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

SURVEY.md §8(f) NEXT #2. PAPER.md P:74 (Sec. 2.4): "there may be multiple
paths ... all such paths are considered valid alignments". SPEC.md S:146-154
(traceback_all): depth-first enumeration from (m, n) along branches that
reproduce the cell's score, at most `cap` alignments, deterministic order.
Readings (R24-R25):

  R24  A branch X of cell (i, j) is optimal when its candidate equals H(i, j)
       (Eq. 1); border cells have the forced branch (U on column 0, L on
       row 0). The number of optimal alignments is the number of
       (m, n) -> (0, 0) paths along optimal branches: N(0, 0) = 1, N on the
       borders = 1, N(i, j) = sum of N(predecessor) over the optimal branches.
  R25  The enumeration is depth-first from (m, n), trying the optimal branches of
       each cell in the tie order pi (SPEC names D, U, L: that is pi = DUL; in
       general the tie order, so that the first path is the canonical traceback,
       S:152). Paths are returned in forward order.

Plain Python loops (exact big integers); small inputs only.
Pins: tests/test_oracle_cooptimal.py.
"""
from __future__ import annotations

D, U, L = 1, 2, 3


def _sub(sc, x: int, y: int) -> int:
    if sc.subst is not None:
        idx = {c: k for k, c in enumerate(sc.alphabet)}
        return int(sc.subst[idx[chr(x)]][idx[chr(y)]])
    return sc.match if x == y else sc.mismatch


def masks_and_counts(a: bytes, b: bytes, sc):
    """(H, M, N): full score grid, optimal-branch bit masks (bit X-1 set when
    branch X is optimal) and exact path counts N, all (m+1) x (n+1) lists."""
    m, n, g = len(a), len(b), sc.gap
    H = [[0] * (n + 1) for _ in range(m + 1)]
    M = [[0] * (n + 1) for _ in range(m + 1)]
    N = [[0] * (n + 1) for _ in range(m + 1)]
    N[0][0] = 1
    for i in range(1, m + 1):
        H[i][0], M[i][0], N[i][0] = i * g, 1 << (U - 1), 1
    for j in range(1, n + 1):
        H[0][j], M[0][j], N[0][j] = j * g, 1 << (L - 1), 1
    for i in range(1, m + 1):
        for j in range(1, n + 1):
            cD = H[i - 1][j - 1] + _sub(sc, a[i - 1], b[j - 1])
            cU = H[i - 1][j] + g
            cL = H[i][j - 1] + g
            h = max(cD, cU, cL)
            H[i][j] = h
            mk = 0
            cnt = 0
            if cD == h:
                mk |= 1 << (D - 1); cnt += N[i - 1][j - 1]
            if cU == h:
                mk |= 1 << (U - 1); cnt += N[i - 1][j]
            if cL == h:
                mk |= 1 << (L - 1); cnt += N[i][j - 1]
            M[i][j], N[i][j] = mk, cnt
    return H, M, N


def count(a: bytes, b: bytes, sc) -> int:
    """Number of optimal global alignments (R24), exact."""
    return masks_and_counts(a, b, sc)[2][len(a)][len(b)]


def enumerate_optimal(a: bytes, b: bytes, sc, cap: int) -> list[list[int]]:
    """First `cap` optimal alignments in depth-first order (R25), forward op codes."""
    _, M, _ = masks_and_counts(a, b, sc)
    out: list[list[int]] = []
    rev: list[int] = []  # ops from (m, n) backwards

    def dfs(i: int, j: int) -> None:
        if len(out) >= cap:
            return
        if i == 0 and j == 0:
            out.append(rev[::-1])
            return
        for x in sc.tie:
            if not (M[i][j] >> (x - 1)) & 1:
                continue
            rev.append(x)
            dfs(i - (x != L), j - (x != U))
            rev.pop()
            if len(out) >= cap:
                return

    import sys
    old = sys.getrecursionlimit()
    sys.setrecursionlimit(max(old, 4 * (len(a) + len(b)) + 100))
    try:
        dfs(len(a), len(b))
    finally:
        sys.setrecursionlimit(old)
    return out
