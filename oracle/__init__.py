"""CPU oracle for the NW hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package. The product path
(paper_2412_21103_b200/) never imports it, and it imports nothing from the
product path; both take their inputs from nwgen/.

Contents:
  nw_oracle.c   plain scalar C: fill (full H or two rows) + full uint8 direction
                matrix, traceback, two-row score-only, threaded batch of scores.
  brute.py      enumeration of every global alignment (tiny inputs): the plain
                definition of the optimum and of the canonical traceback.
  this file     ctypes binding + alignment helpers (render, column score).

Citations: PAPER.md P:24-74 (Sec. 2), P:90 (codes), P:131-135 (pairs).
Parity pins for every function live in tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nw_oracle.c")
_LIB_PATH = os.path.join(_HERE, "libnw_oracle.so")
D, U, L = 1, 2, 3


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"oracle status {status}: {what}")
        self.status = status


def build(force: bool = False) -> str:
    """Compile nw_oracle.c with gcc -O2 (plain C, no intrinsics)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", "-o",
                               _LIB_PATH, _SRC, "-lpthread"])
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        i64, i32, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
        _lib.nw_oracle_fill.argtypes = [vp, i64, vp, i64, ctypes.c_char_p, i32, vp, i32, i32, i32,
                                        vp, vp, vp, vp, vp]
        _lib.nw_oracle_traceback.argtypes = [vp, i64, i64, vp, i64, vp]
        _lib.nw_oracle_score.argtypes = [vp, i64, vp, i64, ctypes.c_char_p, i32, vp, i32, i32, i32,
                                         vp, vp]
        _lib.nw_oracle_batch_score.argtypes = [vp, vp, i32, vp, i64, ctypes.c_char_p, i32, vp, i32,
                                               i32, i32, vp, i32]
        for f in (_lib.nw_oracle_fill, _lib.nw_oracle_traceback, _lib.nw_oracle_score,
                  _lib.nw_oracle_batch_score):
            f.restype = ctypes.c_int
    return _lib


def _buf(x: bytes | np.ndarray) -> np.ndarray:
    if isinstance(x, (bytes, bytearray)):
        return np.frombuffer(bytes(x) + b"\0", dtype=np.uint8)
    return np.ascontiguousarray(x, dtype=np.uint8)


def _ptr(arr) -> int | None:
    return None if arr is None else arr.ctypes.data


def _scoring_args(sc):
    subst = None if sc.subst is None else np.ascontiguousarray(sc.subst, dtype=np.int32)
    return sc.alphabet.encode(), len(sc.alphabet), subst


def fill(a: bytes, b: bytes, sc, full_h: bool = True, dirs: bool = True):
    """(H int64 (m+1,n+1) or None, T uint8 (m+1,n+1) or None, score)."""
    m, n = len(a), len(b)
    alpha, K, subst = _scoring_args(sc)
    H = np.empty((m + 1, n + 1), dtype=np.int64) if full_h else None
    T = np.empty((m + 1, n + 1), dtype=np.uint8) if dirs else None
    tie = np.array(sc.tie, dtype=np.uint8)
    score = ctypes.c_int64(0)
    bad = ctypes.c_int64(-1)
    ab, bb = _buf(a), _buf(b)
    st = lib().nw_oracle_fill(_ptr(ab), m, _ptr(bb), n, alpha, K, _ptr(subst), sc.match,
                              sc.mismatch, sc.gap, _ptr(tie), _ptr(H), _ptr(T),
                              ctypes.addressof(score), ctypes.addressof(bad))
    if st:
        raise OracleError(st, f"fill (bad position {bad.value})")
    return H, T, score.value


def traceback(T: np.ndarray) -> np.ndarray:
    """Forward-order op codes (1 D, 2 U, 3 L) from the direction matrix."""
    m, n = T.shape[0] - 1, T.shape[1] - 1
    T = np.ascontiguousarray(T, dtype=np.uint8)
    ops = np.empty(m + n, dtype=np.uint8)
    ln = ctypes.c_int64(0)
    st = lib().nw_oracle_traceback(_ptr(T), m, n, _ptr(ops), m + n, ctypes.addressof(ln))
    if st:
        raise OracleError(st, "traceback")
    return ops[:ln.value].copy()


def align(a: bytes, b: bytes, sc):
    """(score, ops): fill with two-row H + full T, then traceback."""
    _, T, score = fill(a, b, sc, full_h=False, dirs=True)
    return score, traceback(T)


def score(a: bytes, b: bytes, sc) -> int:
    """Two-row score-only H(m,n)."""
    alpha, K, subst = _scoring_args(sc)
    out = ctypes.c_int64(0)
    bad = ctypes.c_int64(-1)
    ab, bb = _buf(a), _buf(b)
    st = lib().nw_oracle_score(_ptr(ab), len(a), _ptr(bb), len(b), alpha, K, _ptr(subst), sc.match,
                               sc.mismatch, sc.gap, ctypes.addressof(out), ctypes.addressof(bad))
    if st:
        raise OracleError(st, f"score (bad position {bad.value})")
    return out.value


def batch_score(residues: np.ndarray, offs: np.ndarray, pairs: np.ndarray, sc,
                nthreads: int | None = None) -> np.ndarray:
    """int64 scores of every (p, q) row of `pairs`."""
    alpha, K, subst = _scoring_args(sc)
    residues = np.ascontiguousarray(residues, dtype=np.uint8)
    offs = np.ascontiguousarray(offs, dtype=np.int64)
    pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
    out = np.empty(len(pairs), dtype=np.int64)
    nthreads = nthreads or len(os.sched_getaffinity(0))
    st = lib().nw_oracle_batch_score(_ptr(residues), _ptr(offs), len(offs) - 1, _ptr(pairs),
                                     len(pairs), alpha, K, _ptr(subst), sc.match, sc.mismatch,
                                     sc.gap, _ptr(out), nthreads)
    if st:
        raise OracleError(st, "batch_score")
    return out


def render(a: bytes, b: bytes, ops) -> tuple[str, str]:
    """Gapped strings from forward op codes: D -> (a_i, b_j), U -> (a_i, '-'),
    L -> ('-', b_j) (R5)."""
    ra, rb, i, j = [], [], 0, 0
    for op in ops:
        op = int(op)
        if op == D:
            ra.append(chr(a[i])); rb.append(chr(b[j])); i += 1; j += 1
        elif op == U:
            ra.append(chr(a[i])); rb.append("-"); i += 1
        elif op == L:
            ra.append("-"); rb.append(chr(b[j])); j += 1
        else:
            raise ValueError(f"bad op {op}")
    if i != len(a) or j != len(b):
        raise ValueError("ops do not consume both sequences")
    return "".join(ra), "".join(rb)


def column_score(ga: str, gb: str, sc) -> int:
    """Column sum of a gapped alignment (SPEC score_alignment): gap
    columns g, others s(x, y)."""
    if len(ga) != len(gb):
        raise ValueError("gapped strings differ in length")
    idx = {c: k for k, c in enumerate(sc.alphabet)}
    total = 0
    for x, y in zip(ga, gb):
        if x == "-" and y == "-":
            raise ValueError("double-gap column")
        if x == "-" or y == "-":
            total += sc.gap
        elif sc.subst is not None:
            total += int(sc.subst[idx[x]][idx[y]])
        else:
            total += sc.match if x == y else sc.mismatch
    return total
