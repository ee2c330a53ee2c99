"""Seeded synthetic inputs for the NW hot path.

This module is shared by the oracle side (tests/, bench.py cpu_baseline) and the
product side (bench.py, tests). It holds NO arithmetic of the method: it only
draws residues and lengths and carries the scoring *inputs* (alphabets, the
BLOSUM62 table) that both sides receive as arguments.

Recipe: numpy Generator(PCG64(seed)); lengths are drawn
first, then residues sequence by sequence; DNA uniform over ACGT, protein
uniform over the 20 standard amino acids. Base seed 21103 + config index,
overridable with NW_SEED.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

DNA = "ACGT"
PROTEIN = "ARNDCQEGHILKMFPSTWYV"
BASE_SEED = 21103

# BLOSUM62 over PROTEIN's order (Henikoff & Henikoff 1992), the substitution
# matrix input for config C4. Data, not arithmetic.
_BLOSUM62_ROWS = """
 4 -1 -2 -2  0 -1 -1  0 -2 -1 -1 -1 -1 -2 -1  1  0 -3 -2  0
-1  5  0 -2 -3  1  0 -2  0 -3 -2  2 -1 -3 -2 -1 -1 -3 -2 -3
-2  0  6  1 -3  0  0  0  1 -3 -3  0 -2 -3 -2  1  0 -4 -2 -3
-2 -2  1  6 -3  0  2 -1 -1 -3 -4 -1 -3 -3 -1  0 -1 -4 -3 -3
 0 -3 -3 -3  9 -3 -4 -3 -3 -1 -1 -3 -1 -2 -3 -1 -1 -2 -2 -1
-1  1  0  0 -3  5  2 -2  0 -3 -2  1  0 -3 -1  0 -1 -2 -1 -2
-1  0  0  2 -4  2  5 -2  0 -3 -3  1 -2 -3 -1  0 -1 -3 -2 -2
 0 -2  0 -1 -3 -2 -2  6 -2 -4 -4 -2 -3 -3 -2  0 -2 -2 -3 -3
-2  0  1 -1 -3  0  0 -2  8 -3 -3 -1 -2 -1 -2 -1 -2 -2  2 -3
-1 -3 -3 -3 -1 -3 -3 -4 -3  4  2 -3  1  0 -3 -2 -1 -3 -1  3
-1 -2 -3 -4 -1 -2 -3 -4 -3  2  4 -2  2  0 -3 -2 -1 -2 -1  1
-1  2  0 -1 -3  1  1 -2 -1 -3 -2  5 -1 -3 -1  0 -1 -3 -2 -2
-1 -1 -2 -3 -1  0 -2 -3 -2  1  2 -1  5  0 -2 -1 -1 -1 -1  1
-2 -3 -3 -3 -2 -3 -3 -3 -1  0  0 -3  0  6 -4 -2 -2  1  3 -1
-1 -2 -2 -1 -3 -1 -1 -2 -2 -3 -3 -1 -2 -4  7 -1 -1 -4 -3 -2
 1 -1  1  0 -1  0  0  0 -1 -2 -2  0 -1 -2 -1  4  1 -3 -2 -2
 0 -1  0 -1 -1 -1 -1 -2 -2 -1 -1 -1 -1 -2 -1  1  5 -2 -2  0
-3 -3 -4 -4 -2 -2 -3 -2 -2 -3 -2 -3 -1  1 -4 -3 -2 11  2 -3
-2 -2 -2 -3 -2 -1 -2 -3  2 -1 -1 -2 -1  3 -3 -2 -2  2  7 -1
 0 -3 -3 -3 -1 -2 -2 -3 -3  3  1 -2  1 -1 -2 -2  0 -3 -1  4
"""
BLOSUM62 = np.array([[int(x) for x in r.split()] for r in _BLOSUM62_ROWS.strip().splitlines()],
                    dtype=np.int32)
assert BLOSUM62.shape == (20, 20)


@dataclass(frozen=True)
class Scoring:
    """Scoring inputs (north_star: match/mismatch/gap scores, alphabet, tie order).

    tie: permutation of the P:90 codes (1 diag, 2 vertical, 3 horizontal), first
    = highest priority. subst: optional K*K int32 row-major over `alphabet`.
    """
    match: int = 1
    mismatch: int = -1
    gap: int = -1
    alphabet: str = DNA
    subst: np.ndarray | None = field(default=None, compare=False)
    tie: tuple = (1, 2, 3)


PAPER_DNA = Scoring()  # +1 / -1 / -1
PROTEIN_BLOSUM62 = Scoring(match=0, mismatch=0, gap=-5, alphabet=PROTEIN, subst=BLOSUM62)


def seed_for(config_index: int) -> int:
    env = os.environ.get("NW_SEED")
    return int(env) + config_index if env is not None else BASE_SEED + config_index


def random_seq(rng: np.random.Generator, length: int, alphabet: str = DNA) -> bytes:
    idx = rng.integers(0, len(alphabet), size=length)
    return np.frombuffer(alphabet.encode(), dtype=np.uint8)[idx].tobytes()


def random_pair(seed: int, m: int, n: int, alphabet: str = DNA) -> tuple[bytes, bytes]:
    rng = np.random.Generator(np.random.PCG64(seed))
    return random_seq(rng, m, alphabet), random_seq(rng, n, alphabet)


@dataclass
class SeqSet:
    """Concatenated sequences: residues[offs[k]:offs[k+1]] is sequence k."""
    residues: np.ndarray  # uint8
    offs: np.ndarray      # int64, nseq + 1

    @property
    def nseq(self) -> int:
        return len(self.offs) - 1

    def seq(self, k: int) -> bytes:
        return self.residues[self.offs[k]:self.offs[k + 1]].tobytes()

    def lengths(self) -> np.ndarray:
        return np.diff(self.offs)


def random_set(seed: int, nseq: int, lo: int, hi: int, alphabet: str = DNA) -> SeqSet:
    """nseq sequences with lengths uniform in [lo, hi]; lengths drawn first."""
    rng = np.random.Generator(np.random.PCG64(seed))
    lens = rng.integers(lo, hi + 1, size=nseq).astype(np.int64)
    offs = np.zeros(nseq + 1, dtype=np.int64)
    np.cumsum(lens, out=offs[1:])
    idx = rng.integers(0, len(alphabet), size=int(offs[-1]))
    res = np.frombuffer(alphabet.encode(), dtype=np.uint8)[idx]
    return SeqSet(np.ascontiguousarray(res, dtype=np.uint8), offs)


def all_pairs(nseq: int) -> np.ndarray:
    """All p<q in lexicographic order, shape (P, 2) int32."""
    p, q = np.triu_indices(nseq, k=1)
    return np.stack([p, q], axis=1).astype(np.int32)


def consecutive_pairs(npairs: int) -> np.ndarray:
    """(2k, 2k+1) pairs, the C4 protein-batch layout."""
    k = np.arange(npairs, dtype=np.int32)
    return np.stack([2 * k, 2 * k + 1], axis=1)


# ---- the BASELINE.json configs ----

def config_c1():
    """C1: two seeded 1,000-bp DNA sequences, +1/-1/-1, score + traceback."""
    return random_pair(seed_for(1), 1000, 1000)


def config_c2():
    """C2: two seeded 20,000-bp DNA sequences, +1/-1/-1, score + 2-bit traceback."""
    return random_pair(seed_for(2), 20000, 20000)


def config_c3(nseq: int = 2048):
    """C3: 2,048 DNA sequences of 500-2,000 bp; all p<q pairs, score-only."""
    return random_set(seed_for(3), nseq, 500, 2000)


def config_c4(npairs: int = 100_000):
    """C4: npairs protein pairs of 100-1,000 residues (2k, 2k+1), BLOSUM62, g=-5."""
    return random_set(seed_for(4), 2 * npairs, 100, 1000, PROTEIN)


def config_c5(length: int = 1_000_000):
    """C5: two seeded 1,000,000-bp DNA sequences, score-only."""
    return random_pair(seed_for(5), length, length)
