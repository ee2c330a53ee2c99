"""Write tests/golden/digests.json: the CPU oracle's results on the BASELINE.json
configs at FULL size (SURVEY.md §8(c) row "C3 / C5 full-scale").

Imports only oracle/ (the plain scalar-C NW of PAPER.md P:43-72) and nwgen/
(seeded inputs, no method arithmetic) -- never the product package -- so every
stored value is the oracle's. The GPU parity tests (tests/test_gpu_fullsize.py)
recompute the same digests from the product's outputs.

Digest conventions (shared with the tests; they are serialisations, not math):
  scores  -> int32 little-endian array in pair order, SHA-256; plus one SHA-256
             per chunk of CHUNK pairs so a mismatch can be localised.
  ops     -> per pair the forward op codes (1 D, 2 U, 3 L) concatenated in
             pair order (SHA-256), and the int32 op lengths (SHA-256).

Usage: python tools/oracle_digests.py [c3] [c4] [c5] [tall]   (default: all)
Timings on the 8-core dev box: c3 ~8 min (threads), c4 ~1 min (processes),
c5 ~15 min (one core: the oracle is a serial two-row DP), tall ~20 s.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import nwgen  # noqa: E402
import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "digests.json")
CHUNK = 65536

# Tall pair for the packed difference-form path (m >= 76,800 rows): seed and shape.
TALL_SEED = nwgen.BASE_SEED + 10
TALL_M, TALL_N = 80_000, 20_000


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def score_digest(scores: np.ndarray) -> dict:
    s = np.ascontiguousarray(scores, dtype="<i4")
    return {"n": int(len(s)), "sha256": sha(s.tobytes()),
            "chunk": CHUNK,
            "chunks": [sha(s[k:k + CHUNK].tobytes()) for k in range(0, len(s), CHUNK)],
            "sum": int(s.astype(np.int64).sum()),
            "head": [int(x) for x in s[:8]]}


def ops_digest(ops_list: list[np.ndarray]) -> dict:
    lens = np.array([len(o) for o in ops_list], dtype="<i4")
    h = hashlib.sha256()
    for o in ops_list:
        h.update(np.ascontiguousarray(o, dtype=np.uint8).tobytes())
    return {"len_sha256": sha(lens.tobytes()), "ops_sha256": h.hexdigest(),
            "total_len": int(lens.astype(np.int64).sum())}


def _env_check():
    if "NW_SEED" in os.environ:
        raise SystemExit("unset NW_SEED: digests are for the default seeds")


def do_c3() -> dict:
    t0 = time.time()
    st = nwgen.config_c3()
    pairs = nwgen.all_pairs(st.nseq)
    sc = oracle.batch_score(st.residues, st.offs, pairs, nwgen.PAPER_DNA)
    lens = st.lengths()
    cells = int((lens[pairs[:, 0]] * lens[pairs[:, 1]]).sum())
    d = {"seed": nwgen.seed_for(3), "nseq": st.nseq, "npairs": int(len(pairs)), "cells": cells,
         "scoring": "+1/-1/-1", "order": "lexicographic p<q (P:131-135)",
         "scores": score_digest(sc.astype(np.int32)), "oracle_s": round(time.time() - t0, 1)}
    return d


_C4 = None


def _c4_init():
    global _C4
    _C4 = nwgen.config_c4()


def _c4_work(rng):
    lo, hi = rng
    st = _C4
    out = []
    for k in range(lo, hi):
        s, ops = oracle.align(st.seq(2 * k), st.seq(2 * k + 1), nwgen.PROTEIN_BLOSUM62)
        out.append((s, ops))
    return lo, out


def do_c4(npairs: int = 100_000) -> dict:
    t0 = time.time()
    st = nwgen.config_c4(npairs)
    lens = st.lengths()
    cells = int((lens[0::2] * lens[1::2]).sum())
    step = 500
    ranges = [(k, min(k + step, npairs)) for k in range(0, npairs, step)]
    res = {}
    with ProcessPoolExecutor(max_workers=len(os.sched_getaffinity(0)), initializer=_c4_init) as ex:
        for lo, out in ex.map(_c4_work, ranges):
            res[lo] = out
    scores, ops = [], []
    for lo, _ in ranges:
        for s, o in res[lo]:
            scores.append(s)
            ops.append(o)
    d = {"seed": nwgen.seed_for(4), "npairs": npairs, "cells": cells,
         "scoring": "BLOSUM62, gap -5, tie DUL", "pairs": "(2k, 2k+1)",
         "scores": score_digest(np.array(scores, dtype=np.int32)), "ops": ops_digest(ops),
         "oracle_s": round(time.time() - t0, 1)}
    return d


def do_c5() -> dict:
    t0 = time.time()
    a, b = nwgen.config_c5()
    s = oracle.score(a, b, nwgen.PAPER_DNA)
    return {"seed": nwgen.seed_for(5), "m": len(a), "n": len(b), "scoring": "+1/-1/-1",
            "score": int(s), "oracle_s": round(time.time() - t0, 1)}


def do_tall() -> dict:
    t0 = time.time()
    a, b = nwgen.random_pair(TALL_SEED, TALL_M, TALL_N)
    s, ops = oracle.align(a, b, nwgen.PAPER_DNA)
    return {"seed": TALL_SEED, "m": TALL_M, "n": TALL_N, "scoring": "+1/-1/-1, tie DUL",
            "score": int(s), "ops": ops_digest([ops]), "oracle_s": round(time.time() - t0, 1)}


def main(argv):
    _env_check()
    which = argv or ["tall", "c4", "c3", "c5"]
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            data = json.load(f)
    for w in which:
        print(f"[oracle_digests] {w} ...", flush=True)
        data[w] = {"c3": do_c3, "c4": do_c4, "c5": do_c5, "tall": do_tall}[w]()
        data["_about"] = ("Oracle-only digests (tools/oracle_digests.py imports oracle/ and "
                          "nwgen/ only); int32 LE scores, forward op codes 1/2/3 (P:90).")
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)
        print(f"[oracle_digests] {w} done in {data[w]['oracle_s']} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
