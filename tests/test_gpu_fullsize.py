"""Full-size parity on the BASELINE.json configs themselves (SURVEY.md §8(c) row
"C3 / C5 full-scale"; VERDICT r1 "Next round" item 1).

Expected values: tests/golden/digests.json, written by tools/oracle_digests.py,
which imports only oracle/ (the plain scalar-C NW of P:43-72) and nwgen/. Every
output of these configs is compared, through the entry points bench.py times:
  C3  all 2,096,128 scores, nw_align_batch_dev (pairs=NULL)            P:131-135 (Eq. 2)
  C4  all 100,000 scores and op strings, nw_align_batch_dev(TRACEBACK)
  C5  H(m,n) of the seeded 1M x 1M pair: nw_score_only (packed difference form at
      the library's own rows-per-lane) and the column-block pipeline over 8 virtual ranks
  tall  80,000 x 20,000 (the difference form's first shape class): score, the
      full-direction traceback and the checkpointed (linear-memory) traceback.
Digests follow tools/oracle_digests.py: int32 LE scores in pair order; forward op
codes concatenated in pair order, and the int32 path lengths.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import nwgen
import paper_2412_21103_b200 as nwb

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
DIG_PATH = os.path.join(HERE, "golden", "digests.json")


def _dig():
    if not os.path.exists(DIG_PATH):
        pytest.fail("tests/golden/digests.json missing: run tools/oracle_digests.py")
    return json.load(open(DIG_PATH))


@pytest.fixture(scope="module")
def ctx():
    c = nwb.Context(0)
    yield c
    c.close()


def _sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def _check_scores(got: np.ndarray, want: dict):
    got = np.ascontiguousarray(got, dtype="<i4")
    assert len(got) == want["n"]
    if _sha(got.tobytes()) == want["sha256"]:
        return
    ch = want["chunk"]
    bad = [k for k, h in enumerate(want["chunks"]) if _sha(got[k * ch:(k + 1) * ch].tobytes()) != h]
    pytest.fail(f"scores differ from the oracle's in chunks {bad[:10]} (of {len(want['chunks'])}, "
                f"{ch} pairs each); sum {int(got.astype(np.int64).sum())} vs {want['sum']}")


def _check_ops(paths, want: dict):
    lens = np.array([len(p) for p in paths], dtype="<i4")
    h = hashlib.sha256()
    for p in paths:
        h.update(np.ascontiguousarray(p, dtype=np.uint8).tobytes())
    assert int(lens.astype(np.int64).sum()) == want["total_len"]
    assert _sha(lens.tobytes()) == want["len_sha256"]
    assert h.hexdigest() == want["ops_sha256"]


def test_c3_all_pairs_fullsize_dev(ctx):
    """Every C3 score through nw_align_batch_dev, the call bench.py times."""
    import torch
    d = _dig()["c3"]
    ss = nwgen.config_c3()
    assert nwgen.seed_for(3) == d["seed"]
    npairs = ss.nseq * (ss.nseq - 1) // 2
    d_seqs = torch.from_numpy(ss.residues).cuda()
    d_offs = torch.from_numpy(ss.offs).cuda()
    d_scores = torch.zeros(npairs, dtype=torch.int32, device="cuda")
    nwb.nw_align_batch_dev(ctx, d_seqs, d_offs, ss.offs, None, None, npairs, nwgen.PAPER_DNA,
                           nwb.NW_SCORE_ONLY, d_scores)
    ctx.sync()
    _check_scores(d_scores.cpu().numpy(), d["scores"])


def test_c4_protein_fullsize_dev(ctx):
    """Every C4 score and op string through nw_align_batch_dev(NW_TRACEBACK), twice
    (the second call plans on the device once the flag buffer is sized)."""
    import torch
    d = _dig()["c4"]
    ss = nwgen.config_c4()
    pairs = nwgen.consecutive_pairs(ss.nseq // 2)
    npairs = len(pairs)
    oo = nwb.nw_batch_ops_offsets(ss.offs, pairs)
    d_seqs = torch.from_numpy(ss.residues).cuda()
    d_offs = torch.from_numpy(ss.offs).cuda()
    d_pairs = torch.from_numpy(pairs).cuda()
    d_oo = torch.from_numpy(oo).cuda()
    for _ in range(2):
        d_scores = torch.zeros(npairs, dtype=torch.int32, device="cuda")
        d_ops = torch.zeros(int(oo[-1]) + 1, dtype=torch.uint8, device="cuda")
        d_len = torch.zeros(npairs, dtype=torch.int32, device="cuda")
        nwb.nw_align_batch_dev(ctx, d_seqs, d_offs, ss.offs, d_pairs, pairs, npairs,
                               nwgen.PROTEIN_BLOSUM62, nwb.NW_TRACEBACK, d_scores, d_oo, d_ops, d_len)
        ctx.sync()
        _check_scores(d_scores.cpu().numpy(), d["scores"])
        ops, ln = d_ops.cpu().numpy(), d_len.cpu().numpy()
        _check_ops(nwb.batch_paths(ops, oo, ln), d["ops"])


def test_c5_score_fullsize(ctx):
    """The seeded C5 pair's H(m,n): nw_score_only (host) and nw_score_only_dev."""
    import torch
    d = _dig()["c5"]
    a, b = nwgen.config_c5()
    assert nwb.nw_score_only(ctx, a, b, nwgen.PAPER_DNA) == d["score"]
    d_score = torch.zeros(1, dtype=torch.int64, device="cuda")
    nwb.nw_score_only_dev(ctx, torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda(),
                          torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda(),
                          nwgen.PAPER_DNA, d_score)
    ctx.sync()
    assert int(d_score.item()) == d["score"]


@pytest.mark.parametrize("ranks", [8])
def test_c5_cblock_virtual_ranks_fullsize(ctx, ranks):
    """The column-block pipeline (a10) over 8 virtual ranks on the seeded C5 pair."""
    d = _dig()["c5"]
    a, b = nwgen.config_c5()
    assert nwb.nw_score_only_cblock(ctx, a, b, nwgen.PAPER_DNA, ranks) == d["score"]


def test_tall_pair_difference_form(ctx):
    """80,000 x 20,000 random DNA: score-only through the packed difference form
    at its default rows per lane, plus the full-direction and the checkpointed
    tracebacks, against the oracle's score and op string."""
    d = _dig()["tall"]
    a, b = nwgen.random_pair(d["seed"], d["m"], d["n"])
    sc = nwgen.PAPER_DNA
    assert nwb.nw_score_only(ctx, a, b, sc) == d["score"]
    s, tb = nwb.nw_align_pair(ctx, a, b, sc)
    ops = nwb.nw_traceback(ctx, tb)
    tb.free()
    assert s == d["score"]
    _check_ops([ops], d["ops"])
    for budget in (0, 40_000_000):
        s, ops = nwb.nw_align_pair_linear(ctx, a, b, sc, budget)
        assert s == d["score"]
        _check_ops([ops], d["ops"])
