"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit-exact.

Scores and traceback op strings must be identical (north_star: "bit-exact
against this oracle for both scores and traceback strings"); all arithmetic is
integer, so the tolerance is zero. Inputs come from nwgen (seeded), sized to
span several strips (R = 256 rows) and ragged tails.
"""
from __future__ import annotations

import itertools

import numpy as np
import pytest

import nwgen
import oracle
import paper_2412_21103_b200 as nwb

pytestmark = pytest.mark.gpu

ORDERS = [(1, 2, 3), (1, 3, 2), (2, 1, 3), (2, 3, 1), (3, 1, 2), (3, 2, 1)]


@pytest.fixture(scope="module")
def ctx():
    c = nwb.Context(0)
    yield c
    c.close()


def _pair(seed, m, n, alphabet=nwgen.DNA):
    return nwgen.random_pair(seed, m, n, alphabet)


def check_pair(ctx, a, b, sc, with_ops=True):
    want_score, want_ops = oracle.align(a, b, sc)
    got_score, tb = nwb.nw_align_pair(ctx, a, b, sc)
    assert got_score == want_score, (len(a), len(b), sc.tie)
    if with_ops:
        got_ops = nwb.nw_traceback(ctx, tb)
        assert got_ops.tolist() == want_ops.tolist(), (len(a), len(b), sc.tie)
    tb.free()
    assert nwb.nw_score_only(ctx, a, b, sc) == want_score


SIZES = [1, 2, 31, 32, 33, 255, 256, 257, 513, 1000]


@pytest.mark.parametrize("m,n", [(m, n) for m, n in itertools.product(SIZES, SIZES)
                                 if (m * 7 + n) % 3 == 0 or m == n])
def test_pair_dna_sizes(ctx, m, n):
    a, b = _pair(1000 * m + n, m, n)
    check_pair(ctx, a, b, nwgen.PAPER_DNA)


@pytest.mark.parametrize("tie", ORDERS)
def test_pair_tie_orders(ctx, tie):
    for k, (m, n) in enumerate([(300, 277), (64, 700), (1200, 90), (7, 7)]):
        a, b = _pair(77 + k, m, n)
        check_pair(ctx, a, b, nwgen.Scoring(tie=tie))
    # low-complexity inputs make ties frequent
    rng = np.random.Generator(np.random.PCG64(3))
    a = nwgen.random_seq(rng, 600, "AC")
    b = nwgen.random_seq(rng, 555, "AC")
    check_pair(ctx, a, b, nwgen.Scoring(tie=tie))


@pytest.mark.parametrize("tie", [(1, 2, 3), (2, 3, 1)])
def test_pair_protein_blosum62(ctx, tie):
    sc = nwgen.Scoring(match=0, mismatch=0, gap=-5, alphabet=nwgen.PROTEIN,
                       subst=nwgen.BLOSUM62, tie=tie)
    for k, (m, n) in enumerate([(100, 1000), (999, 301), (257, 256), (5, 2)]):
        a, b = _pair(500 + k, m, n, nwgen.PROTEIN)
        check_pair(ctx, a, b, sc)


def test_pair_other_scorings(ctx):
    for k, (ma, mi, g) in enumerate([(2, -3, -2), (5, -4, -10), (1, 0, -1), (0, -1, -1)]):
        a, b = _pair(900 + k, 400, 380)
        check_pair(ctx, a, b, nwgen.Scoring(match=ma, mismatch=mi, gap=g))


def test_empty_and_degenerate(ctx):
    sc = nwgen.PAPER_DNA
    for a, b in [(b"", b""), (b"", b"ACG"), (b"ACGT", b""), (b"A", b"A"), (b"A", b"C")]:
        check_pair(ctx, a, b, sc)
    a = b"ACGT" * 200
    check_pair(ctx, a, a, sc)                      # identical: all diagonal
    check_pair(ctx, b"A" * 700, b"C" * 300, sc)    # disjoint alphabets


@pytest.mark.parametrize("m,n", [(600, 20000), (20000, 600), (3000, 7), (7, 3000)])
def test_long_thin_and_border_paths(ctx, m, n):
    """Paths with long horizontal runs inside one strip (unstaged traceback
    segments) and long vertical runs down column 0 (border moves)."""
    sc = nwgen.PAPER_DNA
    check_pair(ctx, b"A" * m, b"C" * n, sc)
    a, b = _pair(31337 + m, m, n)
    check_pair(ctx, a, b, sc)
    check_pair(ctx, a, b, nwgen.Scoring(tie=(3, 2, 1)))


def test_golden_worked_grid(ctx):
    sc = nwgen.Scoring(alphabet="ACGTU")
    for tie in ORDERS:
        check_pair(ctx, b"GATTACA", b"GCATGCU", nwgen.Scoring(alphabet="ACGTU", tie=tie))
    assert nwb.nw_score_only(ctx, b"GATTACA", b"GCATGCU", sc) == 0


def test_errors(ctx):
    sc = nwgen.PAPER_DNA
    with pytest.raises(nwb.NWError) as e:
        nwb.nw_align_pair(ctx, b"ACGTACGT", b"ACGNAC", sc)
    assert e.value.status == 2 and e.value.bad_pos == 8 + 3
    with pytest.raises(nwb.NWError) as e:
        nwb.nw_score_only(ctx, b"AC", b"AC", nwgen.Scoring(gap=1))
    assert e.value.status == 1
    with pytest.raises(nwb.NWError) as e:
        nwb.nw_score_only(ctx, b"AC", b"AC", nwgen.Scoring(tie=(1, 1, 2)))
    assert e.value.status == 1
    # traceback handle from another context
    other = nwb.Context(0)
    _, tb = nwb.nw_align_pair(other, b"ACGT", b"AGT", sc)
    with pytest.raises(nwb.NWError) as e:
        nwb.nw_traceback(ctx, tb)
    assert e.value.status == 7
    tb.free()
    other.close()


def test_c1_config(ctx):
    a, b = nwgen.config_c1()
    check_pair(ctx, a, b, nwgen.PAPER_DNA)


def test_c2_config_full(ctx):
    """BASELINE configs[1] at full size: 20,000 x 20,000, score + traceback."""
    a, b = nwgen.config_c2()
    check_pair(ctx, a, b, nwgen.PAPER_DNA)


def test_c2_closed_forms(ctx):
    n = 20000
    a = nwgen.config_c2()[0]
    s, tb = nwb.nw_align_pair(ctx, a, a, nwgen.PAPER_DNA)
    assert s == n and (nwb.nw_traceback(ctx, tb) == 1).all()
    s, tb = nwb.nw_align_pair(ctx, b"A" * n, b"C" * (n - 1), nwgen.PAPER_DNA)
    assert s == -n
    ops = nwb.nw_traceback(ctx, tb)
    assert ops.tolist() == [2] + [1] * (n - 1)


def test_dev_variants_match_host(ctx):
    import torch
    a, b = _pair(4242, 3000, 2500)
    sc = nwgen.PAPER_DNA
    want_score, want_ops = oracle.align(a, b, sc)
    da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
    db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
    d_score = torch.zeros(1, dtype=torch.int64, device="cuda")
    tb = nwb.nw_align_pair_dev(ctx, da, db, sc, d_score)
    d_ops = torch.zeros(len(a) + len(b), dtype=torch.uint8, device="cuda")
    d_len = torch.zeros(1, dtype=torch.int64, device="cuda")
    nwb.nw_traceback_dev(ctx, tb, d_ops, d_len)
    ctx.sync()
    assert int(d_score.item()) == want_score
    L = int(d_len.item())
    assert d_ops[:L].cpu().numpy().tolist() == want_ops.tolist()
    tb.free()
    d2 = torch.zeros(1, dtype=torch.int64, device="cuda")
    nwb.nw_score_only_dev(ctx, da, db, sc, d2)
    ctx.sync()
    assert int(d2.item()) == want_score


# ---------------------------------------------------------------- batch

def test_batch_all_pairs_dna(ctx):
    ss = nwgen.random_set(31, 40, 0, 700)
    want = oracle.batch_score(ss.residues, ss.offs, nwgen.all_pairs(ss.nseq), nwgen.PAPER_DNA)
    got = nwb.nw_align_batch(ctx, ss.residues, ss.offs, None, nwgen.PAPER_DNA)
    assert got.tolist() == want.tolist()


@pytest.mark.parametrize("lo,hi,sc", [
    (0, 700, nwgen.Scoring(match=2, mismatch=-5, gap=-2)),   # s - 2g < 0: int32 sweep
    (1, 3000, nwgen.Scoring(match=0, mismatch=-1, gap=-1)),  # edit-distance scoring, packed
    (5000, 9000, nwgen.PAPER_DNA),                           # long rows, packed (H' <= 27000)
])
def test_batch_score_paths(ctx, lo, hi, sc):
    ss = nwgen.random_set(34 + lo, 7, lo, hi)
    pairs = nwgen.all_pairs(ss.nseq)
    want = oracle.batch_score(ss.residues, ss.offs, pairs, sc)
    got = nwb.nw_align_batch(ctx, ss.residues, ss.offs, None, sc)
    assert got.tolist() == want.tolist()
    got2 = nwb.nw_align_batch(ctx, ss.residues, ss.offs, pairs[:, ::-1].copy(), sc)
    assert got2.tolist() == want.tolist()


def test_batch_packed_bound_fallback(ctx):
    """maxlen * max(s') > 65535 must take the int32 sweep (bit-exact either way)."""
    ss = nwgen.random_set(35, 3, 30000, 30500)
    pairs = nwgen.all_pairs(ss.nseq)
    want = oracle.batch_score(ss.residues, ss.offs, pairs, nwgen.PAPER_DNA)
    got = nwb.nw_align_batch(ctx, ss.residues, ss.offs, None, nwgen.PAPER_DNA)
    assert got.tolist() == want.tolist()


def test_batch_explicit_pairs_traceback_protein(ctx):
    ss = nwgen.random_set(32, 60, 0, 600, nwgen.PROTEIN)
    rng = np.random.Generator(np.random.PCG64(9))
    pairs = rng.integers(0, ss.nseq, size=(150, 2)).astype(np.int32)
    for tie in [(1, 2, 3), (3, 1, 2)]:
        sc = nwgen.Scoring(match=0, mismatch=0, gap=-5, alphabet=nwgen.PROTEIN,
                           subst=nwgen.BLOSUM62, tie=tie)
        scores, *flat = nwb.nw_align_batch(ctx, ss.residues, ss.offs, pairs, sc, nwb.NW_TRACEBACK)
        paths = nwb.batch_paths(*flat)
        for k, (p, q) in enumerate(pairs):
            ws, wops = oracle.align(ss.seq(p), ss.seq(q), sc)
            assert scores[k] == ws, k
            assert paths[k].tolist() == wops.tolist(), k


def test_batch_traceback_dna_all_pairs(ctx):
    ss = nwgen.random_set(33, 25, 1, 400)
    sc = nwgen.PAPER_DNA
    scores, *flat = nwb.nw_align_batch(ctx, ss.residues, ss.offs, None, sc, nwb.NW_TRACEBACK)
    paths = nwb.batch_paths(*flat)
    for k, (p, q) in enumerate(nwgen.all_pairs(ss.nseq)):
        ws, wops = oracle.align(ss.seq(p), ss.seq(q), sc)
        assert scores[k] == ws and paths[k].tolist() == wops.tolist()


def test_c3_full_size_sampled(ctx):
    """configs[2] at full size (2,048 seqs, 2,096,128 pairs), sampled vs oracle."""
    ss = nwgen.config_c3()
    got = nwb.nw_align_batch(ctx, ss.residues, ss.offs, None, nwgen.PAPER_DNA)
    pairs = nwgen.all_pairs(ss.nseq)
    assert len(got) == len(pairs) == 2096128
    rng = np.random.Generator(np.random.PCG64(1))
    idx = np.concatenate([rng.integers(0, len(pairs), 150), [0, len(pairs) - 1]])
    want = oracle.batch_score(ss.residues, ss.offs, pairs[idx], nwgen.PAPER_DNA)
    assert got[idx].tolist() == want.tolist()
    # symmetry of the score matrix: reversed pairs through the explicit path
    rev = pairs[idx][:, ::-1].copy()
    got_rev = nwb.nw_align_batch(ctx, ss.residues, ss.offs, rev, nwgen.PAPER_DNA)
    assert got_rev.tolist() == want.tolist()


def test_c4_full_size_sampled(ctx):
    """configs[3] at full size (100,000 protein pairs, traceback), sampled."""
    ss = nwgen.config_c4()
    pairs = nwgen.consecutive_pairs(100_000)
    sc = nwgen.PROTEIN_BLOSUM62
    scores, *flat = nwb.nw_align_batch(ctx, ss.residues, ss.offs, pairs, sc, nwb.NW_TRACEBACK)
    paths = nwb.batch_paths(*flat)
    rng = np.random.Generator(np.random.PCG64(2))
    for k in np.concatenate([rng.integers(0, len(pairs), 60), [0, len(pairs) - 1]]):
        p, q = pairs[k]
        ws, wops = oracle.align(ss.seq(p), ss.seq(q), sc)
        assert scores[k] == ws and paths[k].tolist() == wops.tolist(), k


# ---------------------------------------------------------------- score-only, large

def test_score_only_prefix_and_closed_forms_c5(ctx):
    """configs[4] sequences: a 40k x 40k prefix vs the oracle, and the 1M x 1M
    closed forms (identical -> 1e6; A^m vs C^n -> -1e6; (0,-1,-1) -> -edit distance
    checked at a smaller size)."""
    a, b = nwgen.config_c5()
    pa, pb = a[:40000], b[:40000]
    assert nwb.nw_score_only(ctx, pa, pb, nwgen.PAPER_DNA) == oracle.score(pa, pb, nwgen.PAPER_DNA)
    n = 1_000_000
    assert nwb.nw_score_only(ctx, a, a, nwgen.PAPER_DNA) == n
    assert nwb.nw_score_only(ctx, b"A" * n, b"C" * n, nwgen.PAPER_DNA) == -n
    from pins import myers_edit_distance
    sc = nwgen.Scoring(match=0, mismatch=-1, gap=-1)
    qa, qb = a[:3000], b[:2900]
    assert nwb.nw_score_only(ctx, qa, qb, sc) == -myers_edit_distance(qa, qb)


# ---------------------------------------------------------------- column blocks (a10)

CB_SCORINGS = {"h16": nwgen.PAPER_DNA,                                  # packed H', moving base
               "h16b": nwgen.Scoring(match=2, mismatch=-1, gap=-3),
               "d16": nwgen.PAPER_DNA,                                  # difference form
               "d16b": nwgen.Scoring(match=2, mismatch=-1, gap=-3),
               "int32": nwgen.Scoring(match=2, mismatch=-4, gap=-1)}     # s - 2g < 0: int32 H'


@pytest.mark.parametrize("form", sorted(CB_SCORINGS))
@pytest.mark.parametrize("m,n", [(1, 1), (300, 500), (1000, 5000), (3000, 700), (513, 2049), (2000, 7)])
@pytest.mark.parametrize("ranks,w", [(1, 0), (2, 64), (3, 1000), (8, 0), (5, 257), (4, 1)])
def test_cblock_virtual_ranks(ctx, opts, form, m, n, ranks, w):
    """Column-block wavefront across virtual ranks == oracle score (SURVEY §8(e) C5 path),
    all three arithmetic forms (pair_form 1 selects the difference form over the packed
    H' one), blocks down to one column, many calls on one context (the per-call tags of
    nw_cblock.cuh: buffers are never re-zeroed between calls)."""
    opts(ctx, "pair_form", 1 if form.startswith("d16") else 0)
    a, b = _pair(7000 + m + n, m, n)
    sc = CB_SCORINGS[form]
    assert nwb.nw_score_only_cblock(ctx, a, b, sc, ranks, w) == oracle.score(a, b, sc)


@pytest.mark.parametrize("reb", [1, 2])
def test_cblock_h16_frequent_rebase_tall(ctx, opts, reb):
    """The packed H' column-block form with the base moving every 1-2 groups on a pair
    tall enough for many strips, over 3 virtual ranks (left messages, corners, ring)."""
    opts(ctx, "h16_rebase", reb)
    a, b = _pair(7100 + reb, 40_000, 3_000)
    for sc in (nwgen.PAPER_DNA, nwgen.Scoring(match=31, mismatch=-30, gap=-15)):
        assert nwb.nw_score_only_cblock(ctx, a, b, sc, 3, 700) == oracle.score(a, b, sc)


def test_cblock_c5_prefix_and_closed_forms(ctx):
    a, b = nwgen.config_c5()
    pa, pb = a[:30000], b[:30000]
    sc = nwgen.PAPER_DNA
    assert nwb.nw_score_only_cblock(ctx, pa, pb, sc, 8, 1024) == oracle.score(pa, pb, sc)
    n = 1_000_000
    assert nwb.nw_score_only_cblock(ctx, a, a, sc, 8, 0) == n
    assert nwb.nw_score_only_cblock(ctx, a, b, sc, 4, 0) == nwb.nw_score_only(ctx, a, b, sc)


@pytest.mark.parametrize("m,n", [(100_000, 3000), (80_000, 5), (77_000, 1)])
def test_score_only_tall_difference_form(ctx, m, n):
    """Tall score-only pairs take the packed difference-form sweep (nw_fill_d16.cuh)."""
    a, b = _pair(8000 + n, m, n)
    for sc in (nwgen.PAPER_DNA, nwgen.Scoring(match=2, mismatch=-1, gap=-3)):
        assert nwb.nw_score_only(ctx, a, b, sc) == oracle.score(a, b, sc)


@pytest.mark.parametrize("chains", [0, 2])
@pytest.mark.parametrize("kr", [4, 8, 12, 14, 16, 18, 20, 22, 24, 26, 28, 30, 32])
def test_score_only_difference_form_every_kr(ctx, opts, kr, chains):
    """The packed score-only sweep at every rows-per-lane setting the library can pick
    (strip heights 128..1,024 rows, ragged last strips, one-strip pairs), with one or
    (rows per lane % 4 == 0) two independent chains per lane."""
    opts(ctx, "d16_force", kr)
    opts(ctx, "d16_chains", chains)
    for k, (m, n) in enumerate([(2500, 700), (32 * kr * 3 + 17, 333), (5, 900), (1, 1)]):
        a, b = _pair(9100 + 37 * kr + k, m, n)
        for sc in (nwgen.PAPER_DNA, nwgen.Scoring(match=2, mismatch=-1, gap=-3)):
            assert nwb.nw_score_only(ctx, a, b, sc) == oracle.score(a, b, sc), (kr, m, n)


def test_c5_default_strip_choice(ctx):
    """C5 at full size with the library's own rows-per-lane choice vs the closed forms."""
    a, _ = nwgen.config_c5()
    n = len(a)
    sc = nwgen.PAPER_DNA
    assert nwb.nw_score_only(ctx, a, a, sc) == n                         # a = b: m * match
    assert nwb.nw_score_only(ctx, b"A" * n, b"C" * n, sc) == -n           # disjoint: -max(m, n)


@pytest.mark.parametrize("G,w", [(2, 0), (3, 700)])
def test_cblock_rank_api_concurrent_streams(ctx, opts, G, w):
    """The per-rank (real multi-GPU) entry point, with the G ranks as concurrent
    launches on G streams of one GPU and plain device buffers as 'peer' memory."""
    import torch
    m, n = 5000, 9000
    a, b = _pair(9100 + G, m, n)
    sc = nwgen.PAPER_DNA
    streams = [torch.cuda.Stream() for _ in range(G)]
    ctxs = [nwb.Context(0, s.cuda_stream) for s in streams]
    for c in ctxs:  # every rank's warps must be resident at once: share the GPU
        c.set_option("cblock_warps_per_sm", 4)
    da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
    db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
    nbytes = nwb.nw_cblock_recv_bytes(m)
    bufs = [torch.zeros(nbytes, dtype=torch.uint8, device="cuda") for _ in range(G)]
    parts = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in range(G)]
    torch.cuda.synchronize()
    for r in range(G):
        nwb.nw_score_only_cblock_rank_dev(ctxs[r], da, db, sc, r, G, w, bufs[r], bufs[(r + 1) % G],
                                          parts[r])
    for c in ctxs:
        c.sync()
    assert sum(int(p.item()) for p in parts) == oracle.score(a, b, sc)
    # a second round on the same contexts and buffers (fresh tags, no re-zeroing)
    for p in parts:
        p.zero_()
    for r in range(G):
        nwb.nw_score_only_cblock_rank_dev(ctxs[r], da, db, sc, r, G, w, bufs[r], bufs[(r + 1) % G],
                                          parts[r])
    for c in ctxs:
        c.sync()
    assert sum(int(p.item()) for p in parts) == oracle.score(a, b, sc)
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("tie", ORDERS)
@pytest.mark.parametrize("scname", ["dna", "fallback", "protein"])
def test_batch_traceback_paths_all_orders(ctx, tie, scname):
    """Batch traceback: packed difference-form flags (s - 2g >= 0) and the int32
    fallback (s - 2g < 0), every tie order, ragged lengths across strip edges."""
    if scname == "protein":
        ss = nwgen.random_set(40 + sum(tie), 16, 1, 1100, nwgen.PROTEIN)
        sc = nwgen.Scoring(match=0, mismatch=0, gap=-5, alphabet=nwgen.PROTEIN,
                           subst=nwgen.BLOSUM62, tie=tie)
    else:
        ss = nwgen.random_set(50 + sum(tie), 14, 0, 1100)
        sc = nwgen.Scoring(tie=tie) if scname == "dna" else nwgen.Scoring(match=2, mismatch=-4,
                                                                        gap=-1, tie=tie)
    rng = np.random.Generator(np.random.PCG64(sum(tie)))
    pairs = rng.integers(0, ss.nseq, size=(40, 2)).astype(np.int32)
    scores, *flat = nwb.nw_align_batch(ctx, ss.residues, ss.offs, pairs, sc, nwb.NW_TRACEBACK)
    paths = nwb.batch_paths(*flat)
    for k, (p, q) in enumerate(pairs):
        ws, wops = oracle.align(ss.seq(p), ss.seq(q), sc)
        assert scores[k] == ws and paths[k].tolist() == wops.tolist(), (k, len(ss.seq(p)), len(ss.seq(q)))


@pytest.mark.parametrize("mode", ["waves", "kr16", "implicit", "notranspose", "asymmetric"])
def test_batch_traceback_two_phase_modes(ctx, opts, mode):
    """Two-phase batch traceback (the fill keeps every pair's flags, k_batch_walk walks
    them, one thread per pair; pairs whose last strip would waste more lanes are
    filled transposed under the mirrored tie order): split into many waves by a tiny
    direction budget, 16-rows-per-lane strips, all pairs (pairs=None: tasks in rank
    order over the length-sorted sequences) in waves, no transposition, and an
    asymmetric s (never transposed); pairs include empty sequences and lengths
    across strip edges."""
    subst = nwgen.BLOSUM62
    if mode == "kr16":
        opts(ctx, "batch_kr16", 16)
    elif mode == "notranspose":
        opts(ctx, "batch_no_transpose", 1)
    elif mode == "asymmetric":  # s(x,y) != s(y,x): never filled transposed
        subst = np.array(nwgen.BLOSUM62, dtype=np.int32).copy()
        subst[0, 1] += 2
        subst[5, 9] -= 1
    else:
        opts(ctx, "batch_tb_budget", 300_000)
    ss = nwgen.random_set(61, 30 if mode != "implicit" else 14, 0, 1300, nwgen.PROTEIN)
    rng = np.random.Generator(np.random.PCG64(61))
    pairs = rng.integers(0, ss.nseq, size=(120, 2)).astype(np.int32)
    if mode == "implicit":
        pairs = nwgen.all_pairs(ss.nseq)
    for tie in [(1, 2, 3), (2, 3, 1), (3, 1, 2)]:
        sc = nwgen.Scoring(match=0, mismatch=0, gap=-5, alphabet=nwgen.PROTEIN,
                           subst=subst, tie=tie)
        arg = None if mode == "implicit" else pairs
        scores, *flat = nwb.nw_align_batch(ctx, ss.residues, ss.offs, arg, sc, nwb.NW_TRACEBACK)
        paths = nwb.batch_paths(*flat)
        for k, (p, q) in enumerate(pairs):
            ws, wops = oracle.align(ss.seq(p), ss.seq(q), sc)
            assert scores[k] == ws and paths[k].tolist() == wops.tolist(), (mode, k)


@pytest.mark.parametrize("sym", [True, False])
def test_batch_score_only_orientation(ctx, opts, sym):
    """Score-only batches fill each pair in the orientation that wastes fewer strip
    rows when s is symmetric (Score(a,b) = Score(b,a)); an asymmetric s must keep
    a on the rows. Lengths straddle the 512-row strip edges in both directions."""
    subst = np.array([[3, -1, 0, -2], [-1, 2, -3, 0], [0, -3, 4, -1], [-2, 0, -1, 1]], dtype=np.int32)
    if not sym:
        subst[0, 1], subst[2, 3] = 1, -2  # s(A,C) != s(C,A), s(G,T) != s(T,G)
    sc = nwgen.Scoring(gap=-2, subst=subst)
    ss = nwgen.random_set(71 + sym, 12, 300, 1700)
    pairs = nwgen.all_pairs(ss.nseq)
    want = oracle.batch_score(ss.residues, ss.offs, pairs, sc)
    assert nwb.nw_align_batch(ctx, ss.residues, ss.offs, None, sc).tolist() == want.tolist()
    rev = pairs[:, ::-1].copy()
    assert nwb.nw_align_batch(ctx, ss.residues, ss.offs, rev, sc).tolist() == \
        oracle.batch_score(ss.residues, ss.offs, rev, sc).tolist()
    opts(ctx, "batch_no_transpose", 1)
    assert nwb.nw_align_batch(ctx, ss.residues, ss.offs, None, sc).tolist() == want.tolist()


@pytest.mark.parametrize("kr", [2, 4, 5, 6, 8, 10, 12])
def test_pair_every_rows_per_lane(ctx, opts, kr):
    """The single-pair fill + strip traceback at every rows-per-lane setting (5, 6, 10,
    12: strips of 160 / 192 / 320 / 384 rows, not powers of two), all tie orders on a
    tie-rich pair."""
    opts(ctx, "rows_per_lane", kr)
    for k, (m, n) in enumerate([(32 * kr * 3 + 17, 1500), (2000, 700), (700, 2100), (5, 9)]):
        a, b = _pair(9300 + 11 * kr + k, m, n)
        check_pair(ctx, a, b, nwgen.PAPER_DNA)
    rng = np.random.Generator(np.random.PCG64(kr))
    a = nwgen.random_seq(rng, 1400, "AC")
    b = nwgen.random_seq(rng, 1300, "AC")
    for tie in ORDERS:
        check_pair(ctx, a, b, nwgen.Scoring(tie=tie))
    sc = nwgen.Scoring(match=0, mismatch=0, gap=-5, alphabet=nwgen.PROTEIN,
                       subst=nwgen.BLOSUM62)        # K > 4: KR 5 / 6 fall back to 4
    a, b = _pair(9400 + kr, 900, 1000, nwgen.PROTEIN)
    check_pair(ctx, a, b, sc)


def test_batch_caller_owned_outputs(ctx):
    """nw_align_batch(out=...) fills caller-owned (e.g. page-locked) arrays with the
    same results as freshly allocated ones; too-small buffers are rejected."""
    ss = nwgen.random_set(81, 20, 0, 600, nwgen.PROTEIN)
    rng = np.random.Generator(np.random.PCG64(81))
    pairs = rng.integers(0, ss.nseq, size=(50, 2)).astype(np.int32)
    sc = nwgen.PROTEIN_BLOSUM62
    want = nwb.nw_align_batch(ctx, ss.residues, ss.offs, pairs, sc, nwb.NW_TRACEBACK)
    tot = int(nwb.nw_batch_ops_offsets(ss.offs, pairs)[-1])
    out = (np.empty(50, np.int32), np.empty(tot + 1, np.uint8), np.empty(51, np.int64),
           np.empty(50, np.int32))
    got = nwb.nw_align_batch(ctx, ss.residues, ss.offs, pairs, sc, nwb.NW_TRACEBACK, out=out)
    assert got[0] is out[0] and got[0].tolist() == want[0].tolist()
    assert [p.tolist() for p in nwb.batch_paths(*got[1:])] == \
        [p.tolist() for p in nwb.batch_paths(*want[1:])]
    s_out = np.empty(len(nwgen.all_pairs(ss.nseq)), np.int32)
    s = nwb.nw_align_batch(ctx, ss.residues, ss.offs, None, sc, out=s_out)
    assert s is s_out and s.tolist() == nwb.nw_align_batch(ctx, ss.residues, ss.offs, None, sc).tolist()
    with pytest.raises(ValueError):
        nwb.nw_align_batch(ctx, ss.residues, ss.offs, None, sc, out=s_out[:10])


@pytest.mark.parametrize("host_plan", [False, True])
def test_batch_traceback_device_plan(ctx, opts, host_plan):
    """Large explicit traceback batches (>= 4,096 pairs) are planned on the device
    (LPT buckets, orientation, word offsets) once the kept flag buffer is sized;
    NW_HOST_PLAN forces the host planner. Results are identical either way and equal
    the oracle's (scores of all pairs, paths of a sample)."""
    if host_plan:
        opts(ctx, "host_plan", 1)
    ss = nwgen.random_set(91, 400, 0, 260, nwgen.PROTEIN)
    rng = np.random.Generator(np.random.PCG64(91))
    pairs = rng.integers(0, ss.nseq, size=(5000, 2)).astype(np.int32)
    for tie in [(1, 2, 3), (3, 2, 1)]:
        sc = nwgen.Scoring(match=0, mismatch=0, gap=-5, alphabet=nwgen.PROTEIN,
                           subst=nwgen.BLOSUM62, tie=tie)
        for _ in range(2):  # the first call sizes the buffer (host plan), the second may use the device
            scores, *flat = nwb.nw_align_batch(ctx, ss.residues, ss.offs, pairs, sc, nwb.NW_TRACEBACK)
        want = oracle.batch_score(ss.residues, ss.offs, pairs, sc)
        assert scores.tolist() == want.tolist()
        paths = nwb.batch_paths(*flat)
        for k in rng.choice(len(pairs), 300, replace=False):
            p, q = pairs[k]
            ws, wops = oracle.align(ss.seq(p), ss.seq(q), sc)
            assert paths[k].tolist() == wops.tolist(), (k, tie)


@pytest.mark.parametrize("kr", [0, 1, 8, 16, 32])
def test_batch_score_only_u16_rows_per_lane(ctx, opts, kr):
    """The packed H' batch sweep at 8/16/32 rows per lane (1: 32 or 16 per pair; 0: chosen
    by the median length): pair lengths straddle the 256/512/1,024-row strip edges,
    empty sequences."""
    opts(ctx, "batch_u16_kr", kr)
    ss = nwgen.random_set(80 + kr, 26, 0, 2100)
    pairs = nwgen.all_pairs(ss.nseq)
    want = oracle.batch_score(ss.residues, ss.offs, pairs, nwgen.PAPER_DNA)
    assert nwb.nw_align_batch(ctx, ss.residues, ss.offs, None, nwgen.PAPER_DNA).tolist() == want.tolist()
    rev = pairs[::3, ::-1].copy()
    assert nwb.nw_align_batch(ctx, ss.residues, ss.offs, rev, nwgen.PAPER_DNA).tolist() == \
        oracle.batch_score(ss.residues, ss.offs, rev, nwgen.PAPER_DNA).tolist()


@pytest.mark.parametrize("w,w24", [(1, 0), (0, 1), (0, 0), (100000, 100000)])
def test_batch_u16_mixed_strip_heights(ctx, opts, w, w24):
    """Mixed 1,024/768/512-row strips (batch_u16_kr 1) with the weights pushing every pair
    to 512 rows (w = 1) or 768 rows (w24 = 1), the defaults, or to 1,024 rows; a symmetric
    scoring (the orientation may flip) and an asymmetric substitution matrix (it may not)."""
    opts(ctx, "batch_u16_kr", 1)
    opts(ctx, "batch_mix_w", w)
    opts(ctx, "batch_mix_w24", w24)
    ss = nwgen.random_set(9900 + w % 97 + w24 % 89, 24, 0, 2300)
    pairs = nwgen.all_pairs(ss.nseq)
    asym = np.array([[3, 0, 1, 0], [1, 2, 0, 0], [0, 1, 4, 2], [2, 0, 0, 3]], dtype=np.int32)
    for sc in (nwgen.PAPER_DNA, nwgen.Scoring(gap=-1, subst=asym)):
        want = oracle.batch_score(ss.residues, ss.offs, pairs, sc)
        assert nwb.nw_align_batch(ctx, ss.residues, ss.offs, None, sc).tolist() == want.tolist(), w
