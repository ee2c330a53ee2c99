"""GPU parity of the center-star MSA (nw_msa_center_star)
against oracle/msa.py: the center index and every gapped row identical."""
from __future__ import annotations

import numpy as np
import pytest

import nwgen
import oracle
from oracle import msa as omsa
import paper_2412_21103_b200 as nwb

pytestmark = pytest.mark.gpu

ORDERS = [(1, 2, 3), (1, 3, 2), (2, 1, 3), (2, 3, 1), (3, 1, 2), (3, 2, 1)]


@pytest.fixture(scope="module")
def ctx():
    c = nwb.Context(0)
    yield c
    c.close()


def _flat(seqs):
    offs = np.zeros(len(seqs) + 1, dtype=np.int64)
    offs[1:] = np.cumsum([len(s) for s in seqs])
    return np.frombuffer(b"".join(seqs), dtype=np.uint8) if offs[-1] else np.zeros(1, np.uint8), offs


def _gpu_msa(ctx, seqs, sc):
    res, offs = _flat(seqs)
    h = nwb.nw_msa_center_star(ctx, res, offs, sc)
    try:
        return h.center, h.rows()
    finally:
        h.free()


def _check(ctx, seqs, sc):
    want_c, want_rows = omsa.msa(seqs, sc)
    got_c, got_rows = _gpu_msa(ctx, seqs, sc)
    assert got_c == want_c
    assert got_rows == want_rows


def test_spec_examples(ctx):
    """n = 2, identical sequences, {ACT, AT, ACGT}."""
    sc = nwgen.PAPER_DNA
    assert _gpu_msa(ctx, [b"ACT", b"AT", b"ACGT"], sc) == (0, ["AC-T", "A--T", "ACGT"])
    assert _gpu_msa(ctx, [b"ACGTTGCA"] * 4, sc) == (0, ["ACGTTGCA"] * 4)
    for a, b in [(b"GATTACA", b"GCATGCT"), (b"ACGT", b""), (b"", b"ACG"), (b"AAC", b"CAAGT")]:
        _check(ctx, [a, b], sc)


@pytest.mark.parametrize("seed", range(6))
def test_random_dna_sets(ctx, seed):
    ss = nwgen.random_set(500 + seed, 3 + 5 * seed, 0 if seed % 2 else 1, 60 + 70 * seed)
    _check(ctx, [ss.seq(k) for k in range(ss.nseq)], nwgen.PAPER_DNA)


@pytest.mark.parametrize("tie", ORDERS)
def test_tie_orders_protein(ctx, tie):
    ss = nwgen.random_set(700, 9, 10, 120, nwgen.PROTEIN)
    sc = nwgen.Scoring(match=0, mismatch=0, gap=-5, alphabet=nwgen.PROTEIN, subst=nwgen.BLOSUM62,
                       tie=tie)
    _check(ctx, [ss.seq(k) for k in range(ss.nseq)], sc)


def test_related_family(ctx):
    """Homologous family (SURVEY.md §8(d) C3 variant): a root with ~10% point
    mutations and indels, truncated -- long shared gap blocks in the merge."""
    rng = np.random.Generator(np.random.PCG64(11))
    root = nwgen.random_seq(rng, 400)
    seqs = []
    for k in range(24):
        s = bytearray()
        for ch in root:
            u = rng.random()
            if u < 0.04:
                continue                                   # deletion
            s.append(b"ACGT"[rng.integers(0, 4)] if u < 0.10 else ch)
            if rng.random() < 0.03:
                s += nwgen.random_seq(rng, int(rng.integers(1, 6)))  # insertion
        lo = int(rng.integers(0, 60))
        seqs.append(bytes(s[lo:len(s) - int(rng.integers(0, 60))]))
    _check(ctx, seqs, nwgen.PAPER_DNA)


def test_medium_set(ctx):
    """96 sequences of 50-400 bp (4,560 pairs) in full."""
    ss = nwgen.random_set(900, 96, 50, 400)
    _check(ctx, [ss.seq(k) for k in range(ss.nseq)], nwgen.PAPER_DNA)


def test_dev_variant_matches_host(ctx):
    import torch
    ss = nwgen.random_set(901, 20, 5, 200)
    d_res = torch.from_numpy(ss.residues.copy()).cuda()
    d_offs = torch.from_numpy(ss.offs.copy()).cuda()
    h = nwb.nw_msa_center_star_dev(ctx, d_res, d_offs, ss.offs, nwgen.PAPER_DNA)
    got = (h.center, h.rows())
    h.free()
    assert got == omsa.msa([ss.seq(k) for k in range(ss.nseq)], nwgen.PAPER_DNA)


def test_errors(ctx):
    res, offs = _flat([b"ACGT"])
    with pytest.raises(nwb.NWError) as e:
        nwb.nw_msa_center_star(ctx, res, offs, nwgen.PAPER_DNA)
    assert e.value.status == 1  # NW_E_INVAL: n < 2
    res, offs = _flat([b"ACGT", b"ACXT"])
    with pytest.raises(nwb.NWError) as e:
        nwb.nw_msa_center_star(ctx, res, offs, nwgen.PAPER_DNA)
    assert e.value.status == 2  # NW_E_ALPHABET


def test_c3_full_size_properties(ctx):
    """configs[2] input (2,048 sequences): center = argmax of the (parity-tested)
    batch scores' row sums; rows degap, share one width, have no all-gap column;
    sampled pairwise alignments are intact against the oracle."""
    ss = nwgen.config_c3()
    sc = nwgen.PAPER_DNA
    h = nwb.nw_msa_center_star(ctx, ss.residues, ss.offs, sc)
    rows = h.rows_array()
    c = h.center
    h.free()
    scores = nwb.nw_align_batch(ctx, ss.residues, ss.offs, None, sc).astype(np.int64)
    n = ss.nseq
    p, q = np.triu_indices(n, k=1)
    sums = np.zeros(n, dtype=np.int64)
    np.add.at(sums, p, scores)
    np.add.at(sums, q, scores)
    assert c == int(np.flatnonzero(sums == sums.max())[0])
    gap = ord("-")
    assert rows.shape[0] == n
    assert not np.any(np.all(rows == gap, axis=0)), "all-gap column"
    for k in range(n):
        r = rows[k]
        assert r[r != gap].tobytes() == ss.seq(k)
    rng = np.random.Generator(np.random.PCG64(3))
    for k in rng.choice([x for x in range(n) if x != c], 12, replace=False):
        _, ops = oracle.align(ss.seq(c), ss.seq(int(k)), sc)
        ca, ok = oracle.render(ss.seq(c), ss.seq(int(k)), ops)
        keep = ~((rows[c] == gap) & (rows[k] == gap))
        assert rows[c][keep].tobytes().decode() == ca
        assert rows[k][keep].tobytes().decode() == ok
