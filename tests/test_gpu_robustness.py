"""Error reporting, watchdog and handle lifetimes of the C ABI (SURVEY.md §8(b)
"Errors", §4 T5). GPU tests: every call goes through libnw_b200.so."""
import numpy as np
import pytest

import nwgen
import oracle
import paper_2412_21103_b200 as nwb

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = nwb.Context(0)
    yield c
    c.close()


def _dev(torch, x: bytes):
    return torch.frombuffer(bytearray(x), dtype=torch.uint8).cuda()


def test_dev_alphabet_error_is_sticky(ctx):
    """_dev(bad) then _dev(good) then sync: the first call's NW_E_ALPHABET must
    surface at the sync (the second call must not clear it), then be cleared."""
    import torch
    sc = nwgen.PAPER_DNA
    a, b = nwgen.random_pair(5, 300, 280)
    bad = bytearray(a)
    bad[123] = ord("N")
    d_score = torch.zeros(1, dtype=torch.int64, device="cuda")
    nwb.nw_score_only_dev(ctx, _dev(torch, bytes(bad)), _dev(torch, b), sc, d_score)
    nwb.nw_score_only_dev(ctx, _dev(torch, a), _dev(torch, b), sc, d_score)
    with pytest.raises(nwb.NWError) as e:
        ctx.sync()
    assert e.value.status == nwb.NW_E_ALPHABET and e.value.bad_pos == 123
    ctx.sync()  # reported once, then cleared
    assert nwb.nw_score_only(ctx, a, b, sc) == oracle.score(a, b, sc)


def test_dev_error_reported_by_next_host_call(ctx):
    """A pending _dev error is reported by the next synchronising host entry point."""
    import torch
    sc = nwgen.PAPER_DNA
    a, b = nwgen.random_pair(6, 200, 210)
    bad = bytearray(b)
    bad[7] = ord("x")
    d_score = torch.zeros(1, dtype=torch.int64, device="cuda")
    nwb.nw_score_only_dev(ctx, _dev(torch, a), _dev(torch, bytes(bad)), sc, d_score)
    with pytest.raises(nwb.NWError) as e:
        nwb.nw_score_only(ctx, a, b, sc)
    assert e.value.status == nwb.NW_E_ALPHABET and e.value.bad_pos == len(a) + 7
    assert nwb.nw_score_only(ctx, a, b, sc) == oracle.score(a, b, sc)


@pytest.mark.parametrize("nseq", [0, 1])
@pytest.mark.parametrize("flags", [0, 1])
def test_empty_batches(ctx, nseq, flags):
    """No pairs: an empty result, not NW_E_INVAL, host and device entry points."""
    import torch
    ss = nwgen.random_set(3, nseq, 10, 20)
    r = nwb.nw_align_batch(ctx, ss.residues, ss.offs, None, nwgen.PAPER_DNA, flags)
    scores = r[0] if flags else r
    assert len(scores) == 0
    d_seqs = torch.from_numpy(ss.residues).cuda() if len(ss.residues) else None
    d_offs = torch.from_numpy(ss.offs).cuda()
    nwb.nw_align_batch_dev(ctx, d_seqs, d_offs, ss.offs, None, None, 0, nwgen.PAPER_DNA, flags,
                           torch.zeros(0, dtype=torch.int32, device="cuda"))
    ctx.sync()


def test_handles_outlive_context():
    """Traceback and MSA handles freed after their context is closed: no access to
    the freed context; traceback with a detached handle is NW_E_STATE."""
    c = nwb.Context(0)
    a, b = nwgen.random_pair(8, 500, 450)
    _, tb = nwb.nw_align_pair(c, a, b, nwgen.PAPER_DNA)
    ss = nwgen.random_set(9, 5, 30, 60)
    msa = nwb.nw_msa_center_star(c, ss.residues, ss.offs, nwgen.PAPER_DNA)
    c.close()
    tb.free()
    msa.free()
    c2 = nwb.Context(0)
    _, tb2 = nwb.nw_align_pair(c2, a, b, nwgen.PAPER_DNA)
    c3 = nwb.Context(0)
    with pytest.raises(nwb.NWError) as e:
        nwb.nw_traceback(c3, tb2)
    assert e.value.status == nwb.NW_E_STATE
    tb2.free()
    c2.close()
    c3.close()


@pytest.mark.parametrize("withhold", [1, 3])
@pytest.mark.parametrize("dirs", [False, True])
def test_watchdog_fires_instead_of_hanging(ctx, opts, withhold, dirs):
    """Test hook: strip withhold-1 never publishes its bottom row, so the next
    strip's wait can never be satisfied. With a small watchdog the call must
    return NW_E_DEADLOCK (Code 1's unordered spin is the hazard), and the
    context must be usable afterwards."""
    a, b = nwgen.random_pair(10 + withhold, 2000, 1500)
    sc = nwgen.PAPER_DNA
    opts(ctx, "watchdog_polls", 20_000)
    opts(ctx, "test_withhold", withhold)
    with pytest.raises(nwb.NWError) as e:
        if dirs:
            nwb.nw_align_pair(ctx, a, b, sc)
        else:
            nwb.nw_score_only(ctx, a, b, sc)
    assert e.value.status == nwb.NW_E_DEADLOCK
    ctx.set_option("test_withhold", 0)
    assert nwb.nw_score_only(ctx, a, b, sc) == oracle.score(a, b, sc)


def test_options_validate(ctx):
    with pytest.raises(nwb.NWError) as e:
        ctx.set_option("rows_per_lane", -1)
    assert e.value.status == nwb.NW_E_INVAL
    assert ctx.get_option("rows_per_lane") == 0


def test_small_int32_traceback_batch_with_long_sequences(ctx):
    """int32 traceback batches (s - 2g < 0) size their per-warp scratch by the
    launched warps, which are capped by the pair count: a few pairs of 12k residues
    must run (it asked for ~160 GB before)."""
    sc = nwgen.Scoring(match=2, mismatch=-5, gap=-1)  # s - 2g < 0: int32 path
    ss = nwgen.random_set(12, 3, 12_000, 12_000)
    pairs = np.array([[0, 1], [2, 0]], dtype=np.int32)
    scores, *flat = nwb.nw_align_batch(ctx, ss.residues, ss.offs, pairs, sc, nwb.NW_TRACEBACK)
    paths = nwb.batch_paths(*flat)
    for k, (p, q) in enumerate(pairs):
        ws, wops = oracle.align(ss.seq(p), ss.seq(q), sc)
        assert scores[k] == ws and paths[k].tolist() == wops.tolist()
