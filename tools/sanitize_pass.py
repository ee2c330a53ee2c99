"""One small invocation of every kernel family behind include/nw.h, for
compute-sanitizer:

  compute-sanitizer --tool memcheck  python tools/sanitize_pass.py
  compute-sanitizer --tool synccheck python tools/sanitize_pass.py
  compute-sanitizer --tool racecheck python tools/sanitize_pass.py

Each call's result is also checked against the oracle (a sanitizer run that
changes results would show here). `dist` as the first argument adds the NCCL
dist-context paths (world 1)."""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import nwgen
import oracle
import paper_2412_21103_b200 as nwb

ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
DNA, PROT = nwgen.PAPER_DNA, nwgen.PROTEIN_BLOSUM62
NEG = nwgen.Scoring(match=2, mismatch=-4, gap=-1)  # s - 2g < 0: the int32 forms
done = []


def ok(name, cond):
    if not cond:
        raise SystemExit(f"MISMATCH in {name}")
    done.append(name)


# single pair: fill + directions + strip traceback (int32), several rows-per-lane settings
a, b = nwgen.random_pair(1, 700, 650)
for kr in (0, 2, 8):
    ctx.set_option("rows_per_lane", kr)
    s, tb = nwb.nw_align_pair(ctx, a, b, DNA)
    ops = nwb.nw_traceback(ctx, tb)
    tb.free()
    ws, wops = oracle.align(a, b, DNA)
    ok(f"pair kr{kr}", s == ws and ops.tolist() == wops.tolist())
ctx.set_option("rows_per_lane", 0)
pa, pb = nwgen.random_pair(2, 300, 280, nwgen.PROTEIN)
s, tb = nwb.nw_align_pair(ctx, pa, pb, PROT)
ok("pair protein", s == oracle.align(pa, pb, PROT)[0] and nwb.nw_traceback(ctx, tb).tolist()
   == oracle.align(pa, pb, PROT)[1].tolist())
tb.free()
# score-only: int32 strips and the packed difference form
ok("score int32", nwb.nw_score_only(ctx, a, b, NEG) == oracle.score(a, b, NEG))
ctx.set_option("d16_force", 16)
ok("score d16", nwb.nw_score_only(ctx, a, b, DNA) == oracle.score(a, b, DNA))
ctx.set_option("d16_force", 0)
# packed H' with a moving base (nw_fill_h16), rebasing every group
ctx.set_option("h16_kr", 16)
ctx.set_option("h16_rebase", 1)
ah, bh = nwgen.random_pair(6, 2100, 700)
ok("score h16", nwb.nw_score_only(ctx, ah, bh, DNA) == oracle.score(ah, bh, DNA))
ctx.set_option("h16_kr", 0)
ctx.set_option("h16_rebase", 0)
# batches: u16 score-only (implicit), d16 (long), int32; traceback two-phase + int32
ss = nwgen.random_set(3, 10, 0, 400)
ok("batch u16", nwb.nw_align_batch(ctx, ss.residues, ss.offs, None, DNA).tolist()
   == oracle.batch_score(ss.residues, ss.offs, nwgen.all_pairs(ss.nseq), DNA).tolist())
ctx.set_option("batch_u16_kr", 1)  # mixed 1,024/512-row strips
ok("batch u16 mixed", nwb.nw_align_batch(ctx, ss.residues, ss.offs, None, DNA).tolist()
   == oracle.batch_score(ss.residues, ss.offs, nwgen.all_pairs(ss.nseq), DNA).tolist())
ctx.set_option("batch_u16_kr", 0)
sl = nwgen.random_set(4, 4, 3000, 5000)
ok("batch d16", nwb.nw_align_batch(ctx, sl.residues, sl.offs, None, DNA).tolist()
   == oracle.batch_score(sl.residues, sl.offs, nwgen.all_pairs(sl.nseq), DNA).tolist())
ok("batch int32", nwb.nw_align_batch(ctx, ss.residues, ss.offs, None, NEG).tolist()
   == oracle.batch_score(ss.residues, ss.offs, nwgen.all_pairs(ss.nseq), NEG).tolist())
sp = nwgen.random_set(5, 12, 0, 300, nwgen.PROTEIN)
pairs = np.array([[k, (k * 5 + 1) % 12] for k in range(12)], dtype=np.int32)
for sc, name in ((PROT, "batch tb two-phase"), (nwgen.Scoring(match=0, mismatch=0, gap=-1,
                 alphabet=nwgen.PROTEIN, subst=nwgen.BLOSUM62), "batch tb int32")):
    scores, *flat = nwb.nw_align_batch(ctx, sp.residues, sp.offs, pairs, sc, nwb.NW_TRACEBACK)
    paths = nwb.batch_paths(*flat)
    good = all(scores[k] == oracle.align(sp.seq(p), sp.seq(q), sc)[0] and
               paths[k].tolist() == oracle.align(sp.seq(p), sp.seq(q), sc)[1].tolist()
               for k, (p, q) in enumerate(pairs))
    ok(name, good)
# MSA, co-optimal, per-cell kernel, checkpointed traceback
ms = nwgen.random_set(6, 6, 20, 80)
msa = nwb.nw_msa_center_star(ctx, ms.residues, ms.offs, DNA)
rows = msa.rows()
msa.free()
ok("msa", len(rows) == 6 and all(r.replace("-", "").encode() == ms.seq(k) for k, r in enumerate(rows)))
ca, cb = nwgen.random_pair(7, 60, 55)
cnt, sat, paths = nwb.nw_cooptimal(ctx, ca, cb, DNA, 8)
ok("cooptimal", paths[0].tolist() == oracle.align(ca, cb, DNA)[1].tolist())
s, ops = nwb.nw_align_pair_percell(ctx, ca, cb, DNA)
ok("percell", s == oracle.align(ca, cb, DNA)[0] and ops.tolist() == oracle.align(ca, cb, DNA)[1].tolist())
la, lb = nwgen.random_pair(8, 2000, 1500)
s, ops = nwb.nw_align_pair_linear(ctx, la, lb, DNA, 200_000)
ok("linear", s == oracle.align(la, lb, DNA)[0] and ops.tolist() == oracle.align(la, lb, DNA)[1].tolist())
# column blocks: virtual ranks, both forms
for sc, name in ((DNA, "cblock d16"), (NEG, "cblock int32")):
    ok(name, nwb.nw_score_only_cblock(ctx, la, lb, sc, 3, 300) == oracle.score(la, lb, sc))
if len(sys.argv) > 1 and sys.argv[1] == "dist":
    c2 = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
    c2.set_dist(0, 1, nwb.nw_dist_unique_id())
    ok("dist batch", nwb.nw_align_batch(c2, ss.residues, ss.offs, None, DNA).tolist()
       == oracle.batch_score(ss.residues, ss.offs, nwgen.all_pairs(ss.nseq), DNA).tolist())
    c2.set_option("dist_pipeline", 1)
    ok("dist pipeline", nwb.nw_score_only(c2, la, lb, DNA) == oracle.score(la, lb, DNA))
    c2.close()
ctx.close()
print(f"sanitize pass ok: {len(done)} checks: {', '.join(done)}")
