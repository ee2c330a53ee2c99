"""Tall direction fills: the packed H' direction fill (default at 8+ rows per lane) vs the
int32 fill (pair_form 1), fill-kernel time and the score/path against each other."""
import sys
sys.path.insert(0, '.')
import torch
import nwgen
import paper_2412_21103_b200 as nwb

ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
for m, n in [(100_000, 3_000), (300_000, 2_000), (60_000, 20_000)]:
    a, b = nwgen.random_pair(7 + m, m, n)
    res = {}
    for form in (1, 0):
        ctx.set_option("pair_form", form)
        s0, tb = nwb.nw_align_pair(ctx, a, b, nwgen.PAPER_DNA)
        ops = nwb.nw_traceback(ctx, tb).tolist(); tb.free()
        torch.cuda.synchronize()
        ctx.set_timing(True); ctx.kernel_time(0)
        for _ in range(3):
            _, tb = nwb.nw_align_pair(ctx, a, b, nwgen.PAPER_DNA); tb.free()
        ms, k = ctx.kernel_time(0); ctx.set_timing(False)
        res[form] = (s0, ops, ms / k)
    print(m, n, "int32 %.3f ms, packed %.3f ms" % (res[1][2], res[0][2]), "same:", res[0][:2] == res[1][:2])
