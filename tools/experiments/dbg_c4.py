import os, sys, time
sys.path.insert(0, '.')
import numpy as np, torch, nwgen
import paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
ss = nwgen.config_c4()
pairs = nwgen.consecutive_pairs(ss.nseq // 2)
sc = nwgen.PROTEIN_BLOSUM62
d_seqs = torch.from_numpy(ss.residues).cuda(); d_offs = torch.from_numpy(ss.offs).cuda()
d_pairs = torch.from_numpy(pairs).cuda()
oo = nwb.nw_batch_ops_offsets(ss.offs, pairs); d_oo = torch.from_numpy(oo).cuda()
d_ops = torch.zeros(int(oo[-1]) + 1, dtype=torch.uint8, device="cuda")
d_len = torch.zeros(len(pairs), dtype=torch.int32, device="cuda")
d_sc = torch.zeros(len(pairs), dtype=torch.int32, device="cuda")
for i in range(12):
    t0 = time.time()
    if i == 6: ctx.set_timing(True)
    nwb.nw_align_batch_dev(ctx, d_seqs, d_offs, ss.offs, d_pairs, pairs, len(pairs), sc, nwb.NW_TRACEBACK, d_sc, d_oo, d_ops, d_len)
    torch.cuda.synchronize()
    print(i, "ok", round((time.time() - t0) * 1e3, 2), "ms", flush=True)
    if i == 9:
        print(ctx.kernel_time(0), ctx.kernel_time(1), flush=True); ctx.set_timing(False)
