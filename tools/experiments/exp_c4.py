"""C4 step anatomy: host enqueue time vs device time per nw_align_batch_dev call,
fill and walk kernel times (the in-warp walk variant it was first compared with,
NW_BATCH_WALK_INWARP, is gone: profiles/r01_exp_c4_anatomy.txt)."""
import os, sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import nwgen
import paper_2412_21103_b200 as nwb

ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
ss = nwgen.config_c4()
pairs = nwgen.consecutive_pairs(ss.nseq // 2)
sc = nwgen.PROTEIN_BLOSUM62
d_seqs = torch.from_numpy(ss.residues).cuda()
d_offs = torch.from_numpy(ss.offs).cuda()
d_pairs = torch.from_numpy(pairs).cuda()
oo = nwb.nw_batch_ops_offsets(ss.offs, pairs)
d_oo = torch.from_numpy(oo).cuda()
d_ops = torch.zeros(int(oo[-1]) + 1, dtype=torch.uint8, device="cuda")
d_len = torch.zeros(len(pairs), dtype=torch.int32, device="cuda")
d_sc = torch.zeros(len(pairs), dtype=torch.int32, device="cuda")
for mode in os.environ.get("EXP_KR16", "0,0").split(","):
    ctx.set_option("batch_kr16", int(mode))
    run = lambda: nwb.nw_align_batch_dev(ctx, d_seqs, d_offs, ss.offs, d_pairs, pairs, len(pairs), sc,
                                         nwb.NW_TRACEBACK, d_sc, d_oo, d_ops, d_len)
    run(); run(); torch.cuda.synchronize()
    ctx.set_timing(True); ctx.kernel_time(0); ctx.kernel_time(1)
    host = []; dev = []
    for _ in range(4):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter(); run(); t1 = time.perf_counter()
        e1.record(); torch.cuda.synchronize()
        host.append((t1 - t0) * 1e3); dev.append(e0.elapsed_time(e1))
    f, nf = ctx.kernel_time(0); w, nw = ctx.kernel_time(1)
    ctx.set_timing(False)
    print(f"{mode}: host enqueue {np.median(host):.2f} ms, device {np.median(dev):.2f} ms, "
          f"fill {f/max(nf,1):.2f} ms x{nf//4}, walk {w/max(nw,1):.2f} ms x{nw//4}", flush=True)
