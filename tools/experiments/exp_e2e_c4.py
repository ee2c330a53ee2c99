"""C4 through the host ABI (e2e): per-call wall time with page-locked in/out buffers,
and the same with pageable numpy buffers."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import nwgen
import paper_2412_21103_b200 as nwb
import bench

ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
ss = nwgen.config_c4()
pairs = nwgen.consecutive_pairs(ss.nseq // 2)
sc = nwgen.PROTEIN_BLOSUM62
oo = nwb.nw_batch_ops_offsets(ss.offs, pairs)
pin = lambda a: bench._pinned(torch, a)
h_res, h_offs, h_pairs = pin(ss.residues), pin(ss.offs), pin(pairs)
out = (pin(np.empty(len(pairs), np.int32)), pin(np.empty(int(oo[-1]) + 1, np.uint8)),
       pin(np.empty(len(pairs) + 1, np.int64)), pin(np.empty(len(pairs), np.int32)))
for label, args, kw in (("pinned", (h_res, h_offs, h_pairs), {"out": out}),
                        ("pageable", (ss.residues, ss.offs, pairs), {})):
    ts = []
    for _ in range(6):
        t0 = time.perf_counter()
        nwb.nw_align_batch(ctx, *args, sc, nwb.NW_TRACEBACK, **kw)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    t0 = time.perf_counter(); nwb.nw_batch_ops_offsets(ss.offs, pairs); t1 = time.perf_counter()
    print(label, "ms per call:", [round(t, 1) for t in ts], "ops_offsets host ms", round((t1 - t0) * 1e3, 1), flush=True)
