"""A/B of two library builds (NW_LIB_PATH) on C2 fill, C5 fill and C3 step (not a bench line).
Kernel event time of class 0 (fill) averaged over reps, L2 not flushed."""
import json, os, sys
sys.path.insert(0, '.')
import torch
import nwgen
import paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
out = {"lib": os.environ.get("NW_LIB_PATH", "default")}
d = torch.zeros(1, dtype=torch.int64, device="cuda")
def t(fn, reps):
    fn(); torch.cuda.synchronize(); ctx.set_timing(True); ctx.kernel_time(0)
    for _ in range(reps): fn()
    ms, k = ctx.kernel_time(0); ctx.set_timing(False); return round(ms / max(k, 1), 4)
for wl in sys.argv[1:]:
    if wl == "c2":
        a, b = nwgen.config_c2()
        da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda(); db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
        out["c2_fill_ms"] = t(lambda: nwb.nw_align_pair_dev(ctx, da, db, nwgen.PAPER_DNA, d).free(), 20)
    if wl == "c5":
        a, b = nwgen.config_c5()
        da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda(); db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
        out["c5_fill_ms"] = t(lambda: nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, d), 3)
        out["c5_score"] = int(d.item())
    if wl == "c3":
        ss = nwgen.config_c3()
        ds = torch.from_numpy(ss.residues).cuda(); do = torch.from_numpy(ss.offs).cuda()
        P = ss.nseq * (ss.nseq - 1) // 2
        sc = torch.zeros(P, dtype=torch.int32, device="cuda")
        out["c3_fill_ms"] = t(lambda: nwb.nw_align_batch_dev(ctx, ds, do, ss.offs, None, None, P, nwgen.PAPER_DNA, 0, sc), 3)
print(json.dumps(out))
