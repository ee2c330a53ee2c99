"""Boundary chunks loaded 1 vs 2 groups ahead: C2 fill (+ parity vs oracle) and C5 (not a bench line)."""
import json, sys
sys.path.insert(0, '.')
import torch
import nwgen, oracle
import paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
out = {}
a, b = nwgen.config_c2()
ws, wops = oracle.align(a, b, nwgen.PAPER_DNA)
da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda(); db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
d = torch.zeros(1, dtype=torch.int64, device="cuda")
def t(fn, reps=10):
    fn(); torch.cuda.synchronize(); ctx.set_timing(True); ctx.kernel_time(0)
    for _ in range(reps): fn()
    ms, k = ctx.kernel_time(0); ctx.set_timing(False); return round(ms / k, 4)
for ah in (1, 2):
    ctx.set_option("chunk_ahead", ah)
    for kr in (2, 4, 8):
        ctx.set_option("rows_per_lane", kr)
        out[f"c2_kr{kr}_ahead{ah}_fill_ms"] = t(lambda: nwb.nw_align_pair_dev(ctx, da, db, nwgen.PAPER_DNA, d).free())
    ctx.set_option("rows_per_lane", 0)
    s, tb = nwb.nw_align_pair(ctx, a, b, nwgen.PAPER_DNA); ops = nwb.nw_traceback(ctx, tb); tb.free()
    out[f"c2_ahead{ah}_parity"] = bool(s == ws and ops.tolist() == wops.tolist())
a5, b5 = nwgen.config_c5()
da = torch.frombuffer(bytearray(a5), dtype=torch.uint8).cuda(); db = torch.frombuffer(bytearray(b5), dtype=torch.uint8).cuda()
for ah in (1, 2):
    ctx.set_option("chunk_ahead", ah)
    out[f"c5_ahead{ah}_ms"] = t(lambda: nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, d), reps=3)
    out[f"c5_ahead{ah}_score"] = int(d.item())
print(json.dumps(out, indent=1))
