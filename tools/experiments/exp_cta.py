"""C2 fill: plain one-warp CTAs vs CTAs of 2/3 strips with a shared-memory hand-off (not a bench line)."""
import json, sys
sys.path.insert(0, '.')
import torch
import nwgen, oracle
import paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
out = {}
a, b = nwgen.config_c2()
ws, wops = oracle.align(a, b, nwgen.PAPER_DNA)
d = torch.zeros(1, dtype=torch.int64, device="cuda")
da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda(); db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
def t(fn, reps=10):
    fn(); torch.cuda.synchronize(); ctx.set_timing(True); ctx.kernel_time(0)
    for _ in range(reps): fn()
    ms, k = ctx.kernel_time(0); ctx.set_timing(False); return round(ms / k, 4)
for w in (0, 2, 3):
    ctx.set_option("fill_cta", w)
    out[f"c2_dirs_cta{w}_fill_ms"] = t(lambda: nwb.nw_align_pair_dev(ctx, da, db, nwgen.PAPER_DNA, d).free())
    out[f"c2_score_cta{w}_fill_ms"] = t(lambda: nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, d))
    s, tb = nwb.nw_align_pair(ctx, a, b, nwgen.PAPER_DNA); ops = nwb.nw_traceback(ctx, tb); tb.free()
    out[f"c2_cta{w}_parity"] = bool(s == ws and ops.tolist() == wops.tolist())
    a1, b1 = nwgen.config_c1()
    s1, tb1 = nwb.nw_align_pair(ctx, a1, b1, nwgen.PAPER_DNA); o1 = nwb.nw_traceback(ctx, tb1); tb1.free()
    w1, wo1 = oracle.align(a1, b1, nwgen.PAPER_DNA)
    out[f"c1_cta{w}_parity"] = bool(s1 == w1 and o1.tolist() == wo1.tolist())
print(json.dumps(out, indent=1))
