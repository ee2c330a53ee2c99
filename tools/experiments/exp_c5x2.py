"""C5 fill time: one vs two chains per lane, rows per lane 16..32 (not a bench line)."""
import json, sys
sys.path.insert(0, '.')
import torch
import nwgen
import paper_2412_21103_b200 as nwb
a, b = nwgen.config_c5()
sc = nwgen.PAPER_DNA
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
d = torch.zeros(1, dtype=torch.int64, device="cuda")
out = {}
for kr in [0, 16, 20, 24, 28, 32]:
    for ch in [0, 1]:
        ctx.set_option("d16_kr", kr)
        ctx.set_option("d16_chains", ch)
        nwb.nw_score_only_dev(ctx, da, db, sc, d); torch.cuda.synchronize()
        ctx.set_timing(True); ctx.kernel_time(0)
        for _ in range(3):
            nwb.nw_score_only_dev(ctx, da, db, sc, d)
        ms, k = ctx.kernel_time(0)
        ctx.set_timing(False)
        out[f"kr{kr}_chains{2 if ch == 0 else 1}"] = {"ms": round(ms / k, 2), "TCUPS": round(1e12 / (ms / k) / 1e9, 3), "score": int(d.item())}
print(json.dumps(out, indent=1))
