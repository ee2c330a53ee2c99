"""Pace of the packed difference-form fill vs strips per SM sub-partition (not a bench line).
KR 28 (896 rows per strip), n = 200,000 columns, S strips: ms and cycles per step."""
import json, sys
sys.path.insert(0, '.')
import torch
import nwgen
import paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
ctx.set_option("d16_force", 28)
if len(sys.argv) > 1: ctx.set_option("d16_chains", int(sys.argv[1]))
n = 200_000
out = {}
d = torch.zeros(1, dtype=torch.int64, device="cuda")
for S in [1, 148, 592, 1117]:
    m = 896 * S
    a, b = nwgen.random_pair(9, m, n)
    da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda(); db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
    nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, d); torch.cuda.synchronize()
    ctx.set_timing(True); ctx.kernel_time(0)
    for _ in range(3): nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, d)
    ms, k = ctx.kernel_time(0); ctx.set_timing(False)
    ms /= k
    out[f"S{S}"] = {"ms": round(ms, 3), "cycles_per_column": round(ms * 1e-3 * 1.965e9 / n, 1), "TCUPS": round(m * n / ms / 1e9, 3)}
print(json.dumps(out, indent=1))
