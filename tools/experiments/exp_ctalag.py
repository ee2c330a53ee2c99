"""Lag of the shared-memory hand-off: fill time vs strips for plain and CTA-of-2 kernels (not a bench line)."""
import json, sys
sys.path.insert(0, '.')
import torch
import nwgen
import paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
ctx.set_option("rows_per_lane", 4)
n = 20000
out = {}
d = torch.zeros(1, dtype=torch.int64, device="cuda")
for w in (0, 2):
    ctx.set_option("fill_cta", w)
    for S in (1, 2, 4, 16, 64, 148, 157):
        a, b = nwgen.random_pair(5, 128 * S, n)
        da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda(); db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
        f = lambda: nwb.nw_align_pair_dev(ctx, da, db, nwgen.PAPER_DNA, d).free()
        f(); torch.cuda.synchronize(); ctx.set_timing(True); ctx.kernel_time(0)
        for _ in range(5): f()
        ms, k = ctx.kernel_time(0); ctx.set_timing(False)
        out[f"cta{w}_S{S}_ms"] = round(ms / k, 4)
    T1 = out[f"cta{w}_S1_ms"]
    c = T1 * 1e-3 * 1.965e9 / (n + 31)
    for S in (2, 4, 16, 64, 148, 157):
        out[f"cta{w}_S{S}_lag_steps"] = round((out[f"cta{w}_S{S}_ms"] - T1) * 1e-3 * 1.965e9 / c / (S - 1), 1)
    out[f"cta{w}_cycles_per_step"] = round(c, 1)
print(json.dumps(out, indent=1))
