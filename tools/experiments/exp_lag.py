"""Per-step cost and inter-strip lag of the single-pair fill (not a bench line).
For n = 20000 and m = R*S, fill time T(S) ~ c_step * (n + 31 + lag * (S - 1)):
T(1) gives c_step, the slope in S gives c_step * lag."""
import json, os, sys
sys.path.insert(0, '.')
import torch
import nwgen
import paper_2412_21103_b200 as nwb

ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
n = 20000
res = {}
krs = [int(k) for k in os.environ.get("NW_EXP_KR", "2,4,8").split(",")]
for kr in krs:
    ctx.set_option("rows_per_lane", kr)
    R = 32 * kr
    for S in [int(x) for x in os.environ.get("NW_EXP_S", "1,2,4,16,64,148").split(",")]:
        m = R * S
        a, b = nwgen.random_pair(5, m, n)
        da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
        db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
        ds = torch.zeros(1, dtype=torch.int64, device='cuda')
        for mode in ("score", "dirs"):
            def run():
                if mode == "score":
                    nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, ds)
                else:
                    nwb.nw_align_pair_dev(ctx, da, db, nwgen.PAPER_DNA, ds).free()
            run(); run()
            torch.cuda.synchronize()
            ctx.set_timing(True)
            ctx.kernel_time(0)
            for _ in range(3):
                run()
            ms, k = ctx.kernel_time(0)
            ctx.set_timing(False)
            res[f"kr{kr}_{mode}_S{S}"] = round(ms / k, 4)
    T1 = res[f"kr{kr}_dirs_S1"]; T148 = res[f"kr{kr}_dirs_S148"]
    c = T1 * 1e-3 * 1.965e9 / (n + 31)
    lag = (T148 - T1) * 1e-3 * 1.965e9 / c / 147
    res[f"kr{kr}_dirs_cycles_per_step"] = round(c, 1)
    res[f"kr{kr}_dirs_lag_steps"] = round(lag, 1)
print(json.dumps(res, indent=1))
