"""Per-step cost and strip-to-strip lag of the tall-pair score-only sweeps at 28 rows
per lane: T(S) for m = 896 S, n = N; T(1) / (n + 63) is the lone strip's step, the slope
over S the lag. Packed H' (h16) vs difference form (d16). Not a bench line."""
import json, os, sys
sys.path.insert(0, '.')
import torch
import nwgen
import paper_2412_21103_b200 as nwb

ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
res = {}
for form in os.environ.get("EXP_FORMS", "h16,d16").split(","):
    if form.startswith("h16"):
        ctx.set_option("d16_force", 0); ctx.set_option("h16_kr", 28)
        ctx.set_option("pair_form", 2 if form == "h16c" else 0)
    else:
        ctx.set_option("h16_kr", 0); ctx.set_option("d16_force", 28)
    for S in [int(x) for x in os.environ.get("EXP_S", "1,2,8,74,148,296,592,888,1117,1184").split(",")]:
        m = 896 * S
        a, b = nwgen.random_pair(5, m, n)
        da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
        db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
        ds = torch.zeros(1, dtype=torch.int64, device='cuda')
        nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, ds)
        torch.cuda.synchronize()
        ctx.set_timing(True)
        ctx.kernel_time(0)
        for _ in range(3):
            nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, ds)
        ms, k = ctx.kernel_time(0)
        ctx.set_timing(False)
        t = ms / k
        cyc_per_step = t * 1e-3 * 1.965e9 / (n + 63)
        res[f"{form}_S{S}"] = {"ms": round(t, 3), "cycles_per_column": round(cyc_per_step, 1),
                               "tcups": round(m * n / (t * 1e-3) / 1e12, 3)}
        print(json.dumps({f"{form}_S{S}": res[f"{form}_S{S}"]}), flush=True)
if len(sys.argv) > 2:
    json.dump({"what": __doc__.split("\n")[0], "n": n, "results": res}, open(sys.argv[2], "w"), indent=1)
