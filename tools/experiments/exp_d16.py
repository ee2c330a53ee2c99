"""Fill-kernel event time on C2-shaped pairs: score-only int32 strips (KR 2/4/8)
vs the packed difference form (KR 4/8/16, nw_fill_d16.cuh), and the int32
direction fill. Decides whether the packed form pays for a single 20k pair."""
import json, os, sys
sys.path.insert(0, '.')
import torch
import nwgen
import paper_2412_21103_b200 as nwb

ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
a, b = nwgen.config_c2()
da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
ds = torch.zeros(1, dtype=torch.int64, device='cuda')
res = {}
ref = None


def timed(run, k=5):
    run(); run()
    torch.cuda.synchronize()
    ctx.set_timing(True)
    ctx.kernel_time(0)
    for _ in range(k):
        run()
    ms, n = ctx.kernel_time(0)
    ctx.set_timing(False)
    return round(ms / n, 4)


for kr in ("2", "4", "8"):
    os.environ["NW_KR"] = kr
    res[f"score_int32_kr{kr}"] = timed(lambda: nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, ds))
    ref = int(ds.item())
    res[f"dirs_int32_kr{kr}"] = timed(lambda: nwb.nw_align_pair_dev(ctx, da, db, nwgen.PAPER_DNA, ds).free())
os.environ.pop("NW_KR")
for kr in ("4", "8", "16", "32"):
    os.environ["NW_D16_FORCE"] = kr
    res[f"score_d16_kr{kr}"] = timed(lambda: nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, ds))
    res[f"score_d16_kr{kr}_ok"] = int(ds.item()) == ref
os.environ.pop("NW_D16_FORCE")
print(json.dumps(res, indent=1))
