"""C2 score-only fill vs rows per lane, including strip counts <= 148 (one warp
per SM): KR 4 = 157 strips, 5 = 125, 6 = 105, 8 = 79."""
import json, os, sys
sys.path.insert(0, '.')
import torch, nwgen
import paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
a, b = nwgen.config_c2()
da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
ds = torch.zeros(1, dtype=torch.int64, device='cuda')
res = {}
for kr in ("4", "5", "6", "8", "4", "5"):
    os.environ["NW_KR"] = kr
    run = lambda: nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, ds)
    run(); run(); torch.cuda.synchronize()
    ctx.set_timing(True); ctx.kernel_time(0)
    for _ in range(5): run()
    ms, k = ctx.kernel_time(0); ctx.set_timing(False)
    res[f"kr{kr}"] = (round(ms / k, 4), int(ds.item()))
    print(kr, res[f"kr{kr}"], flush=True)
