"""C2 fill, one vs two columns per lane and step (NW_CPS), KR 4 and 8: fill event
time (score-only and with directions) and H(m, n) agreement."""
import os, sys
sys.path.insert(0, '.')
import torch, nwgen
import paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
shapes = [nwgen.config_c2(), nwgen.random_pair(3, 3001, 2999), nwgen.random_pair(4, 700, 5000)]
for k, (a, b) in enumerate(shapes):
    da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
    db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
    ds = torch.zeros(1, dtype=torch.int64, device='cuda')
    os.environ.pop("NW_CPS", None); os.environ.pop("NW_KR", None)
    ref = nwb.nw_score_only(ctx, a, b, nwgen.PAPER_DNA)
    for kr in ("4", "8"):
        for cps in ("1", "2"):
            os.environ["NW_KR"] = kr; os.environ["NW_CPS"] = cps
            out = {}
            for mode in ("score", "dirs"):
                def run():
                    if mode == "score": nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, ds)
                    else: nwb.nw_align_pair_dev(ctx, da, db, nwgen.PAPER_DNA, ds).free()
                run(); run(); torch.cuda.synchronize()
                ctx.set_timing(True); ctx.kernel_time(0)
                for _ in range(5): run()
                ms, n = ctx.kernel_time(0); ctx.set_timing(False)
                out[mode] = (round(ms / n, 4), int(ds.item()) == ref)
            print(k, len(a), len(b), "kr", kr, "cps", cps, out, flush=True)
