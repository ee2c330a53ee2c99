"""Quick fill-kernel timing experiments on the GPU box (not a bench line):
fill-kernel event time per (shape, mode, KR)."""
import json, os, sys
sys.path.insert(0, '.')
import torch
import nwgen
import paper_2412_21103_b200 as nwb

ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
shapes = {"c2": (20000, 20000), "c1": (1000, 1000), "tall": (80000, 2000), "wide": (2000, 80000)}
if len(sys.argv) > 1:
    shapes = {k: v for k, v in shapes.items() if k in sys.argv[1:]}
res = {}
for name, (m, n) in shapes.items():
    a, b = nwgen.random_pair(5, m, n)
    da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
    db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
    ds = torch.zeros(1, dtype=torch.int64, device='cuda')
    for kr in ("2", "4", "8"):
        os.environ["NW_KR"] = kr
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
            res[f"{name}_{mode}_kr{kr}"] = round(ms / k, 3)
    os.environ.pop("NW_KR")
print(json.dumps(res, indent=1))
