"""C5 (1M x 1M score-only, packed difference form): fill time vs rows per lane
(strip count relative to the 592 SM sub-partitions) and re-poll back-off."""
import json, os, sys
sys.path.insert(0, '.')
import torch
import nwgen
import paper_2412_21103_b200 as nwb

ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
a, b = nwgen.config_c5()
da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
ds = torch.zeros(1, dtype=torch.int64, device='cuda')
res = {}
ref = None
for kr in sys.argv[1].split(","):
    for pn in sys.argv[2].split(","):
        os.environ["NW_D16_KR"] = kr
        os.environ["NW_POLL_NS"] = pn
        nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, ds)
        torch.cuda.synchronize()
        ctx.set_timing(True)
        ctx.kernel_time(0)
        for _ in range(2):
            nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, ds)
        ms, k = ctx.kernel_time(0)
        ctx.set_timing(False)
        sc = int(ds.item())
        ref = sc if ref is None else ref
        res[f"kr{kr}_poll{pn}"] = {"ms": round(ms / k, 2), "tcups": round(1e12 / (ms / k * 1e-3) / 1e12, 3),
                                   "score_same": sc == ref}
        print(json.dumps({f"kr{kr}_poll{pn}": res[f"kr{kr}_poll{pn}"]}), flush=True)
print(json.dumps(res, indent=1))
