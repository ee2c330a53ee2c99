"""C3 batch fill with 8/16/32 rows per lane in the packed H' sweep, or mixed 32/16 per
pair at several weights (not a bench line). usage: exp_u16kr.py [kr:w,...] [out.json]"""
import json, sys
sys.path.insert(0, '.')
import torch, numpy as np
import nwgen, oracle
import paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
ss = nwgen.config_c3()
ds = torch.from_numpy(ss.residues).cuda(); do = torch.from_numpy(ss.offs).cuda()
P = ss.nseq * (ss.nseq - 1) // 2
out = {}
rng = np.random.Generator(np.random.PCG64(1)); idx = np.sort(rng.choice(P, 64, replace=False))
allp = nwgen.all_pairs(ss.nseq)
want = oracle.batch_score(ss.residues, ss.offs, allp[idx], nwgen.PAPER_DNA)
cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["16:0", "32:0", "8:0"]
for cfg in cfgs:
    kr, w, *w24 = (int(x) for x in cfg.split(":"))
    ctx.set_option("batch_u16_kr", kr)
    ctx.set_option("batch_mix_w", w)
    ctx.set_option("batch_mix_w24", w24[0] if w24 else 0)
    sc = torch.zeros(P, dtype=torch.int32, device="cuda")
    f = lambda: nwb.nw_align_batch_dev(ctx, ds, do, ss.offs, None, None, P, nwgen.PAPER_DNA, 0, sc)
    f(); torch.cuda.synchronize(); ctx.set_timing(True); ctx.kernel_time(0)
    for _ in range(3): f()
    ms, k = ctx.kernel_time(0); ctx.set_timing(False)
    out[f"kr{kr}_w{w}" + (f"_w24{w24[0]}" if w24 else "")] = {"ms": round(ms / k, 2), "TCUPS": round(3216418768982 / (ms / k) / 1e9, 3),
                      "sample_ok": bool((sc.cpu().numpy()[idx] == want).all())}
print(json.dumps(out, indent=1))
if len(sys.argv) > 2: json.dump(out, open(sys.argv[2], "w"), indent=1)
