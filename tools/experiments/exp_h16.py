"""C5 (1M x 1M score-only): fill-kernel time of the packed H' sweep with a moving base
(nw_fill_h16.cuh) at several rows per lane / rebase periods (EXP_FORMS: pair_form values), against the difference
form (pair_form 1). Scores must equal the committed oracle digest.
usage: python tools/experiments/exp_h16.py KR,KR,... REB,REB,... [out.json]"""
import json, os, sys
sys.path.insert(0, '.')
import torch
import nwgen
import paper_2412_21103_b200 as nwb

dig = json.load(open('tests/golden/digests.json'))['c5']['score']
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
a, b = nwgen.config_c5()
da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
ds = torch.zeros(1, dtype=torch.int64, device='cuda')
res = {}


def run(name):
    nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, ds)
    torch.cuda.synchronize()
    ctx.set_timing(True)
    ctx.kernel_time(0)
    for _ in range(3):
        nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, ds)
    ms, k = ctx.kernel_time(0)
    ctx.set_timing(False)
    sc = int(ds.item())
    res[name] = {"ms": round(ms / k, 2), "tcups": round(1e12 / (ms / k * 1e-3) / 1e12, 3), "score_ok": sc == dig}
    print(json.dumps({name: res[name]}), flush=True)


ctx.set_option("pair_form", 1)
run("d16_default")
for form in os.environ.get("EXP_FORMS", "0").split(","):
    ctx.set_option("pair_form", int(form))
    for kr in sys.argv[1].split(","):
        for reb in sys.argv[2].split(","):
            ctx.set_option("h16_kr", int(kr))
            ctx.set_option("h16_rebase", int(reb))
            run(f"h16_form{form}_kr{kr}_reb{reb}")
ctx.set_option("pair_form", 0)
ctx.set_option("h16_kr", 0)
ctx.set_option("h16_rebase", 0)
run("h16_default")
if len(sys.argv) > 3:
    json.dump({"what": __doc__.split("\n")[0], "results": res}, open(sys.argv[3], "w"), indent=1)
