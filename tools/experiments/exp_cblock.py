"""Column-block pipeline vs the plain single-pair fill on C5 (not a bench line).
Kernel event times (class 0) of: nw_score_only_dev (plain), the dist-ctx pipeline at
world 1 (NW_OPT_DIST_PIPELINE=1), and nw_score_only_cblock over G virtual ranks."""
import json, sys, time
sys.path.insert(0, '.')
import torch
import nwgen
import paper_2412_21103_b200 as nwb

a, b = nwgen.config_c5()
sc = nwgen.PAPER_DNA
cells = len(a) * len(b)
st = torch.cuda.current_stream().cuda_stream
da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
out = {}

def timed(ctx, fn, reps=3):
    fn(); torch.cuda.synchronize()
    ctx.set_timing(True); ctx.kernel_time(0)
    for _ in range(reps):
        fn()
    ms, k = ctx.kernel_time(0)
    ctx.set_timing(False)
    return ms / max(k, 1)

c = nwb.Context(0, st)
d = torch.zeros(1, dtype=torch.int64, device="cuda")
ms = timed(c, lambda: nwb.nw_score_only_dev(c, da, db, sc, d))
out["plain_ms"] = ms; out["plain_TCUPS"] = cells / ms / 1e9
c2 = nwb.Context(0, st)
c2.set_dist(0, 1, nwb.nw_dist_unique_id())
c2.set_option("dist_pipeline", 1)
ms = timed(c2, lambda: nwb.nw_score_only_dev(c2, da, db, sc, d))
out["dist_pipeline_world1_ms"] = ms; out["dist_pipeline_world1_TCUPS"] = cells / ms / 1e9
out["score_ok"] = int(d.item())
for G in [1, 2, 4, 8]:
    for w in ([0] if G == 1 else [0, 8192, 32768]):
        ms = timed(c, lambda: nwb.nw_score_only_cblock(c, a, b, sc, G, w), reps=2)
        out[f"virtual_G{G}_w{w}_ms"] = ms
        out[f"virtual_G{G}_w{w}_TCUPS"] = cells / ms / 1e9
print(json.dumps(out, indent=1))
if len(sys.argv) > 1: json.dump(out, open(sys.argv[1], "w"), indent=1)
