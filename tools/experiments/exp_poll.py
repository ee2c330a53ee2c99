"""Single-pair fill: strip hand-off re-poll mode (NW_POLL_GAP: 0 = load-check-reload,
g > 0 = a new load every g cycles, 16 in flight) x rows per lane, on C2 (with
directions and score-only). Fill-kernel event time per call."""
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
gaps = sys.argv[1].split(",") if len(sys.argv) > 1 else ["0", "50", "100", "200"]
krs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["2", "4", "8"]


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


res = {}
for kr in krs:
    os.environ["NW_KR"] = kr
    for gap in gaps:
        os.environ["NW_POLL_GAP"] = gap
        d = timed(lambda: nwb.nw_align_pair_dev(ctx, da, db, nwgen.PAPER_DNA, ds).free())
        sc = int(ds.item())
        s = timed(lambda: nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, ds))
        res[f"kr{kr}_gap{gap}"] = {"dirs_ms": d, "score_ms": s, "score": sc, "score2": int(ds.item())}
        print(json.dumps({f"kr{kr}_gap{gap}": res[f"kr{kr}_gap{gap}"]}), flush=True)
