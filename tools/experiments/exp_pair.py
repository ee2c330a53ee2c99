"""Single-pair fill, one strip per warp vs strip pairs (NW_PAIR, nw_fillpair.cuh),
KR 2 and 4: fill and traceback event times, score and path equality with the oracle
path of the one-strip sweep."""
import os, sys
sys.path.insert(0, '.')
import torch, nwgen
import paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
shapes = [nwgen.config_c2(), nwgen.random_pair(3, 3001, 2999), nwgen.random_pair(4, 700, 5000),
          nwgen.random_pair(5, 1000, 1000)]
for k, (a, b) in enumerate(shapes):
    da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
    db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
    ds = torch.zeros(1, dtype=torch.int64, device='cuda')
    ops = torch.zeros(len(a) + len(b), dtype=torch.uint8, device='cuda')
    ln = torch.zeros(1, dtype=torch.int64, device='cuda')
    os.environ.pop("NW_PAIR", None); os.environ.pop("NW_KR", None)
    rs, rtb = nwb.nw_align_pair(ctx, a, b, nwgen.PAPER_DNA)
    rops = nwb.nw_traceback(ctx, rtb).tobytes(); rtb.free()
    for kr in ("2", "4"):
        for pair in ("0", "1"):
            os.environ["NW_KR"] = kr
            if pair == "1": os.environ["NW_PAIR"] = "1"
            else: os.environ.pop("NW_PAIR", None)
            def run():
                tb = nwb.nw_align_pair_dev(ctx, da, db, nwgen.PAPER_DNA, ds)
                nwb.nw_traceback_dev(ctx, tb, ops, ln)
                tb.free()
            run(); run(); torch.cuda.synchronize()
            ctx.set_timing(True); ctx.kernel_time(0); ctx.kernel_time(1)
            for _ in range(5): run()
            f, nf = ctx.kernel_time(0); t, nt = ctx.kernel_time(1); ctx.set_timing(False)
            ok_s = int(ds.item()) == rs
            ok_p = ops[:int(ln.item())].cpu().numpy().tobytes() == rops
            s_only = nwb.nw_score_only(ctx, a, b, nwgen.PAPER_DNA) == rs
            ctx.set_timing(True); ctx.kernel_time(0)
            for _ in range(3): nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, ds)
            fs, nfs = ctx.kernel_time(0); ctx.set_timing(False)
            print(k, len(a), len(b), "kr", kr, "pair", pair, "fill", round(f / nf, 4), "tb",
                  round(t / max(nt, 1), 4), "score-only fill", round(fs / nfs, 4),
                  "ok", ok_s, ok_p, s_only, flush=True)
