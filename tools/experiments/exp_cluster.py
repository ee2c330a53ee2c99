"""Single-pair fill with strips in thread-block clusters (NW_CLUSTER = CTAs per
cluster; the in-cluster hand-off through distributed shared memory) vs one strip
per warp through L2: fill / traceback ms, score and path equality."""
import os, sys
sys.path.insert(0, '.')
import torch, nwgen
import paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
shapes = [nwgen.config_c2(), nwgen.random_pair(3, 3001, 2999), nwgen.random_pair(5, 1000, 1000),
          nwgen.random_pair(6, 40000, 5000)]
for k, (a, b) in enumerate(shapes):
    da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
    db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
    ds = torch.zeros(1, dtype=torch.int64, device='cuda')
    ops = torch.zeros(len(a) + len(b), dtype=torch.uint8, device='cuda')
    ln = torch.zeros(1, dtype=torch.int64, device='cuda')
    os.environ.pop("NW_CLUSTER", None); os.environ.pop("NW_KR", None)
    rs, rtb = nwb.nw_align_pair(ctx, a, b, nwgen.PAPER_DNA)
    rops = nwb.nw_traceback(ctx, rtb).tobytes(); rtb.free()
    for kr in (sys.argv[1] if len(sys.argv) > 1 else "2,4,8").split(","):
        for cl in (sys.argv[2] if len(sys.argv) > 2 else "0,2,4,8").split(","):
            os.environ["NW_KR"] = kr; os.environ["NW_CLUSTER"] = cl
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
            ctx.set_timing(True); ctx.kernel_time(0)
            for _ in range(3): nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, ds)
            fs, nfs = ctx.kernel_time(0); ctx.set_timing(False)
            print(k, len(a), len(b), "kr", kr, "cluster", cl, "fill", round(f / nf, 4), "tb",
                  round(t / max(nt, 1), 4), "score-only", round(fs / nfs, 4), "score-only ok",
                  int(ds.item()) == rs, "ok", ok_s, ok_p, flush=True)
