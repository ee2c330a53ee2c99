"""C2 fill with directions + strip traceback vs rows per lane (KR 4 = 157 strips,
5 = 125, 6 = 105, 8 = 79 on 148 SMs): fill and traceback event times, path equality."""
import os, sys
sys.path.insert(0, '.')
import torch, nwgen
import paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
a, b = nwgen.config_c2()
da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
ds = torch.zeros(1, dtype=torch.int64, device='cuda')
ops = torch.zeros(len(a) + len(b), dtype=torch.uint8, device='cuda')
ln = torch.zeros(1, dtype=torch.int64, device='cuda')
ref = None
for kr in ("4", "5", "6", "8", "4", "5", "6"):
    os.environ["NW_KR"] = kr
    def run():
        tb = nwb.nw_align_pair_dev(ctx, da, db, nwgen.PAPER_DNA, ds)
        nwb.nw_traceback_dev(ctx, tb, ops, ln)
        tb.free()
    run(); run(); torch.cuda.synchronize()
    ctx.set_timing(True); ctx.kernel_time(0); ctx.kernel_time(1)
    for _ in range(5): run()
    f, nf = ctx.kernel_time(0); t, nt = ctx.kernel_time(1); ctx.set_timing(False)
    L = int(ln.item()); path = ops[:L].cpu().numpy().tobytes()
    ref = path if ref is None else ref
    print(kr, "fill", round(f / nf, 4), "tb", round(t / max(nt, 1), 4), "same path", path == ref, flush=True)
