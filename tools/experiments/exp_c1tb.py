"""C1 (1k x 1k + traceback): traceback kernel time vs the sampled-exit band (tb_band samples
per strip, tb_step column spacing); path checked against the default setting."""
import sys
sys.path.insert(0, '.')
import torch
import nwgen
import paper_2412_21103_b200 as nwb

ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
a, b = nwgen.config_c1()
ref = None
for band, step in [(0, 0), (32, 0), (64, 0), (32, 32), (32, 64), (64, 16), (128, 8)]:
    ctx.set_option("tb_band", band); ctx.set_option("tb_step", step)
    s, tb = nwb.nw_align_pair(ctx, a, b, nwgen.PAPER_DNA)
    ops = nwb.nw_traceback(ctx, tb).tolist(); tb.free()
    ref = ops if ref is None else ref
    torch.cuda.synchronize()
    ctx.set_timing(True); ctx.kernel_time(1)
    for _ in range(10):
        s, tb = nwb.nw_align_pair(ctx, a, b, nwgen.PAPER_DNA); nwb.nw_traceback(ctx, tb); tb.free()
    ms, k = ctx.kernel_time(1); ctx.set_timing(False)
    print(f"band {band} step {step}: traceback {ms / max(k,1) * 1e3:.1f} us, same path: {ops == ref}")
