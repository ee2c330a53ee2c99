"""Host-API (e2e) timing breakdown for one pair: nw_align_pair vs nw_traceback."""
import sys, time
sys.path.insert(0, '.')
import torch, nwgen
import paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
a, b = nwgen.config_c2()
for _ in range(3):
    s, tb = nwb.nw_align_pair(ctx, a, b, nwgen.PAPER_DNA); nwb.nw_traceback(ctx, tb); tb.free()
torch.cuda.synchronize()
ta = tt = 0.0
for _ in range(10):
    t0 = time.perf_counter()
    s, tb = nwb.nw_align_pair(ctx, a, b, nwgen.PAPER_DNA)
    t1 = time.perf_counter()
    ops = nwb.nw_traceback(ctx, tb)
    t2 = time.perf_counter()
    tb.free()
    ta += t1 - t0; tt += t2 - t1
print(f"align_pair {ta/10*1e3:.3f} ms, traceback {tt/10*1e3:.3f} ms")
