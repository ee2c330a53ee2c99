"""C2 traceback time vs the sampled-exit band (NW_TB_BAND samples per strip, NW_TB_STEP
columns between samples). Runs each setting in a fresh process (the
library reads both once)."""
import json, os, subprocess, sys
code = r'''
import sys; sys.path.insert(0, ".")
import torch, nwgen, paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
a, b = nwgen.config_c2()
da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda(); db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
ds = torch.zeros(1, dtype=torch.int64, device="cuda"); ops = torch.zeros(len(a)+len(b), dtype=torch.uint8, device="cuda"); ln = torch.zeros(1, dtype=torch.int64, device="cuda")
s0, tb0 = nwb.nw_align_pair(ctx, a, b, nwgen.PAPER_DNA); ref = nwb.nw_traceback(ctx, tb0).tobytes(); tb0.free()
def run():
    tb = nwb.nw_align_pair_dev(ctx, da, db, nwgen.PAPER_DNA, ds); nwb.nw_traceback_dev(ctx, tb, ops, ln); tb.free()
run(); run(); torch.cuda.synchronize(); ctx.set_timing(True); ctx.kernel_time(1)
for _ in range(10): run()
t, n = ctx.kernel_time(1)
print(round(t / n, 4), ops[:int(ln.item())].cpu().numpy().tobytes() == ref)
'''
res = {}
for band in ("64", "128", "256"):
    for step in ("2", "4", "8"):
        env = dict(os.environ, NW_TB_BAND=band, NW_TB_STEP=step)
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True).stdout.split()
        res[f"band{band}_step{step}"] = out
        print(band, step, out, flush=True)
print(json.dumps(res))
