"""Runs the C5 score-only fill twice (warm-up + one profiled launch) for ncu:
python tools/experiments/run_c5_once.py [pair_form] [h16_kr]"""
import sys
sys.path.insert(0, '.')
import torch
import nwgen
import paper_2412_21103_b200 as nwb

ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
if len(sys.argv) > 1: ctx.set_option("pair_form", int(sys.argv[1]))
if len(sys.argv) > 2: ctx.set_option("h16_kr", int(sys.argv[2]))
a, b = nwgen.config_c5()
da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
ds = torch.zeros(1, dtype=torch.int64, device='cuda')
for _ in range(2):
    nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, ds)
torch.cuda.synchronize()
print("score", int(ds.item()))
