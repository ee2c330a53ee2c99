"""One score-only pair fill (warm-up + one profiled launch) for ncu:
python tools/experiments/run_pair_once.py M N [h16_kr] [d16_force]"""
import sys
sys.path.insert(0, '.')
import torch
import nwgen
import paper_2412_21103_b200 as nwb

m, n = int(sys.argv[1]), int(sys.argv[2])
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
if len(sys.argv) > 3 and int(sys.argv[3]): ctx.set_option("h16_kr", int(sys.argv[3]))
if len(sys.argv) > 4 and int(sys.argv[4]): ctx.set_option("d16_force", int(sys.argv[4]))
a, b = nwgen.random_pair(5, m, n)
da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
ds = torch.zeros(1, dtype=torch.int64, device='cuda')
for _ in range(2):
    nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, ds)
torch.cuda.synchronize()
print("score", int(ds.item()))
