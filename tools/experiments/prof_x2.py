"""One C5-shaped launch (KR 28, 1117 strips, n = 200k) with one or two chains per lane, for ncu."""
import sys
sys.path.insert(0, '.')
import torch
import nwgen
import paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
ctx.set_option("d16_force", 28)
ctx.set_option("d16_chains", int(sys.argv[1]))
a, b = nwgen.random_pair(9, 896 * 1117, 200_000)
da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda(); db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
d = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(2):
    nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, d)
torch.cuda.synchronize()
print(int(d.item()))
