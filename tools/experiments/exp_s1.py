"""One single-strip fill (m = 128, n = 20000, KR = 4, directions) for ncu A/B runs."""
import os, sys
sys.path.insert(0, '.')
os.environ.setdefault("NW_KR", "4")
import torch, nwgen
import paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
m = int(os.environ.get("NW_EXP_M", "128"))
a, b = nwgen.random_pair(5, m, 20000)
da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
ds = torch.zeros(1, dtype=torch.int64, device='cuda')
for _ in range(2):
    nwb.nw_align_pair_dev(ctx, da, db, nwgen.PAPER_DNA, ds).free()
torch.cuda.synchronize()
