import os, sys
sys.path.insert(0, '.')
import torch, nwgen
import paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
a, b = nwgen.config_c2()
da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
ds = torch.zeros(1, dtype=torch.int64, device='cuda')
for kr in ("4", "2", "8"):
    os.environ["NW_KR"] = kr
    print("KR", kr, flush=True)
    nwb.nw_align_pair_dev(ctx, da, db, nwgen.PAPER_DNA, ds).free()
    torch.cuda.synchronize()
