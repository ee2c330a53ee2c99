"""One C2 fill with the plain (fill_cta 0) or CTA shared-memory hand-off (2) kernel, for ncu."""
import sys
sys.path.insert(0, '.')
import torch
import nwgen
import paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
ctx.set_option("fill_cta", int(sys.argv[1]))
a, b = nwgen.config_c2()
da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda(); db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
d = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(2):
    nwb.nw_align_pair_dev(ctx, da, db, nwgen.PAPER_DNA, d).free()
torch.cuda.synchronize()
