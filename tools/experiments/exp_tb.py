"""Traceback timing vs sampled-exit spacing (NW_TB_STEP), C2 pair."""
import os, sys, json
sys.path.insert(0, '.')
import torch
import nwgen
import paper_2412_21103_b200 as nwb
import numpy as np
case = os.environ.get("NW_EXP", "c2")
if case == "c2":
    a, b = nwgen.config_c2()
elif case.startswith("rand"):  # rand:M:N unrelated pair
    _, M, N = case.split(":")
    a, b = nwgen.random_pair(7, int(M), int(N))
else:  # indel: b = a with 10% point mutations and a 3000-residue insertion at 1/3
    rng = np.random.Generator(np.random.PCG64(11))
    a = nwgen.random_seq(rng, 20000)
    arr = np.frombuffer(a, dtype=np.uint8).copy()
    mut = rng.random(arr.size) < 0.1
    arr[mut] = np.frombuffer(b"ACGT", dtype=np.uint8)[rng.integers(0, 4, mut.sum())]
    b = arr[:6000].tobytes() + nwgen.random_seq(rng, 3000) + arr[6000:].tobytes()
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
ds = torch.zeros(1, dtype=torch.int64, device='cuda')
dops = torch.zeros(len(a) + len(b), dtype=torch.uint8, device='cuda')
dlen = torch.zeros(1, dtype=torch.int64, device='cuda')
tb = nwb.nw_align_pair_dev(ctx, da, db, nwgen.PAPER_DNA, ds)
os.environ["NW_TB_DEBUG"] = "1"
nwb.nw_traceback(ctx, tb)  # prints the slow-strip count
ctx.set_timing(True)
ctx.kernel_time(1)
for _ in range(5):
    nwb.nw_traceback_dev(ctx, tb, dops, dlen)
ms, k = ctx.kernel_time(1)
print(json.dumps({"case": case, "step": os.environ.get("NW_TB_STEP", "4"), "tb_ms": ms / k}))
