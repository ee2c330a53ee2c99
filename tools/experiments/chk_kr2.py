import os, sys, time
sys.path.insert(0, '.')
import torch, nwgen
import paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
for name, (a, b) in (("c5", nwgen.config_c5()), ("rnd7", nwgen.random_pair(7, 1000000, 1000000))):
    da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
    db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
    ds = torch.zeros(1, dtype=torch.int64, device='cuda')
    for kr in ("28", "14"):
        os.environ["NW_D16_KR"] = kr
        t0 = time.time()
        try:
            h = nwb.nw_score_only(ctx, a, b, nwgen.PAPER_DNA)
        except Exception as e:
            h = str(e)[:80]
        t1 = time.time()
        nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, ds)
        torch.cuda.synchronize()
        t2 = time.time()
        print(name, kr, "host", h, f"{t1-t0:.3f}s", "dev", int(ds.item()), f"{t2-t1:.3f}s", flush=True)
