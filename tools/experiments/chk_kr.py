"""Check the packed score-only fill at every rows-per-lane setting against the
int32 strip fill (scores must agree; errors are reported by the host ABI)."""
import os, sys
sys.path.insert(0, '.')
import torch, nwgen
import paper_2412_21103_b200 as nwb
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
shapes = [(448 * 3 + 17, 1000), (100000, 3000), (300000, 20000), (1000000, 4000)]
if len(sys.argv) > 1:
    shapes = [tuple(int(x) for x in s.split("x")) for s in sys.argv[1].split(",")]
krs = (12, 14, 16, 18, 20, 28) if len(sys.argv) <= 2 else tuple(int(k) for k in sys.argv[2].split(","))
for (m, n) in shapes:
    a, b = nwgen.random_pair(7, m, n)
    os.environ["NW_D16_FORCE"] = "28"
    ref = nwb.nw_score_only(ctx, a, b, nwgen.PAPER_DNA)
    out = {}
    for kr in krs:
        os.environ["NW_D16_FORCE"] = str(kr)
        try:
            out[kr] = nwb.nw_score_only(ctx, a, b, nwgen.PAPER_DNA) - ref
        except Exception as e:
            out[kr] = str(e)[:80]
    print(m, n, ref, out, flush=True)
