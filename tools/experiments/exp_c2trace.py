"""Timeline of the C2 fill (int32 strips with directions) from per-strip timestamps
(experiment build with -DNW_TRACE: lane 0 of every strip stamps %globaltimer every 256
groups = 2,048 columns). Prints each strip's start and pace, and the SM it ran on is not
known here: look for slow strips and where the chain's pace changes.
NW_LIB_PATH=paper_2412_21103_b200/libnw_b200_trace.so python tools/experiments/exp_c2trace.py [kr]"""
import ctypes, json, sys
sys.path.insert(0, '.')
import numpy as np
import torch
import nwgen
import paper_2412_21103_b200 as nwb

ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
kr = int(sys.argv[1]) if len(sys.argv) > 1 else 0
if kr: ctx.set_option("rows_per_lane", kr)
import os
ctx.set_option("pair_form", int(os.environ.get("PAIR_FORM", "0")))
a, b = nwgen.config_c2()
da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
ds = torch.zeros(1, dtype=torch.int64, device='cuda')
for _ in range(3):
    nwb.nw_align_pair_dev(ctx, da, db, nwgen.PAPER_DNA, ds).free()
torch.cuda.synchronize()
S = 400
buf = np.zeros((S, 256), dtype=np.uint64)
L = nwb.lib()
L.nw_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
k = L.nw_debug_trace(buf.ctypes.data, S)
n = len(b)
ng = (n + 31 + 7) // 8
nslot = (ng + 255) // 256
t = buf[:k, :nslot].astype(np.float64)
t = (t - t[0, 0]) / 1e3  # us
start = t[:, 0]
pace = (t[:, nslot - 1] - t[:, 0]) / ((nslot - 1) * 256 * 8) * 1e3  # ns per step
lag = np.diff(start)
print(json.dumps({"strips": int(k), "last_start_us": float(start[-1]),
                  "lag_us": {"median": float(np.median(lag)), "min": float(lag.min()), "max": float(lag.max())},
                  "pace_ns": {"median": float(np.median(pace)), "min": float(pace.min()), "max": float(pace.max())},
                  "pace_cycles_median": float(np.median(pace) * 1.965),
                  "lag_steps_median": float(np.median(lag) / np.median(pace) * 1e3)}))
print("pace by strip (ns/step), every 8th:", [round(float(x), 1) for x in pace[::8]])
print("pace of strips 140..156:", [round(float(x), 1) for x in pace[140:]])
print("lag of strips 1..12 (us):", [round(float(x), 2) for x in lag[:12]])
