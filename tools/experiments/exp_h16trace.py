"""Timeline of the h16 C5 fill from per-strip timestamps (experiment build with
-DNW_TRACE: lane 0 of every strip records %globaltimer every 1024 groups).
NW_LIB_PATH=paper_2412_21103_b200/libnw_b200_trace.so python tools/experiments/exp_h16trace.py FORM KR"""
import ctypes, json, sys
sys.path.insert(0, '.')
import numpy as np
import torch
import nwgen
import paper_2412_21103_b200 as nwb

form, kr = int(sys.argv[1]), int(sys.argv[2])
ctx = nwb.Context(0, torch.cuda.current_stream().cuda_stream)
ctx.set_option("pair_form", form)
ctx.set_option("h16_kr", kr)
a, b = nwgen.config_c5()
da = torch.frombuffer(bytearray(a), dtype=torch.uint8).cuda()
db = torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()
ds = torch.zeros(1, dtype=torch.int64, device='cuda')
for _ in range(2):
    nwb.nw_score_only_dev(ctx, da, db, nwgen.PAPER_DNA, ds)
torch.cuda.synchronize()
S = (len(a) + 32 * kr - 1) // (32 * kr)
buf = np.zeros((S, 256), dtype=np.uint64)
L = nwb.lib()
L.nw_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
k = L.nw_debug_trace(buf.ctypes.data, S)
t = buf[:k].astype(np.float64)
t0 = t[0, 0]
ng = (len(b) + 63 + 7) // 8
nslot = min((ng + 255) // 256, 256)
t = (t[:, :nslot] - t0) / 1e3  # us
start = t[:, 0]
pace = (t[:, nslot - 1] - t[:, 1]) / ((nslot - 2) * 256 * 8) * 1e3  # ns per step
print(json.dumps({"form": form, "kr": kr, "strips": int(k),
                  "start_us": {"s1": float(start[1]), "s100": float(start[100]), "last": float(start[-1])},
                  "lag_steps_mean": float(np.mean(np.diff(start)) / np.median(pace) * 1e3),
                  "pace_ns_per_step": {"min": float(pace.min()), "median": float(np.median(pace)), "max": float(pace.max())},
                  "pace_cycles_median": float(np.median(pace) * 1.965),
                  "end_slot_us_last": float(t[-1, nslot - 1])}))
# per-strip pace over the middle slots: is any strip consistently slower?
mid = np.diff(t[:, 2:nslot - 2], axis=1) / (256 * 8) * 1e3
print("pace spread per slot (ns/step): median of per-slot max-min", float(np.median(mid.max(0) - mid.min(0))))
print("strip 0..7 pace", [round(float(x), 1) for x in pace[:8]])
