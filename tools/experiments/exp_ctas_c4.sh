# C4 batch kernel (56 registers since the in-warp walk left it): CTAs of 4 warps per SM
for c in 6 8 10; do
  echo "ctas=$c c4 $(NW_BATCH_CTAS=$c python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"],3), d["roofline"]["kernel_ms_per_launch"])')"
done
