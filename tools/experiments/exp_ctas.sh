# batch kernels: resident CTAs (4 warps each) per SM -> C3 / C4 step time
for c in 3 4 5 6 8; do
  for w in c4 c3; do
    echo "ctas=$c $w $(NW_BATCH_CTAS=$c python bench.py --workload $w --steps 3 --warmup 3 --no-cpu | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"],2), d["roofline"]["kernel_ms_per_launch"])')"
  done
done
