# C4 path: batch traceback parity (all tie orders, waves, orientation), full-size C4 digest, MSA; C4 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_msa.py tests/test_gpu_dist.py -q -x --timeout 300 -k "batch or c4 or msa or dist" > gpurun_out/pytest_c4.log 2>&1; tail -n 1 gpurun_out/pytest_c4.log
for w in c4 msa; do timeout 300 python bench.py --workload $w --steps 5 --no-cpu > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; python -c "
import json;d=json.load(open('gpurun_out/bench_$w.json'));print('$w', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms_per_launch'], d.get('check'))"; done
