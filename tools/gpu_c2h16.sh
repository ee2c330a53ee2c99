# packed H' fills (C2 with directions, C5 score-only): parity, then the bench lines
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_h16.py tests/test_gpu_robustness.py -q -x --timeout 120 > gpurun_out/pytest_c2h.log 2>&1; tail -1 gpurun_out/pytest_c2h.log
timeout 300 python -m pytest tests/test_gpu_fullsize.py -q -x --timeout 200 -k "c5_score" 2>&1 | tail -1
for w in c2 c5; do timeout 300 python bench.py --workload $w --steps 5 --no-cpu > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; python -c "
import json;d=json.load(open('gpurun_out/bench_$w.json'));print('$w', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms_per_launch'], d['check'])"; done
