# C2 path A/B: single-pair parity (int32 strips, traceback), checkpointed traceback, robustness; C2/C1 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_linear.py tests/test_gpu_robustness.py tests/test_gpu_cooptimal.py tests/test_gpu_percell.py -q -x --timeout 200 > gpurun_out/pytest_c2.log 2>&1; tail -1 gpurun_out/pytest_c2.log
for w in c2 c1 c5tb; do timeout 300 python bench.py --workload $w --steps 5 --no-cpu > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; python -c "
import json;d=json.load(open('gpurun_out/bench_$w.json'));print('$w', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms_per_launch'], d.get('check'))"; done
