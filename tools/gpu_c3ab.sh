# C3 A/B: parity of the batch sweeps, the full-size C3 digest, then the bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "c3 or batch" --timeout 600 > gpurun_out/pytest_c3.log 2>&1; tail -2 gpurun_out/pytest_c3.log
python bench.py --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; python -c "
import json;d=json.load(open('gpurun_out/bench_c3.json'));print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['check'])"
