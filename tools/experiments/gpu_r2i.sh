mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q --timeout 600 -x -k "batch or c3 or partition or world1" > gpurun_out/pytest_c3.log 2>&1; tail -3 gpurun_out/pytest_c3.log
for i in 1 2; do python bench.py --steps 5 --no-cpu > gpurun_out/bench_c3_$i.json 2>gpurun_out/bench_c3.err; python -c "import json;d=json.load(open('gpurun_out/bench_c3_$i.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['check'])"; done
