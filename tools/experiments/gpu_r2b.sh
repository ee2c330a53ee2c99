# prefix-form C2 fill: parity suite + bench C2 + launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -k "not c5_score_fullsize and not c5_cblock_virtual" > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for i in 1 2; do timeout 600 python bench.py --workload c2 --steps 20 --no-cpu > gpurun_out/bench_c2_$i.json 2> gpurun_out/bench_c2.err; head -c 400 gpurun_out/bench_c2_$i.json; echo; done
python -c "import json;d=json.load(open('gpurun_out/bench_c2_1.json'));print(d['roofline']['kernel_ms_per_launch'], d['check'])"
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu --no-check > /dev/null 2>&1
grep k_fill gpurun_out/launches_c2.csv | head -8
