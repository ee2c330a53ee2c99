# One measurement pass on the GPU box: bench lines, launch list, ncu capture.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for w in c1 c5 c3 c4; do timeout 300 python bench.py --workload $w --no-cpu --steps 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fill_pair -s 3 -c 1 -o gpurun_out/prof_c2_fill -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tb_walk -s 3 -c 1 -o gpurun_out/prof_c2_tb -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_c2tb.log 2>&1
cat gpurun_out/bench_*.json
