# Round-end style measurement pass: GPU tests, smoke, the default bench line
# (C2 + cpu_baseline), every other workload, the reference arm, the C2 launch
# list and full ncu captures of the dominant kernels (fill, traceback walks).
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for w in c1 c3 c4 c5 c5tb msa c1p; do timeout 900 python bench.py --workload $w --steps 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fill_pair -s 3 -c 1 -o gpurun_out/prof_c2_fill -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tb_spec -s 3 -c 1 -o gpurun_out/prof_c2_tbspec -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_c2spec.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tb_chain -s 3 -c 1 -o gpurun_out/prof_c2_tbchain -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_c2chain.log 2>&1
head -c 1500 gpurun_out/bench_c2.json
