# Round-end style measurement pass: GPU tests, smoke, the default bench line
# (C2 + cpu_baseline), every other workload, the reference arm, the C2 launch
# list and full ncu captures of the dominant kernels (fill, traceback walks, batch).
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for w in c1 c3 c4 c5 c5tb msa c1p c1co c2co; do timeout 900 python bench.py --workload $w --steps 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
head -c 1500 gpurun_out/bench_c2.json
