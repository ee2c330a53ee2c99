set -x
ncu --set full --clock-control none --import-source on -k regex:k_batch -s 1 -c 1 -o gpurun_out/prof_c4_packed -f python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fill_pair -s 3 -c 1 -o gpurun_out/prof_c5_fill -f python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_c5.log 2>&1
tail -1 gpurun_out/ncu_c4.log gpurun_out/ncu_c5.log
