# ncu captures of the batch / score-only kernels (one launch each).
set -x
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_batch -s 1 -c 1 -o gpurun_out/prof_c3_batch -f python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_batch -s 1 -c 1 -o gpurun_out/prof_c4_batch -f python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fill_pair -s 3 -c 1 -o gpurun_out/prof_c2_fill_v4 -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_c2.log 2>&1
tail -2 gpurun_out/ncu_c3.log gpurun_out/ncu_c4.log gpurun_out/ncu_c2.log
