# Full ncu captures of the dominant kernels (split from gpu_round.sh: gpurun brings
# back at most 64 MiB per call). Usage: bash tools/experiments/gpu_prof_round.sh [c2|batch]
set -x
mkdir -p gpurun_out
if [ "$1" != batch ]; then
ncu --set full --clock-control none --import-source on -k regex:k_fill_pair -s 3 -c 1 -o gpurun_out/prof_c2_fill -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tb_spec -s 3 -c 1 -o gpurun_out/prof_c2_tbspec -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_c2spec.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tb_chain -s 3 -c 1 -o gpurun_out/prof_c2_tbchain -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_c2chain.log 2>&1
fi
if [ "$1" != c2 ]; then
ncu --set full --clock-control none --import-source on -k regex:k_batch -s 1 -c 2 -o gpurun_out/prof_c4_batch -f python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_batch -s 1 -c 1 -o gpurun_out/prof_c3_batch -f python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fill_pair -s 3 -c 1 -o gpurun_out/prof_c5_fill -f python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_c5.log 2>&1
fi
