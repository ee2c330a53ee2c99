mkdir -p gpurun_out
./tools/peaks_int > gpurun_out/peaks_int.json 2>&1 || (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks_int tools/peaks_int.cu && ./tools/peaks_int > gpurun_out/peaks_int.json)
NW_EXP_KR=2,4,8 NW_EXP_S=1,148 python tools/experiments/exp_lag.py > gpurun_out/exp_lag.json 2>&1; cat gpurun_out/exp_lag.json
ncu --set full --clock-control none --import-source on -k regex:k_fill_pair -s 3 -c 1 -o gpurun_out/prof_c2_fill_r2 -f python bench.py --workload c2 --steps 1 --warmup 3 --no-cpu --no-check > gpurun_out/ncu_c2.log 2>&1; tail -2 gpurun_out/ncu_c2.log
