mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_fill_pair -s 1 -c 1 -o gpurun_out/prof_c5_fill_r2 -f python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu --no-check > gpurun_out/ncu_c5.log 2>&1; tail -1 gpurun_out/ncu_c5.log
ncu --set full --clock-control none --import-source on -k regex:k_batch -s 1 -c 1 -o gpurun_out/prof_c3_batch_r2 -f python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu --no-check > gpurun_out/ncu_c3.log 2>&1; tail -1 gpurun_out/ncu_c3.log
