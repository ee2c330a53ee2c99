# Round-2 measurement pass: all GPU tests, smoke, every bench line (default C3 + cpu_baseline),
# the reference arm, per-kernel traffic, launch lists, ncu captures of the dominant kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; head -c 400 gpurun_out/bench_c3.json; echo
for w in c1 c2 c4 c5 c5tb msa c1p c1co c2co; do timeout 900 python bench.py --workload $w --steps 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w: $(head -c 200 gpurun_out/bench_$w.json)"; done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_c3.json 2> gpurun_out/bench_ref_c3.err; head -c 300 gpurun_out/bench_ref_c3.json; echo
for w in c2 c3 c4 c5; do timeout 900 python tools/traffic.py $w > /dev/null 2>&1; done; ls profiles/r02_traffic_* 
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-check > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu --no-check > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_batch -s 1 -c 1 -o gpurun_out/prof_c3_batch_r2b -f python bench.py --steps 1 --warmup 3 --no-cpu --no-check > gpurun_out/ncu_c3.log 2>&1; tail -1 gpurun_out/ncu_c3.log
