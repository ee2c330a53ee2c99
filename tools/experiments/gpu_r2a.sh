# Round-2 first pass: all GPU tests (new: robustness, dist, full-size digests), smoke, bench C3 (default) and C2.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 2700 python -m pytest tests -m gpu -q --timeout 900 -k "not c5_score_fullsize and not c5_cblock_virtual" > gpurun_out/pytest_gpu.log 2>&1; tail -30 gpurun_out/pytest_gpu.log
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; head -c 3000 gpurun_out/bench_c3.json; tail -5 gpurun_out/bench_c3.err
timeout 600 python bench.py --workload c2 --steps 20 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; head -c 600 gpurun_out/bench_c2.json
