mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_h16.py -q -x --timeout 600 > gpurun_out/pytest_h16.log 2>&1; tail -3 gpurun_out/pytest_h16.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill_pair -s 1 -c 1 -o gpurun_out/prof_c5_h16 -f python tools/experiments/run_c5_once.py 0 28 > gpurun_out/ncu_h16.log 2>&1; tail -2 gpurun_out/ncu_h16.log
