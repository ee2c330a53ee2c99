mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x -k "difference_form or c5 or cblock or tall" > gpurun_out/pytest_x2.log 2>&1; tail -3 gpurun_out/pytest_x2.log
python tools/experiments/exp_c5x2.py > gpurun_out/exp_c5x2.json 2>&1; cat gpurun_out/exp_c5x2.json
