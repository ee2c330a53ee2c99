mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_parity.py -q --timeout 600 -x -k "cblock or pipeline or c5 or two_process or world1" > gpurun_out/pytest_cb.log 2>&1; tail -25 gpurun_out/pytest_cb.log
