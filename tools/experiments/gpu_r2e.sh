mkdir -p gpurun_out
python tools/experiments/exp_cblock.py > gpurun_out/exp_cblock.json 2>&1; cat gpurun_out/exp_cblock.json
