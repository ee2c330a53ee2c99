python tools/experiments/exp_fill.py c2 wide > gpurun_out/exp_tbe.json 2>&1
NW_EXP_NO_TBE=1 python tools/experiments/exp_fill.py c2 wide > gpurun_out/exp_notbe.json 2>&1
paste gpurun_out/exp_tbe.json gpurun_out/exp_notbe.json
