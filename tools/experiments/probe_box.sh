set -x
nvidia-smi; nvidia-smi topo -m; nproc; lscpu | head -20
python -c "import os;print('affinity',len(os.sched_getaffinity(0)))"
mkdir -p gpurun_out
./tools/peaks_int > gpurun_out/peaks_int.json; cat gpurun_out/peaks_int.json
