for i in 1 2; do
NW_LIB_PATH=paper_2412_21103_b200/libnw_b200_r1.so python bench.py --workload c1 --steps 20 --no-cpu --no-check 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('r1',d['ms_per_step'],d['roofline']['kernel_ms_per_launch'],d['roofline']['traceback_ms_per_step'],d['gpu_launches'])"
python bench.py --workload c1 --steps 20 --no-cpu --no-check 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('r2',d['ms_per_step'],d['roofline']['kernel_ms_per_launch'],d['roofline']['traceback_ms_per_step'],d['gpu_launches'])"
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python bench.py --workload c1 --steps 2 --warmup 3 --no-cpu --no-check > /dev/null 2>&1
NW_LIB_PATH=paper_2412_21103_b200/libnw_b200_r1.so ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1_r1.csv python bench.py --workload c1 --steps 2 --warmup 3 --no-cpu --no-check > /dev/null 2>&1
