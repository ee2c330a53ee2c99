for lib in libnw_b200.so libnw_b200_mb4.so libnw_b200_mb5.so; do
  NW_LIB_PATH=paper_2412_21103_b200/$lib python tools/experiments/exp_ab.py c3 c4x 2>/dev/null
done
for lib in libnw_b200_mb4.so libnw_b200_mb5.so; do
  NW_LIB_PATH=paper_2412_21103_b200/$lib python bench.py --workload c4 --steps 5 --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$lib c4', d['value'], d['check'])"
done
python bench.py --workload c4 --steps 5 --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('base c4', d['value'], d['check'])"
