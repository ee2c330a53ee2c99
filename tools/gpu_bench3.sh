mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; head -c 300 gpurun_out/bench_c3.json; echo
for w in c2 c5; do timeout 900 python bench.py --workload $w --steps 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; head -c 300 gpurun_out/bench_$w.json; echo; python -c "import json;d=json.load(open('gpurun_out/bench_$w.json'));print(d['roofline']['frac'], d.get('check'))"; done
