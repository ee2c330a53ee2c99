# Round-2 final measurement pass, part 1: tests, bench lines, traffic, launch lists (ncu --set full captures run as separate calls: each report is ~30 MB and gpurun_out/ must stay under 64 MiB)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; tail -n 2 gpurun_out/pytest_gpu.log
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
for w in c1 c2 c4 c5 c5tb msa c1p c1co c2co; do timeout 900 python bench.py --workload $w --steps 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_c3.json 2> gpurun_out/bench_ref_c3.err
for w in c3 c1 c2 c4 c5 c5tb msa c1p c1co c2co; do python -c "
import json;d=json.load(open('gpurun_out/bench_$w.json'));r=d['roofline'];print('$w', round(d['value'],2), round(d['ms_per_step'],3), round(r['frac'] or 0,3), round(d['e2e']['value'],2), d.get('check',{}).get('mismatches'), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; done
for w in c2 c3 c4 c5 msa; do timeout 900 python tools/traffic.py $w > /dev/null 2>&1; done
for w in c1 c2 c3 c4 c5; do ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv python bench.py --workload $w --steps 2 --warmup 3 --no-cpu --no-check > /dev/null 2>&1; done

