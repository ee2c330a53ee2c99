mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
for w in c1 c2 c4 c5 c5tb msa c1p c1co c2co; do timeout 900 python bench.py --workload $w --steps 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
for w in c3 c1 c2 c4 c5 c5tb msa c1p c1co c2co; do python -c "
import json;d=json.load(open('gpurun_out/bench_$w.json'));r=d['roofline'];print('$w', round(d['value'],2), round(d['ms_per_step'],3), round(r['frac'] or 0,3), round(d['e2e']['value'],2), d.get('check',{}).get('mismatches'), d.get('cpu_baseline',{}).get('value'), d['clocks'].get('sm_mhz'))"; done
