# final round-2 bench lines at HEAD (fill kernels): C2 (with cpu_baseline and e2e), C3, C5, deterministic, launch list
mkdir -p gpurun_out
timeout 400 python bench.py > gpurun_out/r2h_bench_c2.json 2> gpurun_out/r2h_bench_c2.err
for c in c1 c3 c4a c5; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2h_bench_$c.json 2> gpurun_out/r2h_bench_$c.err; done
timeout 400 python bench.py --deterministic --no-cpu-baseline --no-e2e > gpurun_out/r2h_bench_c2_det.json 2> gpurun_out/r2h_bench_c2_det.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2h_launches_bench_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for f in gpurun_out/r2h_bench_*.json; do echo "$f: $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline',{}); print(d.get('ms_per_step'), d.get('value'), r.get('frac'), (d.get('e2e') or {}).get('value'), d.get('clocks',{}).get('reasons'))" 2>&1 | tail -1)"; done
