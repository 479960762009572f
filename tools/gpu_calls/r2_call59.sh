# final HEAD: GPU suite, smoke, all bench lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2y_pytest.txt 2>&1; tail -1 gpurun_out/r2y_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2y_smoke.log 2>&1; tail -1 gpurun_out/r2y_smoke.log
timeout 400 python bench.py > gpurun_out/r2y_bench_c2.json 2> gpurun_out/r2y_bench_c2.err
for c in c1 c3 c4a c5; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2y_bench_$c.json 2> gpurun_out/r2y_bench_$c.err; done
timeout 900 python bench.py --config c4b --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2y_bench_c4b.json 2> gpurun_out/r2y_bench_c4b.err
timeout 400 python bench.py --deterministic --no-cpu-baseline --no-e2e > gpurun_out/r2y_bench_c2_det.json 2> gpurun_out/r2y_bench_c2_det.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2y_launches_bench_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for f in gpurun_out/r2y_bench_*.json; do echo "$f: $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline',{}); print(d.get('ms_per_step'), d.get('value'), r.get('frac'), (d.get('e2e') or {}).get('value'), d.get('clocks',{}).get('reasons'))" 2>&1 | tail -1)"; done
