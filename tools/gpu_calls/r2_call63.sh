# final HEAD: full GPU suite + smoke + C2 bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2x_pytest.txt 2>&1; tail -1 gpurun_out/r2x_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2x_smoke.log 2>&1; tail -1 gpurun_out/r2x_smoke.log
timeout 400 python bench.py > gpurun_out/r2x_bench_c2.json 2> gpurun_out/r2x_bench_c2.err
python -c "import json; d=json.loads(open('gpurun_out/r2x_bench_c2.json').read().strip().splitlines()[-1]); r=d['roofline']; print(d['ms_per_step'], d['value'], r['frac'], r['launch_ms'], d['e2e']['value'], d['clocks']['reasons'], d['cpu_baseline']['value'])"
