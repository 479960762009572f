# tiled k_adamw_keys + item record loaded once in k_fit: GPU suite, bench, launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2c44_pytest.txt 2>&1; tail -2 gpurun_out/r2c44_pytest.txt
for r in 1 2; do python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["ms_per_step"], r["frac"], r["launch_ms"])'; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r2c44_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
grep -c k_adamw_keys gpurun_out/r2c44_launches.csv
