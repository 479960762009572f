# k_adamw_keys (AdamW + S0 key records fused): full GPU suite, bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2c36_pytest.txt 2>&1
tail -3 gpurun_out/r2c36_pytest.txt
for r in 1 2; do python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["ms_per_step"], r["frac"], r["launch_ms"], d["gpu_launches"])'; done > gpurun_out/r2c36_bench.txt
cat gpurun_out/r2c36_bench.txt
