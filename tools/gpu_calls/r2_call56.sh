# k_query_bins shift + k_adamw_keys 32-node tiles of 256 threads: GPU suite, step trace, bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2c56_pytest.txt 2>&1; tail -1 gpurun_out/r2c56_pytest.txt
timeout 300 python tools/step_kernels.py --steps 10 --graph > gpurun_out/r2c56_graph.txt 2>&1; grep "span" gpurun_out/r2c56_graph.txt; grep -E "k_query_bins|k_adamw_keys" gpurun_out/r2c56_graph.txt | head -2
for r in 1 2 3; do python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["ms_per_step"], r["frac"], r["launch_ms"])'; done
